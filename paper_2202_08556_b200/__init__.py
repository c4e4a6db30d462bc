"""paper_2202_08556_b200 — B200-native DA-SpMM (arXiv 2202.08556) behind spmmkit's API.

The compute lives in libdaspmm.so (hand-written sm_100a CUDA, C-ABI in
include/daspmm.h). This package holds its ctypes binding (`_lib`), the reference-
named host API (`spmmkit`), the multi-GPU row-panel layer (`multi`), the synthetic
input generators used by tests and bench (`gen`), and the in-tree build (`build`).
"""
from . import _lib  # noqa: F401

__version__ = "0.1.0"


def load():
    """Load the CUDA library (raises if it was not built — no CPU fallback)."""
    return _lib.lib()
