"""CPU tests of the C-ABI library: every declared symbol is exported, the host-side
selector path (model parse + predict_kernel) reproduces the reference's predictions
on its golden probes, errors map to the reference's exception kinds, and the product
refuses to compute without a GPU (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sk():
    from paper_2202_08556_b200 import build

    build.build()
    from paper_2202_08556_b200 import spmmkit

    spmmkit.lib()
    return spmmkit


def test_library_exports_every_declared_symbol(sk):
    from paper_2202_08556_b200 import _lib

    header = open(os.path.join(ROOT, "include", "daspmm.h")).read()
    declared = set(re.findall(r"\b(daspmm_[a-z0-9_]+)\s*\(", header))
    assert len(declared) >= 20
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)


@pytest.mark.parametrize("tag", ["plain", "unified"])
def test_host_predict_matches_reference_golden(sk, golden, tag):
    text = open(os.path.join(ROOT, "tests", "golden", f"selector_{tag}.txt")).read()
    m = sk.load_selector(text)
    assert m.uses_hardware == (tag == "unified")
    probes, preds = golden[f"selector_{tag}/probes"], golden[f"selector_{tag}/preds"]
    for p, want in zip(probes, preds):
        f = sk.FeatureVector(int(p[0]), int(p[1]), float(p[2]), int(p[3]),
                             int(p[4]) if tag == "unified" else None)
        assert sk.predict_kernel(m, f).index() == want


def test_model_format_errors(sk):
    text = open(os.path.join(ROOT, "tests", "golden", "selector_plain.txt")).read()
    with pytest.raises(sk.ModelFormatError, match="not a selector stream"):
        sk.load_selector("spmmkit-gbdt v1\n")
    with pytest.raises(sk.ModelFormatError, match="unsupported selector version"):
        sk.load_selector(text.replace("spmmkit-selector v1", "spmmkit-selector v2"))
    with pytest.raises(sk.ModelFormatError, match="truncated"):
        sk.load_selector(text[: len(text) // 2])
    with pytest.raises(sk.ModelFormatError, match="tree out of order"):
        sk.load_selector(text.replace("tree 0 1 ", "tree 0 2 ", 1))
    m = sk.load_selector(text)
    with pytest.raises(ValueError, match="hardware_id"):
        sk.predict_kernel(sk.load_selector(open(os.path.join(
            ROOT, "tests", "golden", "selector_unified.txt")).read()), sk.FeatureVector(1, 1, 0.0, 4))
    assert sk.predict_kernel(m, sk.FeatureVector(0, 0, 0.0, 4)).index() in range(8)


def test_host_logic_mirrors_reference(sk):
    """kernel_id.hpp / worker.hpp semantics (test_spmm.cpp:283-293 and friends)."""
    K = sk.KernelId
    assert [K.from_index(i).name() for i in range(8)] == [
        "RB+RM+SR", "RB+RM+PR", "RB+CM+SR", "RB+CM+PR", "EB+RM+SR", "EB+RM+PR", "EB+CM+SR",
        "EB+CM+PR"]
    assert all(K.parse(K.from_index(i).name()).index() == i for i in range(8))
    assert K.parse("RB+RM+XX") is None and K.parse("RBRM+SR") is None
    assert sk.recommended_col_block(K.parse("RB+RM+PR"), 100) == 4
    assert sk.recommended_col_block(K.parse("RB+RM+SR"), 100) == 8
    assert sk.recommended_col_block(K.parse("EB+CM+PR"), 2) == 2
    assert sk.recommended_col_block(K.parse("EB+CM+SR"), 1) == 1
    cfg = sk.make_config(K.from_index(1), 16, 3, 4)
    assert (cfg.num_workers, cfg.group_width, cfg.col_block) == (3, 4, 4) and sk.is_valid(cfg)
    assert len(sk.validate_config(sk.WorkerConfig(0, 3, 0))) == 3


def test_no_cpu_fallback(sk):
    """Without a device the library refuses to build a handle (it never computes on
    the host)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        sk.DeviceCsr.from_host(sk.CsrMatrix.identity(4))
    with pytest.raises(RuntimeError):
        sk.spmm(sk.KernelId.from_index(0), sk.CsrMatrix.identity(4),
                sk.DenseMatrix.from_logical(np.ones((4, 2))), sk.WorkerConfig())
