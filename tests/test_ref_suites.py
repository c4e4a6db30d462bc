"""The reference's own hot-path GoogleTest suites (proj/tests/test_{types,partition,reduce,
features,spmm,matrix_market}.cpp), compiled UNCHANGED against include/spmmkit by
tests/cpp/build_ref_suites.py (gtest_shim for GoogleTest, the reference R-MAT generator
as the only reference header), run here.

CPU: the suites build (when the reference tree is present) and the host-only ones pass.
GPU: every suite passes with the compute on the B200 (spmm, partition_elements and
extract_features behind these headers run on the device).
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "cpp"))
import build_ref_suites as B  # noqa: E402

HOST_ONLY = ["test_types", "test_reduce", "test_matrix_market"]


def _run(name):
    exe = os.path.join(B.BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (needs the reference tree at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    tail = r.stdout[-3000:] + r.stderr[-3000:]
    assert r.returncode == 0, tail
    assert "[  PASSED  ]" in r.stdout
    return r.stdout


def test_reference_suites_build():
    if not os.path.isdir(B.REF_TESTS):
        pytest.skip("reference tree absent")
    from paper_2202_08556_b200 import build

    build.build()
    assert len(B.build()) == len(B.SUITES) + len(B.LOCAL)


@pytest.mark.parametrize("name", HOST_ONLY)
def test_reference_host_suites(name):
    _run(name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", B.SUITES)
def test_reference_suites_on_gpu(name):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = _run(name)
    print(out.splitlines()[-2])


@pytest.mark.gpu
def test_acceptance_gates_on_gpu():
    """C1 (38,400 kernel runs vs spmm_reference), C2, C8, C9 with spmm on the B200."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = _run("acceptance_b200")
    assert "4 tests" in out or "[  PASSED  ] 4 tests." in out
