"""RB+CM+SR with lanes over rows (csrc/spmm_cm.cu): the launch variant of the column-major
design point. Same fmaf sequence per output as the base walk (lanes over columns), so
bit-identical in fast mode; within the fp64 oracle's gamma bound; every N (column blocks
of 1..8), padded leading dimensions, empty rows."""
import os

import numpy as np
import pytest

import helpers as H
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sk():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2202_08556_b200 import spmmkit

    spmmkit.lib()
    return spmmkit


def _run(sk, d, Bcm, n, rows_variant: bool):
    import torch

    os.environ["DASPMM_CM_ROWS"] = "2" if rows_variant else "0"  # 2: skewed rows too
    sk.reload_env()
    try:
        C = torch.full((d.num_rows, n), float("nan"), device="cuda")
        sk.spmm_device(2, d, Bcm, C)
        v = sk.plan_info(2, d, Bcm, C)[0]
        torch.cuda.synchronize()
        return C, v
    finally:
        os.environ.pop("DASPMM_CM_ROWS", None)
        sk.reload_env()


@pytest.mark.parametrize("skew", [0.0, 1.3])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 13, 32, 64, 128])
def test_cm_rows_bit_identical_and_within_gamma(sk, n, skew):
    import torch

    a = H.random_csr(3001, 2500, 40000, seed=31 + n, dtype=np.float32, skew=skew)
    d = sk.DeviceCsr.from_host(a)
    x = np.random.default_rng(n).uniform(-1, 1, (a.num_cols, n)).astype(np.float32)
    Bcm = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()  # N x K buffer
    Cb, vb = _run(sk, d, Bcm, n, False)
    Cr, vr = _run(sk, d, Bcm, n, True)
    assert vr == "cm_rows" and vb != "cm_rows"
    assert torch.equal(Cb, Cr)
    y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
    err = np.abs(Cr.cpu().numpy().astype(np.float64) - y64)
    assert (err <= H.gamma_bound(a, x, np.float32)).all()


def test_cm_rows_default_gate(sk):
    """By default lanes-over-rows serves unskewed rows only (a lane alone on a long row
    stalls its warp); skewed rows keep the base walk."""
    import torch

    for skew, want in ((0.0, True), (1.3, False)):
        a = H.random_csr(3001, 2500, 40000, seed=5, dtype=np.float32, skew=skew)
        d = sk.DeviceCsr.from_host(a)
        Bcm = torch.rand(16, 2500, device="cuda")
        C = torch.empty(3001, 16, device="cuda")
        assert (sk.plan_info(2, d, Bcm, C)[0] == "cm_rows") == want


def test_cm_rows_padded_ld_and_empty_rows(sk):
    import torch

    a = H.csr_from_counts([6, 2, 0, 3, 1, 0, 0, 9] * 50, 40, dtype=np.float32)
    d = sk.DeviceCsr.from_host(a)
    n = 11
    x = np.random.default_rng(3).uniform(-1, 1, (40, n)).astype(np.float32)
    buf = torch.zeros(n, 44, device="cuda")  # ldb = 44 > K
    buf[:, :40] = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    Bcm = buf[:, :40]
    Cw = torch.full((a.num_rows, 16), 5.0, device="cuda")
    sk.spmm_device(2, d, Bcm, Cw[:, :n])
    torch.cuda.synchronize()
    assert sk.plan_info(2, d, Bcm, Cw[:, :n])[0] == "cm_rows"
    y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
    err = np.abs(Cw[:, :n].cpu().numpy().astype(np.float64) - y64)
    assert (err <= H.gamma_bound(a, x, np.float32)).all()
    assert bool((Cw[:, n:] == 5.0).all())
