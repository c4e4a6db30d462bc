"""Dense row-panel tiles (csrc/tile.cuh): the RB+RM+SR launch variant for row-local
matrices. It must (1) be chosen only when the tiles pay (rows column-sorted, tiles at
least half full), (2) give the base walk's bits (same fmaf sequence per output), (3) hold
the fp64 oracle's gamma bound, and (4) propagate Inf / NaN exactly as the reference
(spmm.hpp:85-88): an absent entry must never turn a non-finite B element into NaN."""
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


def _banded(rows, b, seed, cols=None, drop=0.0):
    """Row r holds columns [r - b, r + b] (clipped), a fraction `drop` removed at random."""
    from paper_2202_08556_b200.spmmkit import CsrMatrix

    cols = cols or rows
    rng = np.random.default_rng(seed)
    rp, ci = [0], []
    for r in range(rows):
        c = np.arange(max(0, r - b), min(cols, r + b + 1))
        if drop > 0:
            c = c[rng.random(c.size) >= drop]
        ci.extend(c.tolist())
        rp.append(len(ci))
    ci = np.asarray(ci, np.int64)
    return CsrMatrix(rows, cols, np.asarray(rp, np.int64), ci,
                     rng.uniform(-1, 1, ci.size).astype(np.float32), np.float32)


def _run(sk, d, B, tile: bool, rl: int = 0):
    """One RB+RM+SR call with the tile walk forced on (DASPMM_TILE=2: any grid size, so
    test-sized matrices take it) or off; rl forces its row lanes (1 or 8)."""
    import torch

    os.environ["DASPMM_TILE"] = "2" if tile else "0"
    if rl:
        os.environ["DASPMM_TILE_RL"] = str(rl)
    sk.reload_env()
    try:
        C = torch.full((d.num_rows, B.shape[1]), float("nan"), device="cuda")
        sk.spmm_device(0, d, B, C)
        variant = sk.plan_info(0, d, B, C)[0]
        torch.cuda.synchronize()
        return C, variant
    finally:
        os.environ.pop("DASPMM_TILE", None)
        os.environ.pop("DASPMM_TILE_RL", None)
        sk.reload_env()


@pytest.mark.parametrize("case", ["banded_b8", "banded_b4_ragged", "banded_b8_dropped",
                                  "short_last_panel", "empty_rows"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8, 16, 32, 33, 64, 128, 200])
def test_tiles_bit_identical_to_base_and_within_gamma(sk, case, n):
    import torch

    if case == "banded_b8":
        a = _banded(3000, 8, 1)
    elif case == "banded_b4_ragged":
        a = _banded(2501, 4, 2, cols=2600)
    elif case == "banded_b8_dropped":
        a = _banded(4000, 8, 3, drop=0.2)
    elif case == "short_last_panel":
        a = _banded(1003, 5, 4)
    else:  # empty rows and whole empty panels inside a band
        a = _banded(2048, 6, 5)
        rp = a.row_offsets.copy()
        keep = np.ones(a.num_rows, bool)
        keep[100:130] = False  # rows 100..129 emptied (panels 13..15 empty)
        keep[777] = False
        lens = np.diff(rp) * keep
        new_rp = np.concatenate([[0], np.cumsum(lens)])
        ci = np.concatenate([a.col_indices[rp[r]:rp[r + 1]] for r in range(a.num_rows) if keep[r]])
        va = np.concatenate([a.values[rp[r]:rp[r + 1]] for r in range(a.num_rows) if keep[r]])
        a = sk.CsrMatrix(a.num_rows, a.num_cols, new_rp.astype(np.int64), ci.astype(np.int64),
                         va.astype(np.float32), np.float32)
    d = sk.DeviceCsr.from_host(a)
    B = torch.rand(a.num_cols, n, device="cuda") * 2 - 1
    Cb, vb = _run(sk, d, B, False)
    Ct, vt = _run(sk, d, B, True)
    assert vt == "rb_tile", vt
    assert vb != "rb_tile"
    assert torch.equal(Cb, Ct), "tile walk must reproduce the base walk bit for bit"
    x64 = B.cpu().numpy().astype(np.float64)
    y64 = O.spmm_reference(H.to_oracle(a), x64)
    err = np.abs(Ct.cpu().numpy().astype(np.float64) - y64)
    assert (err <= H.gamma_bound(a, x64, np.float32)).all()


@pytest.mark.parametrize("rl", [1, 8])
@pytest.mark.parametrize("n", [1, 2, 4, 8, 16])
def test_tiles_both_row_mappings(sk, rl, n):
    """Narrow N runs either a lane per row (RL = 8) or a lane per column slot with all
    eight rows (RL = 1): both give the base walk's bits."""
    import torch

    a = _banded(1777, 8, 21)
    d = sk.DeviceCsr.from_host(a)
    B = torch.rand(a.num_cols, n, device="cuda") - 0.5
    Cb, _ = _run(sk, d, B, False)
    Ct, vt = _run(sk, d, B, True, rl=rl)
    assert vt == "rb_tile"
    assert torch.equal(Cb, Ct)


def test_tiles_default_only_on_large_grids(sk):
    """Without forcing, the tile walk needs >= 65536 threads (8-row panels x lanes):
    a 2^20-row banded matrix takes it, a 3000-row one keeps the base walk."""
    import torch

    from paper_2202_08556_b200 import gen

    M, K, rp, ci, va = gen.banded(1 << 20, 8, seed=3)
    big = sk.DeviceCsr.from_device(M, K, rp, ci, va)
    B = torch.rand(K, 32, device="cuda")
    C = torch.empty(M, 32, device="cuda")
    assert sk.plan_info(0, big, B, C)[0] == "rb_tile"
    small = sk.DeviceCsr.from_host(_banded(3000, 8, 1))
    Bs = torch.rand(3000, 32, device="cuda")
    Cs = torch.empty(3000, 32, device="cuda")
    assert sk.plan_info(0, small, Bs, Cs)[0] != "rb_tile"


def test_tiles_strided_operands(sk):
    """B and C with leading dimensions above N (views into wider buffers)."""
    import torch

    a = _banded(1500, 8, 7)
    d = sk.DeviceCsr.from_host(a)
    Bw = torch.rand(a.num_cols, 40, device="cuda")
    B = Bw[:, :36]
    os.environ["DASPMM_TILE"] = "0"
    sk.reload_env()
    Cw0 = torch.full((a.num_rows, 44), 7.0, device="cuda")
    sk.spmm_device(0, d, B, Cw0[:, :36])
    os.environ["DASPMM_TILE"] = "2"
    sk.reload_env()
    Cw1 = torch.full((a.num_rows, 44), 7.0, device="cuda")
    sk.spmm_device(0, d, B, Cw1[:, :36])
    assert sk.plan_info(0, d, B, Cw1[:, :36])[0] == "rb_tile"
    os.environ.pop("DASPMM_TILE", None)
    sk.reload_env()
    torch.cuda.synchronize()
    assert torch.equal(Cw0, Cw1)
    assert bool((Cw1[:, 36:] == 7.0).all()), "columns past N must stay untouched"


def test_tiles_nonfinite_b_matches_base(sk):
    """Inf / NaN rows of B that some rows of a panel do not reference: the tile walk's
    0 * Inf would be NaN; the CSR replay must give the base (and reference) results."""
    import torch

    a = _banded(2000, 8, 9)
    d = sk.DeviceCsr.from_host(a)
    B = torch.rand(a.num_cols, 32, device="cuda")
    B[1000, :] = float("inf")
    B[1500, 3] = float("nan")
    B[20, 7] = float("-inf")
    Cb, _ = _run(sk, d, B, False)
    Ct, vt = _run(sk, d, B, True)
    assert vt == "rb_tile"
    assert torch.equal(Cb.isnan(), Ct.isnan())
    assert torch.equal(Cb.nan_to_num(0.5), Ct.nan_to_num(0.5))
    # rows far from the poisoned columns stay finite (no spurious NaN from 0 * Inf)
    assert bool(Ct[1200:1400].isfinite().all())
    x = B.cpu().numpy().astype(np.float64)
    y = O.spmm_reference(H.to_oracle(a), x)
    assert np.array_equal(np.isnan(y), Ct.isnan().cpu().numpy())
    assert np.array_equal(np.isposinf(y), Ct.isposinf().cpu().numpy())


def test_tiles_not_used_where_they_do_not_pay(sk):
    """Scattered columns (fill far below 1/2) and rows listed out of column order keep
    the base walk."""
    import torch

    os.environ["DASPMM_TILE"] = "2"  # any grid size: only eligibility decides
    sk.reload_env()
    u = H.random_csr(3000, 3000, 48000, seed=11, dtype=np.float32)
    d = sk.DeviceCsr.from_host(u)
    B = torch.rand(3000, 32, device="cuda")
    C = torch.empty(3000, 32, device="cuda")
    assert sk.plan_info(0, d, B, C)[0] != "rb_tile"
    a = _banded(1000, 8, 12)
    rp, ci, va = a.row_offsets, a.col_indices.copy(), a.values.copy()
    ci[rp[500]:rp[501]] = ci[rp[500]:rp[501]][::-1].copy()  # one row in descending order
    va[rp[500]:rp[501]] = va[rp[500]:rp[501]][::-1].copy()
    b = sk.CsrMatrix(1000, 1000, rp, ci, va, np.float32)
    db = sk.DeviceCsr.from_host(b)
    B = torch.rand(1000, 32, device="cuda")
    C = torch.empty(1000, 32, device="cuda")
    assert sk.plan_info(0, db, B, C)[0] != "rb_tile"
    sk.spmm_device(0, db, B, C)
    x64 = B.cpu().numpy().astype(np.float64)
    y64 = O.spmm_reference(H.to_oracle(b), x64)
    assert (np.abs(C.cpu().numpy() - y64) <= H.gamma_bound(b, x64, np.float32)).all()
    os.environ.pop("DASPMM_TILE", None)
    sk.reload_env()


def test_tiles_through_da_spmm(sk):
    """DA-SpMM (device selector, graph and direct paths) on a banded matrix: when the
    selector picks RB+RM+SR the tile walk serves it; results hold the gamma bound."""
    import torch

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    model = sk.load_selector(open(os.path.join(root, "paper_2202_08556_b200", "models",
                                               "b200_selector.txt")).read())
    os.environ["DASPMM_TILE"] = "2"
    sk.reload_env()
    a = _banded(20000, 8, 13)
    d = sk.DeviceCsr.from_host(a)
    for n in (8, 64, 128):
        B = torch.rand(a.num_cols, n, device="cuda") - 0.5
        C = torch.full((a.num_rows, n), float("nan"), device="cuda")
        kout = torch.zeros(1, dtype=torch.int32, device="cuda")
        for _ in range(2):  # graph path, then the published direct path
            sk.spmm_selected(d, model, B, C, kernel_out=kout)
        torch.cuda.synchronize()
        x64 = B.cpu().numpy().astype(np.float64)
        y64 = O.spmm_reference(H.to_oracle(a), x64)
        err = np.abs(C.cpu().numpy().astype(np.float64) - y64)
        assert (err <= H.gamma_bound(a, x64, np.float32)).all()
    os.environ.pop("DASPMM_TILE", None)
    sk.reload_env()


def test_tiles_follow_values_updated(sk):
    """A borrowed CSR whose values change in place: after values_updated() the tile walk
    uses the new values (the tiles are a copy)."""
    import torch

    from paper_2202_08556_b200 import gen

    M, K, rp, ci, va = gen.banded(1 << 17, 8, seed=9)
    d = sk.DeviceCsr.from_device(M, K, rp, ci, va)  # borrows va
    B = torch.rand(K, 32, device="cuda")
    C1 = torch.empty(M, 32, device="cuda")
    sk.spmm_device(0, d, B, C1)
    assert sk.plan_info(0, d, B, C1)[0] == "rb_tile"
    va.mul_(-2.0)  # exact in fp32
    d.values_updated()
    C2 = torch.empty(M, 32, device="cuda")
    sk.spmm_device(0, d, B, C2)
    torch.cuda.synchronize()
    assert torch.equal(C2, -2.0 * C1)
