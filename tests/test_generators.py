"""The device synthetic-matrix generators (paper_2202_08556_b200/gen.py) against the
reference's R-MAT generator (proj/include/spmmkit/rmat.hpp:46-99, run unmodified through
oracle/_ref) — CPU tests (torch on the host device).

The two draw different random streams (the reference: one mt19937_64 sequence; gen.py:
batched torch draws on the GPU), so equality is statistical for the structure and exact
for the contract: distinct sorted cells, exactly the target count when reachable, the 10x
draw cap with the 0.99 shortfall error, values in (0, 1], and the parameter checks."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O


def _ref_rmat(scale, nnz, a, b, c, d, seed):
    R = O.ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    h = R.ref_rmat(scale, nnz, a, b, c, d, seed)
    if not h:
        return None, R.ref_last_error().decode()
    M, K, n = C.c_int64(), C.c_int64(), C.c_int64()
    R.ref_csr_info(h, C.byref(M), C.byref(K), C.byref(n))
    rp = np.zeros(M.value + 1, np.int64)
    ci = np.zeros(n.value, np.int64)
    va = np.zeros(n.value, np.float64)
    R.ref_csr_copy(h, rp, ci, va)
    R.ref_csr_free(h)
    return (rp, ci, va), None


def _gen_rmat(scale, nnz, a, b, c, d, seed):
    import torch

    from paper_2202_08556_b200 import gen

    M, K, rp, ci, va = gen.rmat(scale, nnz, a, b, c, d, seed=seed, dtype=torch.float64,
                                device="cpu")
    return rp.numpy().astype(np.int64), ci.numpy().astype(np.int64), va.numpy()


def _contract(rp, ci, va, M, nnz):
    assert rp[0] == 0 and rp[-1] == ci.size == va.size
    assert (np.diff(rp) >= 0).all()
    keys = np.repeat(np.arange(M), np.diff(rp)) * (1 << 31) + ci
    assert (np.diff(keys) > 0).all()  # sorted by (row, col), no duplicate cell
    assert (va > 0).all() and (va <= 1).all()
    assert ci.size == nnz


@pytest.mark.parametrize("params", [(12, 16 * 4096, 0.25, 0.25, 0.25, 0.25),
                                    (12, 16 * 4096, 0.57, 0.19, 0.19, 0.05),
                                    (13, 8 * 8192, 0.45, 0.22, 0.22, 0.11)])
def test_rmat_structure_matches_reference(params):
    scale, nnz, a, b, c, d = params
    (rp_r, ci_r, va_r), err = _ref_rmat(scale, nnz, a, b, c, d, 7)
    assert err is None
    rp_g, ci_g, va_g = _gen_rmat(scale, nnz, a, b, c, d, 7)
    M = 1 << scale
    _contract(rp_r, ci_r, va_r, M, nnz)
    _contract(rp_g, ci_g, va_g, M, nnz)
    lr, lg = np.diff(rp_r).astype(float), np.diff(rp_g).astype(float)
    # same quadrant-descent distribution: row-length moments and extremes agree
    assert abs(lg.std() / lr.std() - 1) < 0.05, (lr.std(), lg.std())
    assert abs(lg.max() / lr.max() - 1) < 0.2, (lr.max(), lg.max())
    assert abs((lg == 0).mean() - (lr == 0).mean()) < 0.02
    cr = np.bincount(ci_r, minlength=M).astype(float)
    cg = np.bincount(ci_g, minlength=M).astype(float)
    assert abs(cg.std() / cr.std() - 1) < 0.05
    # values: uniform on (0, 1]
    assert abs(va_g.mean() - 0.5) < 0.01 and abs(va_r.mean() - 0.5) < 0.01


def test_rmat_draw_cap_and_parameter_checks():
    import torch

    from paper_2202_08556_b200 import gen

    # a target too dense for the skew: the reference exhausts its 10x draw cap and
    # throws; the device generator refuses the same way
    _, err = _ref_rmat(6, 3000, 0.9, 0.04, 0.04, 0.02, 1)
    assert err is not None and "draw cap" in err
    with pytest.raises(RuntimeError, match="draw cap exhausted"):
        gen.rmat(6, 3000, 0.9, 0.04, 0.04, 0.02, seed=1, device="cpu")
    for bad in [dict(scale=31, nnz=1), dict(scale=4, nnz=300), dict(scale=4, nnz=10, a=0.5)]:
        args = dict(a=0.25, b=0.25, c=0.25, d=0.25, seed=0, device="cpu")
        args.update({k: v for k, v in bad.items() if k in "abcd"})
        with pytest.raises(ValueError):
            gen.rmat(bad["scale"], bad["nnz"], args["a"], args["b"], args["c"], args["d"],
                     seed=0, device="cpu")
    # uniform parameters: the uniform generator and R-MAT 0.25^4 agree on the row spread
    M, K, rp, ci, va = gen.uniform(4096, 4096, 65536, seed=3, dtype=torch.float64, device="cpu")
    _contract(rp.numpy().astype(np.int64), ci.numpy().astype(np.int64), va.numpy(), 4096, 65536)
