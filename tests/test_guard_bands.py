"""Bounds checks of our own around every kernel (the memcheck/initcheck substitute:
compute-sanitizer is closed on the GPU pool, see test_sanitizer.py).

Each operand lives inside a larger buffer: guard bands before and after it and the
padding columns of a strided leading dimension hold a signalling-NaN canary bit
pattern. After each call
  * the guards and padding of C are bit-identical to the canary (no stray stores),
  * no canary is left inside C (every element written — the initcheck condition),
  * C is within the order-independent fp32/fp64 γ-bound of the fp64 oracle
    (a read of a B guard or padding element would carry a NaN into the sum),
  * B's buffer, guards included, is unchanged (kernels never write their inputs).
Coverage follows tools/sanitize.py: the 8 design points, fast and exact, f32 and f64,
W 4/32, N 1..128 incl. ragged widths, odd leading dimensions and a C offset by one
element (vector width planning), plus the forced launch variants (lean RB, TMA gather4
EB, shared-memory B window, row-panel tiles, CM lanes over rows) and the replicated
row epilogue (spmm_rows_to)."""
import os

import numpy as np
import pytest

import helpers as H
from oracle import oracle as O

GUARD = 4096  # elements on each side
CANARY32 = np.uint32(0x7FA0DEAD)  # signalling NaN payloads no kernel produces
CANARY64 = np.uint64(0x7FF4DEADBEEF0001)


def _canary_tensor(n, dt, dev):
    import torch

    if dt == torch.float32:
        return torch.full((n,), int(CANARY32.view(np.int32)), dtype=torch.int32,
                          device=dev).view(torch.float32)
    return torch.full((n,), int(CANARY64.view(np.int64)), dtype=torch.int64,
                      device=dev).view(torch.float64)


def _bits(t):
    import torch

    return t.view(torch.int32 if t.dtype == torch.float32 else torch.int64)


class Guarded:
    """rows x cols view with leading dimension ld inside a canary-filled buffer;
    `shift` offsets the view by that many elements (misaligned operands)."""

    def __init__(self, rows, cols, ld, dt, dev, shift=0):
        self.rows, self.cols, self.ld, self.shift = rows, cols, ld, shift
        self.n_in = rows * ld
        self.buf = _canary_tensor(2 * GUARD + shift + self.n_in, dt, dev)
        self.base = GUARD + shift
        self.view = self.buf[self.base:self.base + self.n_in].view(rows, ld)[:, :cols]

    def canary_mask(self):
        import torch

        m = torch.ones(self.buf.numel(), dtype=torch.bool, device=self.buf.device)
        inner = m[self.base:self.base + self.n_in].view(self.rows, self.ld)
        inner[:, :self.cols] = False
        return m

    def intact_outside(self):
        c = _canary_tensor(1, self.buf.dtype, self.buf.device)
        m = self.canary_mask()
        return bool((_bits(self.buf)[m] == _bits(c)[0]).all())

    def any_canary_inside(self):
        c = _canary_tensor(1, self.buf.dtype, self.buf.device)
        return bool((_bits(self.view.contiguous()) == _bits(c)[0]).any())


def _operands(a, n, dt, dev, cm, ld_pad, shift, seed):
    import torch

    g = torch.Generator(device="cpu").manual_seed(seed)
    K = a.num_cols
    host = torch.rand(K, n, generator=g, dtype=torch.float64) * 2 - 1
    if cm:
        B = Guarded(n, K, K + ld_pad, dt, dev)
        B.view.copy_(host.t().to(dt))
    else:
        B = Guarded(K, n, n + ld_pad, dt, dev)
        B.view.copy_(host.to(dt))
    C = Guarded(a.num_rows, n, n + ld_pad, dt, dev, shift=shift)
    x = host.to(dt).to(torch.float64).numpy()
    return B, C, x


def _check(a, B, C, x, dtype, before_b, what):
    assert C.intact_outside(), f"{what}: store outside C (guard band or padding changed)"
    assert not C.any_canary_inside(), f"{what}: element of C never written"
    assert bool((_bits(B.buf) == before_b).all()), f"{what}: B's buffer was written"
    y = C.view.double().cpu().numpy()
    y64 = O.spmm_reference(H.to_oracle(a), x)
    bound = H.gamma_bound(a, x, dtype)
    err = np.abs(y - y64)
    assert np.all(np.isfinite(y)), f"{what}: non-finite output (a guard or padding read?)"
    assert np.all(err <= bound), f"{what}: max err {err.max():.3e} over the γ-bound"


def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_every_design_point_stays_in_bounds(dtype):
    torch = _gpu()
    from paper_2202_08556_b200 import spmmkit as sk

    dt = torch.float32 if dtype == np.float32 else torch.float64
    a = H.random_csr(700, 600, 9000, seed=4, dtype=dtype, skew=1.4)
    d = sk.DeviceCsr.from_host(a)
    cases = [(1, 0, 0), (2, 0, 0), (3, 1, 1), (4, 0, 0), (8, 3, 1), (16, 0, 0), (33, 2, 0),
             (64, 0, 2), (128, 0, 0)]
    for n, ld_pad, shift in cases:
        for k in range(8):
            cm = bool(k & 2)
            B, C, x = _operands(a, n, dt, "cuda", cm, ld_pad, shift, seed=n * 8 + k)
            before_b = _bits(B.buf).clone()
            for exact in (False, True):
                for W in (4, 32):
                    C.view.copy_(_canary_tensor(C.view.numel(), dt, "cuda").view(C.rows, n))
                    sk.spmm_device(k, d, B.view, C.view, W=W, P=(64 if exact else 0),
                                   exact=exact)
                    torch.cuda.synchronize()
                    _check(a, B, C, x, dtype, before_b,
                           f"k={k} n={n} ld+{ld_pad} shift={shift} exact={exact} W={W}")


def _banded(n_rows=2000, half=4):
    from paper_2202_08556_b200 import spmmkit as sk

    rows = np.repeat(np.arange(n_rows), 2 * half + 1)
    cols = rows + np.tile(np.arange(-half, half + 1), n_rows)
    keep = (cols >= 0) & (cols < n_rows)
    rp = np.concatenate([[0], np.cumsum(np.bincount(rows[keep], minlength=n_rows))])
    return sk.CsrMatrix(n_rows, n_rows, rp.astype(np.int64), cols[keep].astype(np.int64),
                        np.random.default_rng(1).uniform(-1, 1, keep.sum()).astype(np.float32),
                        np.float32)


# (environment, kernel id, matrix, widths): the opt-in and forced launch variants
VARIANTS = [
    ({"DASPMM_LEAN_RB": "1"}, 0, "skewed", (8, 16, 33, 128)),
    ({"DASPMM_TMA": "1"}, 4, "skewed", (32, 64, 100, 128)),
    ({"DASPMM_WIN": "1"}, 0, "banded", (2, 8, 32, 128)),
    ({"DASPMM_TILE": "2", "DASPMM_TILE_RL": "1"}, 0, "banded", (1, 2, 16, 33, 128, 200)),
    ({"DASPMM_TILE": "2", "DASPMM_TILE_RL": "8"}, 0, "banded", (1, 4, 8, 64, 200)),
    ({"DASPMM_CM_ROWS": "2"}, 2, "banded", (1, 3, 8, 13, 64)),
    ({"DASPMM_EB_CHUNK": "256"}, 4, "skewed", (2, 16, 64, 128)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("env,k,mat,widths", VARIANTS,
                         ids=[",".join(f"{a}={b}" for a, b in v[0].items()) for v in VARIANTS])
def test_launch_variants_stay_in_bounds(env, k, mat, widths):
    torch = _gpu()
    from paper_2202_08556_b200 import spmmkit as sk

    a = H.random_csr(700, 600, 9001, seed=5, dtype=np.float32, skew=1.2) if mat == "skewed" \
        else _banded()
    d = sk.DeviceCsr.from_host(a)
    saved = {key: os.environ.get(key) for key in env}
    os.environ.update(env)
    sk.reload_env()
    try:
        for n in widths:
            for ld_pad, shift in ((0, 0), (3, 1)):
                B, C, x = _operands(a, n, torch.float32, "cuda", bool(k & 2), ld_pad, shift,
                                    seed=n)
                before_b = _bits(B.buf).clone()
                sk.spmm_device(k, d, B.view, C.view)
                torch.cuda.synchronize()
                _check(a, B, C, x, np.float32, before_b, f"{env} k={k} n={n} ld+{ld_pad}")
    finally:
        for key, v in saved.items():
            if v is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = v
        sk.reload_env()


@pytest.mark.gpu
def test_replicated_epilogue_stays_in_bounds():
    torch = _gpu()
    from paper_2202_08556_b200 import spmmkit as sk

    a = _banded()
    d = sk.DeviceCsr.from_host(a)
    for n in (3, 32, 128):
        B, C0, x = _operands(a, n, torch.float32, "cuda", False, 0, 0, seed=n)
        outs = [C0] + [Guarded(a.num_rows, n, n, torch.float32, "cuda") for _ in range(2)]
        before_b = _bits(B.buf).clone()
        sk.spmm_rows_to(d, B.view, [o.view for o in outs])
        torch.cuda.synchronize()
        for i, o in enumerate(outs):
            _check(a, B, o, x, np.float32, before_b, f"rows_to n={n} destination {i}")
