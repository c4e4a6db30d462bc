"""TEST INFRASTRUCTURE ONLY — row- and column-sampled parity for full-size calls.

Rows of C depend only on the same rows of A, columns of C only on the same columns of B
(spmm_reference, proj/include/spmmkit/spmm.hpp:16-32). So any row subset x column subset
of a device result can be checked exactly against the fp64 oracle on the sub-problem:
the sampled rows of A (gathered on the device), the B rows they reference (renumbered),
and the sampled columns. The bound is the order-independent one of SURVEY §8c:

    |y - y64| <= 2 * gamma(len + 1) * sum_e |a_e * x_e| + 1e-30,
    gamma(n) = n u / (1 - n u),  u = 2^-24 (fp32) or 2^-53 (fp64)

Used by tests/test_gpu_scale.py and by bench.py's per-call parity map (outside the timed
region). Never imported by the product package.
"""
from __future__ import annotations

import numpy as np

from . import oracle as O


def sample_rows(rp_host: np.ndarray, n_random: int = 384, seed: int = 0,
                boundary_strides=(7, 12, 32, 64, 256, 448, 768, 2048), n_boundary: int = 48):
    """Random rows plus rows holding the elements where EB chunks / CTA tiles of the
    given strides begin (the split rows that take atomics), plus the first and last
    non-empty rows and one empty row if any."""
    M = rp_host.size - 1
    nnz = int(rp_host[-1])
    rng = np.random.default_rng(seed)
    picks = [rng.integers(0, M, size=min(n_random, M))] if M else []
    if nnz > 0:
        for s in boundary_strides:
            k = nnz // s
            if k < 1:
                continue
            e = rng.integers(0, k + 1, size=min(n_boundary, k + 1)) * s
            e = e[e < nnz]
            picks.append(np.searchsorted(rp_host, e, side="right") - 1)
        lens = np.diff(rp_host)
        nz = np.flatnonzero(lens)
        if nz.size:
            picks.append(np.array([nz[0], nz[-1]]))
        z = np.flatnonzero(lens == 0)
        if z.size:
            picks.append(z[:1])
    rows = np.unique(np.concatenate(picks)) if picks else np.zeros(0, np.int64)
    return rows.astype(np.int64)


def check(rp, ci, va, K, B, Cout, rows, cols=None, b_colmajor=False, dtype=None, row0=0,
          exact=False):
    """Check rows x cols of Cout (device M x N row-major) = A @ B on the sampled entries.
    ``row0``: Cout holds rows [row0, ...) of A only (a row panel's output).

    rp/ci/va: device CSR tensors (int32/int64 offsets and columns); B: device tensor,
    K x N row-major, or the N x K buffer of a column-major B when b_colmajor. Returns a
    dict with rows/cols checked, worst err/bound ratio and ok. ``exact``: ok only if
    every sampled entry equals spmm_reference's (fp64 sequential sum) bit for bit — the
    bar for the RB+SR kernels in exact mode on fp64 operands."""
    import torch

    dev = rp.device
    dtype = np.dtype(dtype or (np.float32 if va.dtype == torch.float32 else np.float64))
    u = 2.0 ** -24 if dtype == np.float32 else 2.0 ** -53
    rows_t = torch.as_tensor(rows, device=dev, dtype=torch.int64)
    s = rp[rows_t].to(torch.int64)
    e = rp[rows_t + 1].to(torch.int64)
    lens = e - s
    total = int(lens.sum().item())
    if total:
        starts = torch.repeat_interleave(s, lens)
        offs = torch.cumsum(lens, 0) - lens
        idx = starts + torch.arange(total, device=dev) - torch.repeat_interleave(offs, lens)
        sub_ci = ci[idx].to(torch.int64)
        sub_va = va[idx].to(torch.float64)
        U, inv = torch.unique(sub_ci, return_inverse=True)
    else:
        sub_ci = torch.zeros(0, dtype=torch.int64, device=dev)
        sub_va = torch.zeros(0, dtype=torch.float64, device=dev)
        U = torch.zeros(0, dtype=torch.int64, device=dev)
        inv = sub_ci
    n = B.shape[0] if b_colmajor else B.shape[1]
    cols_t = None if cols is None else torch.as_tensor(cols, device=dev, dtype=torch.int64)
    if b_colmajor:
        xs = B[:, U].t() if U.numel() else B.new_zeros(0, n)
    else:
        xs = B[U] if U.numel() else B.new_zeros(0, n)
    if cols_t is not None:
        xs = xs[:, cols_t]
    y = Cout[rows_t - row0]
    if cols_t is not None:
        y = y[:, cols_t]
    xs = xs.to(torch.float64).cpu().numpy()
    y = y.to(torch.float64).cpu().numpy()
    sub_rp = np.concatenate([[0], np.cumsum(lens.cpu().numpy())]).astype(np.int64)
    a = O.Csr(len(rows), max(int(U.numel()), 1), sub_rp, inv.cpu().numpy(),
              sub_va.cpu().numpy())
    if xs.shape[0] == 0:
        xs = np.zeros((1, xs.shape[1]))
    y64 = O.spmm_reference(a, xs)
    absa = O.Csr(a.num_rows, a.num_cols, a.row_offsets, a.col_indices, np.abs(a.values))
    mag = O.spmm_reference(absa, np.abs(xs))
    ln = np.diff(sub_rp).astype(np.float64)
    g = (ln + 1) * u / (1 - (ln + 1) * u)
    bound = 2 * g[:, None] * mag + 1e-30
    err = np.abs(y - y64)
    ratio = float((err / bound).max()) if err.size else 0.0
    return {"rows": int(len(rows)), "cols": int(y.shape[1]), "nnz": total,
            "max_ratio": ratio, "max_abs_err": float(err.max()) if err.size else 0.0,
            "nan": bool(np.isnan(y).any()),
            "ok": (bool(np.array_equal(y, y64)) if exact
                   else bool((err <= bound).all()) and not np.isnan(y).any())}
