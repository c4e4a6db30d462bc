"""Shared test helpers (test infrastructure; may use the oracle)."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


def csr_from_counts(counts, ncols, dtype=np.float64):
    """tests/test_util.hpp:39-46: columns packed from 0, value 1 + position."""
    from paper_2202_08556_b200.spmmkit import CsrMatrix

    rp = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    ci = np.concatenate([np.arange(c) for c in counts]).astype(np.int64) if rp[-1] else \
        np.zeros(0, np.int64)
    va = (1.0 + ci).astype(dtype)
    return CsrMatrix(len(counts), ncols, rp, ci, va, dtype)


def random_csr(rows, cols, nnz, seed, dtype=np.float64, skew=0.0):
    """Random CSR; skew > 0 gives power-law row lengths."""
    from paper_2202_08556_b200.spmmkit import CsrMatrix

    rng = np.random.default_rng(seed)
    if skew > 0:
        w = 1.0 / np.arange(1, rows + 1) ** skew
        rng.shuffle(w)
        lens = rng.multinomial(nnz, w / w.sum())
        lens = np.minimum(lens, cols)
    else:
        lens = rng.multinomial(nnz, np.ones(rows) / rows)
        lens = np.minimum(lens, cols)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(cols, size=l, replace=False)) if l else
                         np.zeros(0, np.int64) for l in lens]).astype(np.int64)
    va = rng.uniform(-1.0, 1.0, ci.size).astype(dtype)
    return CsrMatrix(rows, cols, rp, ci, va, dtype)


def to_oracle(a):
    return O.Csr(a.num_rows, a.num_cols, a.row_offsets, a.col_indices,
                 a.values.astype(np.float64))


def gamma_bound(a, x, dtype):
    """Order-independent error bound for an fp32/fp64 row sum:
    |y - y64| <= 2*gamma(len+1) * sum_e |a_e * x_e| (+ tiny), gamma(n)=n u/(1-n u)."""
    u = 2.0 ** -24 if np.dtype(dtype) == np.float32 else 2.0 ** -53
    lens = np.diff(a.row_offsets).astype(np.float64)
    g = (lens + 1) * u / (1 - (lens + 1) * u)
    absa = O.Csr(a.num_rows, a.num_cols, a.row_offsets, a.col_indices,
                 np.abs(a.values.astype(np.float64)))
    mag = O.spmm_reference(absa, np.abs(x.astype(np.float64)))
    return 2 * g[:, None] * mag + 1e-30


def split_rows(a, P):
    """Rows shared by >= 2 EB chunks of partition_elements(a, P)."""
    b, e, _ = O.partition_elements(to_oracle(a), P)
    rp = a.row_offsets
    s, t = rp[:-1], rp[1:]
    cnt = ((b[None, :] < t[:, None]) & (e[None, :] > s[:, None])).sum(1)
    return cnt >= 2
