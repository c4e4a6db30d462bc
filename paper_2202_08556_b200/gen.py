"""Synthetic CSR inputs for the BASELINE.json configs, generated on the GPU.

Input synthesis is not the hot path (the reference's R-MAT generator
is CPU-bound at ~1.8 us/nnz, far too slow for 10^8-10^9 nonzeros), so these use torch
for plumbing: quadrant descent in parallel, dedup by sort/unique, CSR by bincount.

  rmat(scale, nnz, a, b, c, d)   R-MAT quadrant descent (rmat.hpp:46-99 semantics:
                                 distinct cells, values in (0, 1]); uniform when
                                 a = b = c = d = 0.25
  uniform(rows, cols, nnz)       uniform random cells
  banded(rows, half_width)       row r holds columns [r - b, r + b] ∩ [0, cols)
  reddit_like()                  233K x 233K power-law graph with ~114.6M nnz
                                 (R-MAT s18, Graph500 skew, cropped)

Every generator returns (M, K, row_offsets int32, col_indices int32, values) as
CUDA tensors, sorted by (row, col) with no duplicate cells.
"""
from __future__ import annotations

import math

import torch

GRAPH500 = (0.57, 0.19, 0.19, 0.05)


def _to_csr(rows: torch.Tensor, cols: torch.Tensor, M: int, K: int, seed: int, dtype):
    key = rows.to(torch.int64) * K + cols.to(torch.int64)
    key = torch.unique(key)  # sorted, distinct
    r = (key // K).to(torch.int32)
    c = (key % K).to(torch.int32)
    del key
    counts = torch.bincount(r, minlength=M)
    rp = torch.zeros(M + 1, dtype=torch.int64, device=r.device)
    rp[1:] = torch.cumsum(counts, 0)
    g = torch.Generator(device=r.device)
    g.manual_seed(seed ^ 0x9E3779B97F4A7C15 & 0x7FFFFFFFFFFFFFFF)
    vals = 1.0 - torch.rand(c.numel(), generator=g, device=r.device, dtype=torch.float64)
    return M, K, rp.to(torch.int32), c, vals.to(dtype)


def _rmat_draws(scale, n, a, b, c, g, device):
    rows = torch.zeros(n, dtype=torch.int64, device=device)
    cols = torch.zeros(n, dtype=torch.int64, device=device)
    for _ in range(scale):
        u = torch.rand(n, generator=g, device=device)
        right = ((u >= a) & (u < a + b)) | (u >= a + b + c)
        down = u >= a + b
        rows = rows * 2 + down.to(torch.int64)
        cols = cols * 2 + right.to(torch.int64)
    return rows, cols


def rmat(scale: int, nnz: int, a=0.25, b=0.25, c=0.25, d=0.25, seed: int = 0,
         dtype=torch.float32, device="cuda", crop: int | None = None):
    """R-MAT with ~nnz distinct cells (draws in batches until the target is met or
    the reference's 10x draw cap is hit, rmat.hpp:52-76)."""
    # parameter checks and the draw-cap contract of rmat.hpp:22-36, 77-80
    if scale < 0 or scale > 30:
        raise ValueError("rmat: scale must be in [0, 30]")
    if any(q < 0.0 or q > 1.0 for q in (a, b, c, d)):
        raise ValueError("rmat: quadrant probabilities must be in [0, 1]")
    if abs(a + b + c + d - 1.0) > 1e-9:
        raise ValueError("rmat: quadrant probabilities must sum to 1")
    if nnz < 0:
        raise ValueError("rmat: target_nnz must be nonnegative")
    if nnz > (crop or (1 << scale)) ** 2:
        raise ValueError("rmat: target_nnz exceeds 2^(2*scale) cells")
    dim = 1 << scale
    M = K = crop or dim
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    keys = torch.empty(0, dtype=torch.int64, device=device)
    drawn = 0
    while keys.numel() < nnz and drawn < 10 * nnz:
        need = int((nnz - keys.numel()) * 1.15) + 1024
        r, cc = _rmat_draws(scale, need, a, b, c, g, device)
        if crop:
            keep = (r < crop) & (cc < crop)
            r, cc = r[keep], cc[keep]
        drawn += need
        keys = torch.unique(torch.cat([keys, r * K + cc]))
        del r, cc
    if keys.numel() < 0.99 * nnz:
        raise RuntimeError(f"rmat: draw cap exhausted at {keys.numel()} of {nnz} target nonzeros")
    if keys.numel() > nnz:  # keep a uniformly random subset of exactly nnz cells
        perm = torch.randperm(keys.numel(), generator=g, device=device)[:nnz]
        keys = torch.sort(keys[perm]).values
    rows, cols = keys // K, keys % K
    del keys
    return _to_csr(rows, cols, M, K, seed, dtype)


def uniform(rows: int, cols: int, nnz: int, seed: int = 0, dtype=torch.float32, device="cuda"):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    keys = torch.empty(0, dtype=torch.int64, device=device)
    while keys.numel() < nnz:
        need = int((nnz - keys.numel()) * 1.05) + 1024
        k = torch.randint(0, rows * cols, (need,), generator=g, device=device, dtype=torch.int64)
        keys = torch.unique(torch.cat([keys, k]))
    if keys.numel() > nnz:
        perm = torch.randperm(keys.numel(), generator=g, device=device)[:nnz]
        keys = torch.sort(keys[perm]).values
    return _to_csr(keys // cols, keys % cols, rows, cols, seed, dtype)


def banded(rows: int, half_width: int, seed: int = 0, dtype=torch.float32, device="cuda"):
    r = torch.arange(rows, device=device, dtype=torch.int64).repeat_interleave(2 * half_width + 1)
    off = torch.arange(-half_width, half_width + 1, device=device, dtype=torch.int64).repeat(rows)
    c = r + off
    keep = (c >= 0) & (c < rows)
    return _to_csr(r[keep], c[keep], rows, rows, seed, dtype)


def reddit_like(seed: int = 7, dtype=torch.float32, device="cuda"):
    """c3: M = K = 232,965 power-law graph, ~114.6M nnz (Reddit's size, average degree
    ~492). R-MAT (0.45, 0.22, 0.22, 0.11) at scale 18, cropped: the Graph500 skew would
    ask row 0 for ~825K distinct columns out of 233K, this one for ~85K."""
    return rmat(18, 114_615_892, 0.45, 0.22, 0.22, 0.11, seed=seed, dtype=dtype, device=device,
                crop=232_965)


def dense_operand(rows: int, cols: int, seed: int, dtype=torch.float32, device="cuda"):
    """U[-1, 1] dense operand (types.hpp:185-193 distribution)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return (torch.rand(rows, cols, generator=g, device=device, dtype=torch.float32) * 2 - 1).to(dtype)


def suite(device="cuda", dtype=torch.float32, small: bool = False):
    """c2: uniform / banded / power-law inputs, 10K-1M rows (BASELINE.json configs[1]).
    Yields (name, csr tuple)."""
    scales = (14, 17) if small else (14, 17, 20)
    for s in scales:
        n = 1 << s
        yield f"uniform_s{s}_d16", (lambda n=n, s=s: uniform(n, n, 16 * n, seed=s, dtype=dtype,
                                                             device=device))
        yield f"powerlaw_s{s}_d16", (lambda s=s: rmat(s, 16 * (1 << s), *GRAPH500, seed=s,
                                                      dtype=dtype, device=device))
        yield f"banded_s{s}_b8", (lambda n=n, s=s: banded(n, 8, seed=s, dtype=dtype,
                                                          device=device))


def workload(name: str, device="cuda", dtype=torch.float32, small: bool = False):
    """The BASELINE.json configs as (matrix name, generator, [N...]) lists.

      suite  configs[1]: uniform / banded / power-law, 2^14..2^20 rows, N = 2..128
      c1     configs[0]: uniform 4096 x 4096, ~1% density, N = 32
      c3     configs[2]: Reddit-scale power-law graph (233K nodes, ~114.6M nnz), N = 128
      c4     configs[3]: R-MAT scale 22 (Graph500 skew and a = 0.7), N = 16 and 64
      c5     configs[4]: R-MAT scale 25 (~503M nnz), N = 256
    """
    ns_suite = [2, 4, 8, 16, 32, 64, 128]
    if name == "suite":
        return [(n, mk, ns_suite) for n, mk in suite(device=device, dtype=dtype, small=small)]
    if name == "c1":
        return [("c1_uniform4096_1pct", lambda: uniform(4096, 4096, 167_772, seed=1, dtype=dtype,
                                                        device=device), [32])]
    if name == "c3":
        return [("c3_reddit_like", lambda: reddit_like(dtype=dtype, device=device), [128])]
    if name == "c4":
        s22 = 16 << 22
        return [("c4_rmat_s22_graph500", lambda: rmat(22, s22, *GRAPH500, seed=22, dtype=dtype,
                                                      device=device), [16, 64]),
                ("c4_rmat_s22_a0.7", lambda: rmat(22, s22, 0.7, 0.1, 0.1, 0.1, seed=23, dtype=dtype,
                                                  device=device), [16, 64])]
    if name == "c5":
        return [("c5_rmat_s25", lambda: rmat(25, 15 << 25, *GRAPH500, seed=25, dtype=dtype,
                                             device=device), [256])]
    raise ValueError(f"unknown workload {name}")


def algorithmic_bytes(M: int, nnz: int, N: int, cols_touched: int, elem: int = 4,
                      off: int = 4) -> int:
    """off*(M+1) + 8*nnz + elem*N*K_touched + elem*N*M (int32 cols,
    fp32 values -> 8 B/nnz)."""
    return off * (M + 1) + (4 + elem) * nnz + elem * N * cols_touched + elem * N * M


def flops(nnz: int, N: int) -> int:
    return 2 * nnz * N


__all__ = ["rmat", "uniform", "banded", "reddit_like", "dense_operand", "suite", "workload",
           "algorithmic_bytes", "flops", "GRAPH500", "math"]
