"""Multi-GPU DA-SpMM on one box: one process per GPU, torch.distributed
for plumbing, NCCL over NVLink only where the output must be assembled.

Rows of C depend only on rows of A and columns of C only on the same columns of B
(spmm.hpp:23-30), so the path shards without any exchange:

  row panels (B replicated)  rank p owns rows [cut[p], cut[p+1]) with cuts at
                             row_of_element(A, floor(p * nnz / P)) (partition.hpp:27-30,
                             45-64, snapped to row starts) — whole rows, ~equal nnz, no
                             cross-GPU atomics; each rank runs the device selector on its
                             own panel's features.
  N-split (A replicated)     rank p owns columns [N*p/P, N*(p+1)/P) of B and C.

A workload of many independent calls (the synthetic suite: 63 (matrix, N) calls) is
sharded by `schedule_units`: calls too large for one rank's share are split into P row
panels (panel p on rank p), the rest are assigned whole, longest first, to the least
loaded rank (LPT). Every unit runs on exactly one rank; there is no collective on the
data path.

C stays sharded by default. `gather_rows` / `gather_cols` assemble it on every rank
with NCCL all-gather when a consumer needs the full matrix (timed separately), and
`spmm_rows_allgather` fuses the assembly into the SpMM itself: C lives in symmetric
memory, and each rank's row-panel kernel stores every finished row into all ranks'
copies over NVLink (daspmm_spmm_rows_to) — no collective after the kernel, one barrier.
"""
from __future__ import annotations

import numpy as np


def row_of_element(row_offsets: np.ndarray, e: int) -> int:
    """partition.hpp:27-30: upper_bound(row_offsets, e) - 1."""
    return int(np.searchsorted(row_offsets, e, side="right")) - 1


def row_panel_cuts(row_offsets, parts: int) -> np.ndarray:
    """nnz-balanced row cuts: cut[p] = first row whose start is >= floor(p*nnz/P)
    snapped down to the start of the row holding that element. Returns parts+1 cuts,
    cut[0] = 0, cut[parts] = M, nondecreasing."""
    rp = np.asarray(row_offsets, dtype=np.int64)
    M = rp.size - 1
    nnz = int(rp[-1])
    cuts = np.zeros(parts + 1, dtype=np.int64)
    cuts[parts] = M
    for p in range(1, parts):
        e = (p * nnz) // parts
        if nnz == 0:
            cuts[p] = (p * M) // parts
            continue
        r = row_of_element(rp, min(e, nnz - 1))
        cuts[p] = max(r, cuts[p - 1])
    return cuts


def estimate_call_us(nnz: int, N: int, launch_us: float = 8.0) -> float:
    """Rough B200 time of one DA-SpMM call for load balancing: a fixed launch cost plus
    2 nnz N flops at ~3.5 TFLOP/s (the suite's measured average rate)."""
    return launch_us + 2.0 * nnz * N / 3.5e6


def schedule_units(costs, parts: int, split_frac: float = 0.5):
    """Assign independent units (costs[i] = estimated time) to `parts` ranks.

    A unit whose cost exceeds split_frac x the ideal per-rank load (sum / parts) is
    split into `parts` row panels, panel p on rank p. The remaining units go whole,
    largest first, to the rank with the least load so far (LPT).
    Returns (assign, split): assign[r] = list of unit indices rank r runs (whole or its
    panel); split[i] = True when unit i is row-split across all ranks."""
    costs = [float(c) for c in costs]
    parts = max(1, int(parts))
    ideal = sum(costs) / parts
    split = [parts > 1 and c > split_frac * ideal for c in costs]
    load = [0.0] * parts
    assign = [[] for _ in range(parts)]
    for i, c in enumerate(costs):
        if split[i]:
            for r in range(parts):
                assign[r].append(i)
                load[r] += c / parts
    for i in sorted((i for i in range(len(costs)) if not split[i]), key=lambda i: -costs[i]):
        r = min(range(parts), key=lambda r: load[r])
        assign[r].append(i)
        load[r] += costs[i]
    for r in range(parts):
        assign[r].sort()
    return assign, split


def col_split(N: int, parts: int):
    return [(N * p) // parts for p in range(parts + 1)]


SPLIT_AUTO, SPLIT_ROWS, SPLIT_COLS = -1, 0, 1


def plan(d, parts: int, N: int, mode: int = SPLIT_AUTO):
    """daspmm_multi_plan on a DeviceCsr: ('rows' | 'cols', bounds[parts + 1]). Rows: nnz-
    balanced cuts at partition_elements' chunk starts (device partition kernel); cols:
    floor(N p / parts); auto: fewer per-GPU compulsory bytes."""
    import ctypes as C

    from . import _lib

    out_mode = C.c_int()
    bounds = np.zeros(parts + 1, dtype=np.int64)
    _lib.check(_lib.lib().daspmm_multi_plan(d._h, parts, N, mode, C.byref(out_mode),
                                            bounds.ctypes.data))
    return ("rows" if out_mode.value == SPLIT_ROWS else "cols"), bounds


class Comm:
    """NCCL communicator of the C ABI (daspmm_comm) for one rank of a torch.distributed
    job: rank 0 makes the unique id, the process group broadcasts it."""

    def __init__(self, group=None):
        import ctypes as C

        import torch.distributed as dist

        from . import _lib

        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        uid = bytearray(128)
        if self.rank == 0:
            buf = (C.c_char * 128)()
            _lib.check(_lib.lib().daspmm_comm_unique_id(buf))
            uid = bytearray(buf.raw)
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        raw = (C.c_char * 128).from_buffer_copy(box[0])
        self._c = C.c_void_p()
        _lib.check(_lib.lib().daspmm_comm_create(self.nranks, self.rank, raw, C.byref(self._c)))

    def close(self):
        from . import _lib

        if self._c:
            _lib.lib().daspmm_comm_destroy(self._c)
            self._c = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def spmm(comm, d, model, B, C_full, mode: int = SPLIT_AUTO, assemble: bool = False,
         kernel_out=None, hw: int = -1, stream=None):
    """daspmm_multi_spmm: this rank's exchange-free share of C = A·B by DA-SpMM into its
    rows / columns of C_full (M x N row-major on every rank); with ``assemble`` the
    shares of all ranks are gathered over NCCL. ``comm`` None = a single rank."""
    from . import _lib
    from . import spmmkit as sk

    sk._check_operands(d, B, C_full, sk.Layout.RowMajor, "multi_spmm")
    kp = kernel_out.data_ptr() if kernel_out is not None else None
    _lib.check(_lib.lib().daspmm_multi_spmm(comm._c if comm is not None else None, d._h, model._m,
                                            hw, B.data_ptr(), sk._ld(B), B.shape[1],
                                            C_full.data_ptr(), sk._ld(C_full), mode,
                                            1 if assemble else 0, kp, sk._stream_ptr(stream)))
    return C_full


def choose_partition(M: int, K: int, nnz: int, N: int, parts: int, elem: int = 4) -> str:
    """Pick 'rows' or 'cols' by per-GPU compulsory bytes:
    rows: A/P + B + C/P ; cols: A + B/P + C/P."""
    a = 4 * (M + 1) + (4 + elem) * nnz
    b = elem * K * N
    c = elem * M * N
    rows = a / parts + b + c / parts
    cols = a + b / parts + c / parts
    return "rows" if rows <= cols else "cols"


def gather_rows(local_c, cuts, group=None):
    """All-gather row panels of C (unequal sizes) into the full M x N matrix on every
    rank: pad to the largest panel, one all-gather (NCCL over NVLink on GPUs, gloo on
    CPU), then trim."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [int(cuts[p + 1] - cuts[p]) for p in range(world)]
    mx = max(sizes)
    n = local_c.shape[1]
    dev = _comm_device(local_c, group)
    pad = torch.zeros(mx, n, dtype=local_c.dtype, device=dev)
    pad[: local_c.shape[0]].copy_(local_c)
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([outs[p][: sizes[p]] for p in range(world)], 0).to(local_c.device)


def gather_cols(local_c, bounds, group=None):
    """All-gather N-split column slices into the full M x N row-major C."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    widths = [int(bounds[p + 1] - bounds[p]) for p in range(world)]
    mx = max(widths)
    M = local_c.shape[0]
    dev = _comm_device(local_c, group)
    pad = torch.zeros(M, mx, dtype=local_c.dtype, device=dev)
    pad[:, : local_c.shape[1]].copy_(local_c)
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([outs[p][:, : widths[p]] for p in range(world)], 1).to(local_c.device)


def _comm_device(t, group=None):
    """Where the collective's buffers live: the tensor's device under NCCL, host memory
    under gloo (the multi-rank logic is exercised with gloo on CPU-only or 1-GPU hosts)."""
    import torch.distributed as dist

    return "cpu" if dist.get_backend(group) == "gloo" else t.device


def spmm_rows_allgather(panel, B, M: int, r0: int, group=None, C_full=None):
    """Row-panel SpMM fused with the all-gather of C (one process per GPU, NVLink).

    `panel` is this rank's DeviceCsr of rows [r0, r0 + panel.num_rows). C (M x N, fp32)
    is allocated in PyTorch symmetric memory (or passed in, allocated that way); the
    rank's RB+RM+SR kernel writes each finished row into every rank's copy through the
    peer mappings, then all ranks meet at the symmetric-memory barrier. Returns the
    assembled C on every rank."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem

    from . import spmmkit as sk

    group = group or dist.group.WORLD
    N = B.shape[1]
    if C_full is None:
        C_full = symm_mem.empty(M, N, dtype=torch.float32, device=B.device)
    hdl = symm_mem.rendezvous(C_full, group)
    world = dist.get_world_size(group)
    rows = panel.num_rows
    dsts = []
    for q in range(world):  # own copy first (it carries the vector-width checks)
        peer = (dist.get_rank(group) + q) % world
        full = hdl.get_buffer(peer, (M, N), torch.float32)
        dsts.append(full[r0:r0 + rows])
    hdl.barrier()  # every copy is allocated before anyone writes into it
    sk.spmm_rows_to(panel, B, dsts)
    hdl.barrier()  # all panels have landed everywhere
    return C_full
