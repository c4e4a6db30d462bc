"""Multi-GPU layer host logic on CPU: world_size-2 gloo process groups.

Each rank takes its nnz-balanced row panel (or its N-split columns), computes its
part with the CPU oracle standing in for the device kernel, and the NCCL/gloo
assembly (multi.gather_rows / gather_cols) must rebuild exactly the single-process
result — i.e. the sharding needs no exchange besides the optional assembly.
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        import helpers as H
        from oracle import oracle as O
        from paper_2202_08556_b200 import multi

        a = H.random_csr(700, 500, 9000, seed=11, skew=1.4)
        x = np.random.default_rng(5).uniform(-1, 1, (500, 12))
        full = O.spmm_reference(H.to_oracle(a), x)
        # row panels, B replicated
        cuts = multi.row_panel_cuts(a.row_offsets, world)
        r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
        rp = a.row_offsets[r0:r1 + 1] - a.row_offsets[r0]
        s, e = a.row_offsets[r0], a.row_offsets[r1]
        panel = O.Csr(r1 - r0, 500, rp, a.col_indices[s:e], a.values[s:e])
        local = torch.from_numpy(O.spmm_reference(panel, x))
        got = multi.gather_rows(local, cuts).numpy()
        ok_rows = bool(np.array_equal(got, full))
        # N-split, A replicated
        bounds = multi.col_split(12, world)
        lc = torch.from_numpy(np.ascontiguousarray(
            O.spmm_reference(H.to_oracle(a), np.ascontiguousarray(x[:, bounds[rank]:bounds[rank + 1]]))))
        got_c = multi.gather_cols(lc, bounds).numpy()
        ok_cols = bool(np.array_equal(got_c, full))
        # balance: every panel's nnz within one max-row of the ideal share
        nnz_p = [int(a.row_offsets[cuts[p + 1]] - a.row_offsets[cuts[p]]) for p in range(world)]
        maxrow = int(np.diff(a.row_offsets).max())
        balanced = all(abs(v - a.row_offsets[-1] / world) <= maxrow for v in nnz_p)
        q.put((rank, ok_rows, ok_cols, balanced))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_panels_and_nsplit_assemble_exactly(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert len(res) == world
    for rank, ok_rows, ok_cols, balanced in res:
        assert ok_rows and ok_cols and balanced, (rank, ok_rows, ok_cols, balanced)


def test_row_panel_cuts_properties():
    from paper_2202_08556_b200 import multi

    rng = np.random.default_rng(1)
    for trial in range(50):
        counts = rng.integers(0, 50, rng.integers(1, 40))
        if trial % 5 == 0:
            counts[rng.integers(0, counts.size)] = 5000  # one huge row
        rp = np.concatenate([[0], np.cumsum(counts)])
        for parts in (1, 2, 3, 8):
            cuts = multi.row_panel_cuts(rp, parts)
            assert cuts[0] == 0 and cuts[-1] == counts.size
            assert (np.diff(cuts) >= 0).all()
            # panel starts are row starts of the rows holding floor(p*nnz/P)
            nnz = rp[-1]
            for p in range(1, parts):
                if nnz:
                    e = min((p * nnz) // parts, nnz - 1)
                    r = multi.row_of_element(rp, e)
                    assert cuts[p] == max(r, cuts[p - 1])


def test_choose_partition_prefers_nsplit_for_wide_b():
    from paper_2202_08556_b200 import multi

    # c5 at P=8: rows 39.2 GB/GPU vs N-split 12.75 GB/GPU
    assert multi.choose_partition(1 << 25, 1 << 25, 503_316_480, 256, 8) == "cols"
    # narrow B, big A: row panels
    assert multi.choose_partition(1 << 22, 1 << 22, 67_108_864, 2, 8) == "rows"


def test_schedule_units_covers_and_balances():
    """Every unit runs exactly once (whole on one rank, or split on all ranks), big units
    are split, and LPT keeps the per-rank load within one small unit of the ideal."""
    from paper_2202_08556_b200 import multi

    rng = np.random.default_rng(3)
    costs = list(rng.uniform(5, 50, 60)) + [900.0, 1200.0, 400.0]
    for parts in (1, 2, 4, 8):
        assign, split = multi.schedule_units(costs, parts)
        seen = {}
        for r, units in enumerate(assign):
            for i in units:
                seen.setdefault(i, []).append(r)
        assert sorted(seen) == list(range(len(costs)))
        for i, ranks in seen.items():
            assert (sorted(ranks) == list(range(parts))) if split[i] else len(ranks) == 1
        loads = [sum(costs[i] / parts if split[i] else costs[i] for i in units)
                 for units in assign]
        ideal = sum(costs) / parts
        assert max(loads) <= ideal + 50.0
        if parts > 1:
            assert split[-2]  # the largest unit always exceeds half a rank's share
        if parts >= 4:
            assert split[-3]
        if parts >= 8:
            assert split[-1]
    assert multi.schedule_units([1.0, 2.0], 1) == ([[0, 1]], [False, False])
