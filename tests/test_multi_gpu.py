"""Multi-GPU layer on the device, on a 1-GPU box.

* world size 2, both ranks on cuda:0 over gloo: bench.shard_calls -> device DA-SpMM on each
  rank's share (nnz-balanced row panels, or N-split column slices) -> multi.gather_rows /
  gather_cols, checked against the fp64 oracle on sampled rows: the sharding needs no
  exchange besides the optional assembly.
* the C-ABI entry (daspmm_multi_plan / daspmm_multi_spmm): device row cuts, the automatic
  rows-vs-columns choice, one-rank shares, and a one-rank NCCL communicator's assembly.
* the fused SpMM + all-gather over symmetric memory needs one device per rank: run only
  where two GPUs are visible.
"""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, split_mode, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["RANK"], os.environ["WORLD_SIZE"] = str(rank), str(world)
    os.environ["DASPMM_SPLIT_FRAC"] = "0.05"
    os.environ["DASPMM_SPLIT_MODE"] = split_mode
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from oracle import sampled as S
        from paper_2202_08556_b200 import gen, multi
        from paper_2202_08556_b200 import spmmkit as sk

        model = sk.load_selector(open(os.path.join(ROOT, "paper_2202_08556_b200", "models",
                                                   "b200_selector.txt")).read())
        mats = []
        for name, mk in [("powerlaw", lambda: gen.rmat(14, 16 << 14, *gen.GRAPH500, seed=1)),
                         ("uniform", lambda: gen.uniform(1 << 14, 1 << 14, 16 << 14, seed=2))]:
            M, K, rp, ci, va = mk()
            mats.append(dict(name=name, M=M, K=K, nnz_total=int(ci.numel()),
                             full=sk.DeviceCsr.from_device(M, K, rp, ci, va), rp=rp, ci=ci,
                             va=va, ns=[8, 64]))
        mine, units = bench.shard_calls(mats, None, rank, world)
        results = []
        for m, n, d, rows, (c0, c1) in mine:
            B = gen.dense_operand(m["K"], n, seed=1000 + n)
            Bl = B[:, c0:c1].contiguous() if (c1 - c0) != n else B
            Cl = torch.full((d.num_rows, c1 - c0), float("nan"), device="cuda")
            sk.spmm_selected(d, model, Bl, Cl)
            torch.cuda.synchronize()
            results.append((m, n, rows, (c0, c1), B, Cl))
        # every split unit is assembled by all ranks in the same order
        ok = True
        nsplit = 0
        for m, n, rows, (c0, c1), B, Cl in results:
            split_rows = rows != (0, m["M"])
            split_cols = (c1 - c0) != n
            if not (split_rows or split_cols):
                full = Cl
            elif split_rows:
                nsplit += 1
                _, cuts = multi.plan(m["full"], world, n, multi.SPLIT_ROWS)
                assert (int(cuts[rank]), int(cuts[rank + 1])) == rows
                full = multi.gather_rows(Cl, cuts)
            else:
                nsplit += 1
                full = multi.gather_cols(Cl, multi.col_split(n, world))
            rp_h = m["rp"].cpu().numpy().astype(np.int64)
            res = S.check(m["rp"], m["ci"], m["va"], m["K"], B, full,
                          S.sample_rows(rp_h, n_random=256, seed=n))
            ok = ok and res["ok"]
        q.put((rank, ok, nsplit, len(units)))
    except Exception as ex:  # report, do not hang the parent
        q.put((rank, repr(ex), -1, -1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("split_mode", ["rows", "cols"])
def test_two_ranks_shard_compute_gather(split_mode):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, split_mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, nsplit, nunits in res:
        assert ok is True, (rank, ok)
        assert nsplit >= 1 and nunits == 4


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)
    from paper_2202_08556_b200 import gen, multi
    from paper_2202_08556_b200 import spmmkit as sk

    model = sk.load_selector(open(os.path.join(ROOT, "paper_2202_08556_b200", "models",
                                               "b200_selector.txt")).read())
    return torch, gen, multi, sk, model


def test_plan_cuts_and_auto_choice(env):
    torch, gen, multi, sk, model = env
    M, K, rp, ci, va = gen.rmat(16, 16 << 16, *gen.GRAPH500, seed=4)
    d = sk.DeviceCsr.from_device(M, K, rp, ci, va)
    rp_h = rp.cpu().numpy().astype(np.int64)
    nnz = int(rp_h[-1])
    maxrow = int(np.diff(rp_h).max())
    for parts in (1, 2, 3, 8):
        mode, cuts = multi.plan(d, parts, 32, multi.SPLIT_ROWS)
        assert mode == "rows" and cuts[0] == 0 and cuts[-1] == M
        assert (np.diff(cuts) >= 0).all()
        share = np.diff(rp_h[cuts])
        assert (np.abs(share - nnz / parts) <= maxrow + 1).all(), share
        b, e, r = sk.partition_elements(d, parts)  # cut p = chunk p's start row
        for p in range(1, parts):
            assert cuts[p] == max(cuts[p - 1], min(r[p], M))
        mode, bounds = multi.plan(d, parts, 256, multi.SPLIT_COLS)
        assert mode == "cols" and list(bounds) == multi.col_split(256, parts)
    # automatic: per-GPU compulsory bytes, matching multi.choose_partition
    for N in (2, 16, 256, 4096):
        mode, _ = multi.plan(d, 8, N)
        assert mode == multi.choose_partition(M, K, nnz, N, 8), N


@pytest.mark.parametrize("mode", ["rows", "cols"])
def test_multi_spmm_single_rank_and_one_rank_comm(env, mode):
    torch, gen, multi, sk, model = env
    import ctypes as C

    from oracle import sampled as S
    from paper_2202_08556_b200 import _lib

    M, K, rp, ci, va = gen.rmat(15, 16 << 15, *gen.GRAPH500, seed=7)
    d = sk.DeviceCsr.from_device(M, K, rp, ci, va)
    n = 48
    B = gen.dense_operand(K, n, seed=3)
    Cf = torch.full((M, n), float("nan"), device="cuda")
    md = multi.SPLIT_ROWS if mode == "rows" else multi.SPLIT_COLS
    multi.spmm(None, d, model, B, Cf, mode=md)
    torch.cuda.synchronize()
    rows = S.sample_rows(rp.cpu().numpy().astype(np.int64), seed=1)
    assert S.check(rp, ci, va, K, B, Cf, rows)["ok"]
    # a one-rank NCCL communicator: the assembly path runs (no peers to receive from)
    uid = (C.c_char * 128)()
    rc = _lib.lib().daspmm_comm_unique_id(uid)
    if rc == _lib.ERR_NCCL:
        pytest.skip("libnccl.so.2 not loadable")
    _lib.check(rc)
    comm = C.c_void_p()
    _lib.check(_lib.lib().daspmm_comm_create(1, 0, uid, C.byref(comm)))

    class _C:
        _c = comm

    C2 = torch.full((M, n), float("nan"), device="cuda")
    multi.spmm(_C, d, model, B, C2, mode=md, assemble=True)
    torch.cuda.synchronize()
    assert S.check(rp, ci, va, K, B, C2, rows)["ok"]
    _lib.lib().daspmm_comm_destroy(comm)


def test_fused_rows_allgather_two_gpus():
    import torch

    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("the symmetric-memory fused all-gather needs one GPU per rank (>= 2 GPUs)")
    import subprocess

    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
                        os.path.join(ROOT, "tools", "experiments", "p2p_allgather_check.py")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("equals single-GPU C: True") == 2, r.stdout


def test_bench_two_ranks_under_torchrun():
    """The driver's N>1 launch of bench.py (torch.distributed.run, one process per rank)
    on a 1-GPU box: both ranks on cuda:0 over gloo (NCCL refuses two ranks on one GPU).
    Rank 0 prints one JSON line for the whole job; the other exits 0."""
    import json
    import subprocess

    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, DASPMM_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--small", "--no-cpu", "--no-cusparse"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 2
    assert d["e2e"] is not None and d["e2e"]["value"] > 0
    assert d["parity"]["calls_passed"] == d["parity"]["calls_checked"] > 0
