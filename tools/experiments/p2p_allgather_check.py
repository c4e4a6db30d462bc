"""2-rank check of multi.spmm_rows_allgather (fused row-panel SpMM + all-gather through
symmetric memory). On a 1-GPU box both ranks share cuda:0 (gloo process group); on a
multi-GPU box run one rank per GPU. Compares the assembled C with a single-GPU SpMM.

python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
    --master-port 29512 tools/experiments/p2p_allgather_check.py
"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2202_08556_b200 import gen, multi  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
torch.cuda.set_device(local)
backend = os.environ.get("DASPMM_DIST_BACKEND", "nccl" if torch.cuda.device_count() >= world else "gloo")
if backend == "nccl":
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
else:
    dist.init_process_group(backend)
M, K, rp, ci, va = gen.rmat(16, 16 << 16, *gen.GRAPH500, seed=7)
full = sk.DeviceCsr.from_device(M, K, rp, ci, va)
cuts = multi.row_panel_cuts(rp.cpu().numpy(), world)
r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
panel = full.panel(r0, r1)
B = gen.dense_operand(K, 64, seed=3)
C = multi.spmm_rows_allgather(panel, B, M, r0)
ref = torch.empty(M, 64, device="cuda")
sk.spmm_device(0, full, B, ref)
torch.cuda.synchronize()
ok = torch.equal(C, ref)
print(f"rank {rank}: backend {backend}, rows [{r0},{r1}), assembled C equals single-GPU C: {ok}",
      flush=True)
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
