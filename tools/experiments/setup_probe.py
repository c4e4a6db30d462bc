"""Handle-creation cost from host int64 arrays (daspmm_csr_create_host), each suite
matrix ingested three times in a row, with the pieces timed apart: the pageable H2D
copies alone (torch), and the whole create. Tells a one-off (lazy module load, pool
growth) from a steady cost."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2202_08556_b200 import gen  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402

for name, mk, _ in gen.workload("suite"):
    M, K, rp, ci, va = mk()
    a = sk.CsrMatrix(M, K, rp.cpu().numpy().astype(np.int64), ci.cpu().numpy().astype(np.int64),
                     va.cpu().numpy(), np.float32)
    out = []
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = sk.DeviceCsr.from_host(a)
        torch.cuda.synchronize()
        out.append((time.perf_counter() - t0) * 1e3)
        h.close()
    t0 = time.perf_counter()
    x = torch.from_numpy(a.col_indices).cuda()
    torch.cuda.synchronize()
    t_copy = (time.perf_counter() - t0) * 1e3
    print(f"{name:20s} nnz={ci.numel():9d} create_host_ms={[round(v, 2) for v in out]} "
          f"h2d_ci_int64_ms={t_copy:.2f}", flush=True)
    del x, a, rp, ci, va
