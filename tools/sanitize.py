"""compute-sanitizer driver: every kernel (8 design points x fast/exact, f32/f64) plus
the selector and graph dispatch on small skewed inputs. Run under
compute-sanitizer --tool {memcheck,racecheck,synccheck}."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import helpers as H  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402

model = sk.load_selector(open(os.path.join(os.path.dirname(sk.__file__), "models",
                                           "b200_selector.txt")).read())
for dtype in (np.float32, np.float64):
    a = H.random_csr(700, 600, 9000, seed=4, dtype=dtype, skew=1.4)
    d = sk.DeviceCsr.from_host(a)
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    for n in (1, 2, 3, 4, 8, 16, 33, 64, 128):
        B = torch.rand(600, n, dtype=tdt, device="cuda")
        Bcm = B.t().contiguous()
        C = torch.empty(700, n, dtype=tdt, device="cuda")
        for k in range(8):
            for exact in (False, True):
                for W in (4, 32):
                    sk.spmm_device(k, d, Bcm if k & 2 else B, C, W=W, P=(64 if exact else 0),
                                   exact=exact)
        if dtype == np.float32:
            kout = torch.zeros(1, dtype=torch.int32, device="cuda")
            sk.spmm_selected(d, model, B, C, kernel_out=kout)
            sk.spmm_selected(d, model, B, C, kernel_out=kout)
# opt-in launch variants: lean RB walk, TMA gather4 EB kernel, shared-memory B window
os.environ["DASPMM_LEAN_RB"] = "1"
sk.reload_env()
a = H.random_csr(700, 600, 9000, seed=4, dtype=np.float32, skew=1.4)
d = sk.DeviceCsr.from_host(a)
for n in (8, 16, 33, 128):
    B = torch.rand(600, n, device="cuda")
    C = torch.empty(700, n, device="cuda")
    sk.spmm_device(0, d, B, C)
del os.environ["DASPMM_LEAN_RB"]
sk.reload_env()
a = H.random_csr(700, 600, 9001, seed=5, dtype=np.float32, skew=1.2)
d = sk.DeviceCsr.from_host(a)
os.environ["DASPMM_TMA"] = "1"
sk.reload_env()
for n in (32, 64, 100, 128):
    B = torch.rand(600, n, device="cuda")
    C = torch.empty(700, n, device="cuda")
    sk.spmm_device(4, d, B, C)
del os.environ["DASPMM_TMA"]
sk.reload_env()
rows = np.repeat(np.arange(2000), 9)
cols = rows + np.tile(np.arange(-4, 5), 2000)
keep = (cols >= 0) & (cols < 2000)
rp = np.concatenate([[0], np.cumsum(np.bincount(rows[keep], minlength=2000))]).astype(np.int64)
band = sk.CsrMatrix(2000, 2000, rp, cols[keep].astype(np.int64),
                    np.random.default_rng(1).uniform(-1, 1, keep.sum()).astype(np.float32),
                    np.float32)
d = sk.DeviceCsr.from_host(band)
os.environ["DASPMM_WIN"] = "1"
sk.reload_env()
for n in (2, 8, 32, 128):
    B = torch.rand(2000, n, device="cuda")
    C = torch.empty(2000, n, device="cuda")
    sk.spmm_device(0, d, B, C)
del os.environ["DASPMM_WIN"]
sk.reload_env()
# dense row-panel tile walks (forced at this size): direct (N <= 16) and staged (N >= 32),
# both row mappings, a non-finite B row (CSR replay path), strided B
os.environ["DASPMM_TILE"] = "2"
for rl in ("1", "8"):
    os.environ["DASPMM_TILE_RL"] = rl
    sk.reload_env()
    for n in (1, 2, 4, 8, 16, 33, 64, 128, 200):
        B = torch.rand(2000, n, device="cuda")
        B[777, 0] = float("inf")
        C = torch.empty(2000, n, device="cuda")
        sk.spmm_device(0, d, B, C)
    Bw = torch.rand(2000, 40, device="cuda")[:, :36]
    sk.spmm_device(0, d, Bw, torch.empty(2000, 36, device="cuda"))
del os.environ["DASPMM_TILE"], os.environ["DASPMM_TILE_RL"]
sk.reload_env()
# RB+CM+SR lanes over rows (forced on every shape): column blocks of 1..8, ragged N
os.environ["DASPMM_CM_ROWS"] = "2"
sk.reload_env()
for n in (1, 3, 8, 13, 64):
    Bcm = torch.rand(n, 2000, device="cuda")
    sk.spmm_device(2, d, Bcm, torch.empty(2000, n, device="cuda"))
del os.environ["DASPMM_CM_ROWS"]
sk.reload_env()
# replicated RB+RM+SR epilogue (fused row-panel SpMM + all-gather), three destinations
for n in (3, 32, 128):
    B = torch.rand(2000, n, device="cuda")
    outs = [torch.empty(2000, n, device="cuda") for _ in range(3)]
    sk.spmm_rows_to(d, B, outs)
torch.cuda.synchronize()
print("sanitize driver done")
