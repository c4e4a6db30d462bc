"""Would column-band passes (B band L2-resident, C accumulated across passes) beat the
single pass on uniform s20 at N = 16/32/64? Upper-bound probe with the existing kernels:
A split by column band into NB handles (each a full-height CSR over K/NB columns), each
pass run separately into its own C (the real scheme would accumulate; the extra C
traffic is reported as the add's time)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2202_08556_b200 import gen  # noqa: E402
from paper_2202_08556_b200 import spmmkit as sk  # noqa: E402

flush = torch.empty(64 << 20, device="cuda")


def t(fn, reps=7):
    for _ in range(2):
        fn()
    best = 1e9
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) * 1e3)
    return best


M, K, rp, ci, va = gen.uniform(1 << 20, 1 << 20, 16 << 20, seed=20)
full = sk.DeviceCsr.from_device(M, K, rp, ci, va)
rows = torch.repeat_interleave(torch.arange(M, device="cuda"), (rp[1:] - rp[:-1]).long())
for NB in (2, 4):
    bands = []
    for b in range(NB):
        lo, hi = b * K // NB, (b + 1) * K // NB
        keep = (ci >= lo) & (ci < hi)
        r, c, v = rows[keep], ci[keep] - lo, va[keep]
        rpb = torch.zeros(M + 1, dtype=torch.int64, device="cuda")
        rpb[1:] = torch.cumsum(torch.bincount(r, minlength=M), 0)
        bands.append((sk.DeviceCsr.from_device(M, hi - lo, rpb.to(torch.int32), c.to(torch.int32),
                                                v.contiguous()), lo, hi))
    for n in (16, 32, 64):
        B = gen.dense_operand(K, n, seed=n)
        C = torch.empty(M, n, device="cuda")
        Cs = [torch.empty(M, n, device="cuda") for _ in range(NB)]
        t_full = t(lambda: sk.spmm_device(0, full, B, C))
        Bb = [B[lo:hi] for _, lo, hi in bands]

        def passes():
            for i, (d, lo, hi) in enumerate(bands):
                sk.spmm_device(0, d, Bb[i], Cs[i])
        t_pass = t(passes)
        t_add = t(lambda: torch.stack(Cs).sum(0, out=C) if False else C.copy_(Cs[0]).add_(Cs[1]))
        print(f"NB={NB} N={n}: single {t_full:7.1f} us | {NB} band passes {t_pass:7.1f} us "
              f"| + C accumulate (~{t_add:6.1f} us for 2 bands)", flush=True)
