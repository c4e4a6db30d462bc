import os, sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2202_08556_b200 import gen, spmmkit as sk
def coo(M, K, rp, ci, va):
    rows = torch.repeat_interleave(torch.arange(M, device="cuda"), (rp[1:] - rp[:-1]).long())
    perm = torch.randperm(rows.numel(), device="cuda")
    return rows[perm], ci.long()[perm], va[perm]
mats = {n: mk for n, mk, ns in gen.workload("suite") if "s20" in n}
for name in ["powerlaw_s20_d16", "uniform_s20_d16", "powerlaw_s20_d16", "uniform_s20_d16"]:
    M, K, rp, ci, va = mats[name]()
    cr, cc, cv = coo(M, K, rp, ci, va)
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        h = sk.DeviceCsr.from_coo_device(M, K, cr, cc, cv)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        h.close()
        print(name, rep, f"{(t1-t0)*1e3:.2f} ms", flush=True)
    # sorted input (no shuffle)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rows = torch.repeat_interleave(torch.arange(M, device="cuda"), (rp[1:] - rp[:-1]).long())
    h = sk.DeviceCsr.from_coo_device(M, K, rows, ci.long(), va)
    torch.cuda.synchronize(); print(name, "sorted input", f"{(time.perf_counter()-t0)*1e3:.2f} ms")
    h.close()
