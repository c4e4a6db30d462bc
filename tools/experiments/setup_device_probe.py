import time, torch, sys, os
sys.path.insert(0,'/root/repo')
from paper_2202_08556_b200 import gen, spmmkit as sk
for name, mk in [("banded_s20", lambda: gen.banded(1<<20, 8, seed=20)), ("powerlaw_s20", lambda: gen.rmat(20, 16<<20, *gen.GRAPH500, seed=20)), ("uniform_s20", lambda: gen.uniform(1<<20,1<<20,16<<20, seed=20))]:
    M,K,rp,ci,va = mk()
    for rep in range(5):
        torch.cuda.synchronize(); t=time.perf_counter()
        d = sk.DeviceCsr.from_device(M,K,rp,ci,va)
        torch.cuda.synchronize(); print(name, 'from_device ms', round((time.perf_counter()-t)*1e3,3), flush=True)
        d.close()
