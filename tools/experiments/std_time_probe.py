import time, torch, sys
sys.path.insert(0,'/root/repo')
from paper_2202_08556_b200 import gen, spmmkit as sk
for name, mk in [("uniform_s20", lambda: gen.uniform(1<<20, 1<<20, 16<<20, seed=1)), ("powerlaw_s20", lambda: gen.rmat(20, 16<<20, *gen.GRAPH500, seed=2)), ("rmat_s24", lambda: gen.rmat(24, 16<<24, *gen.GRAPH500, seed=3))]:
    M,K,rp,ci,va = mk()
    for rep in range(2):
        d = sk.DeviceCsr.from_device(M,K,rp,ci,va)
        torch.cuda.synchronize(); t=time.perf_counter(); f=sk.extract_features(d, 8); t=(time.perf_counter()-t)*1e3
        print(name, M, 'extract_features exact ms', round(t,3), f.std_row, flush=True)
        d.close()
    del rp, ci, va; torch.cuda.empty_cache()
