import os, sys, torch
sys.path.insert(0,'/root/repo')
from paper_2202_08556_b200 import gen, spmmkit as sk
model = sk.load_selector(open('/root/repo/paper_2202_08556_b200/models/b200_selector.txt').read())
flush = torch.ones((256 << 20) // 4, device="cuda")
def t(fn, reps=20):
    for _ in range(3): fn()
    tot=0.0
    for _ in range(reps):
        flush.sum(); s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); tot+=s.elapsed_time(e)
    return tot/reps*1e3
M,K,rp,ci,va = gen.banded(1<<14, 8, seed=14)
d = sk.DeviceCsr.from_device(M,K,rp,ci,va)
B = gen.dense_operand(K, 4, seed=1004); C = torch.empty(M,4,device='cuda')
kout = torch.zeros(1, dtype=torch.int32, device='cuda')
sk.spmm_selected(d, model, B, C, kernel_out=kout); torch.cuda.synchronize(); print('decided', int(kout.item()))
print('selected', t(lambda: sk.spmm_selected(d, model, B, C)))
print('k0', t(lambda: sk.spmm_device(0, d, B, C)), sk.plan_info(0, d, B, C))
print('k1', t(lambda: sk.spmm_device(1, d, B, C)))
Bcm=B.t().contiguous()
print('k2', t(lambda: sk.spmm_device(2, d, Bcm, C)), sk.plan_info(2, d, Bcm, C))
print('selected again', t(lambda: sk.spmm_selected(d, model, B, C)))
