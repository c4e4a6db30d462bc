# Cross-evaluation of selector models trained on two timing collections (train split of each),
# scored on each collection's test split (tools/train_selector.py's split and metric).
import sys, ctypes as C, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tools')
import train_selector as T
from oracle import oracle as O
R=O.ref()
def trained(path):
    ids,f,t=T.load(path); lab=T.split_by_matrix(ids)
    order=np.concatenate([np.where(lab==0)[0],np.where(lab==1)[0]])
    ptr=R.ref_selector_train(len(order),int((lab==0).sum()),np.ascontiguousarray(f[order].reshape(-1)),None,np.ascontiguousarray(t[order].reshape(-1)),100,4,5)
    txt=C.cast(ptr,C.c_char_p).value.decode(); R.ref_free(ptr); return R.ref_selector_load(txt.encode())
def ev(m, path):
    ids,f,t=T.load(path); lab=T.split_by_matrix(ids); test=np.where(lab==2)[0]
    ch=[]
    for i in test:
        k=C.c_int(); R.ref_selector_predict(m,int(f[i,0]),int(f[i,1]),float(f[i,2]),int(f[i,3]),-1,C.byref(k)); ch.append(k.value)
    s=T.normalized(t[test],np.array(ch)); return float(np.exp(np.log(s).mean()))
old = "data/b200_timings_r01.csv"; new = "data/b200_timings_r01g.csv"
mo=trained(old); mn=trained(new)
print('old model: old-test',ev(mo,old),'new-test',ev(mo,new))
print('new model: old-test',ev(mn,old),'new-test',ev(mn,new))
