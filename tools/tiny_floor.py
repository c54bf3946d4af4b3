import torch, sys, os
sys.path.insert(0, os.getcwd())
from paper_2407_16847_b200 import splat as S
from workloads import CONFIG_BY_NAME
cfg = CONFIG_BY_NAME['tiny']
Q,K,V = ((torch.rand(1,1,256,64,device='cuda')*2-1) for _ in range(3)); O=torch.empty_like(Q)
a = S.Acsr(cfg.pattern)
flush = torch.empty(64*1024*1024, device='cuda'); x = torch.zeros(1, device='cuda')
def t(fn, n=50):
    for _ in range(5): fn()
    torch.cuda.synchronize(); ts=[]
    for i in range(n):
        flush.fill_(float(i)); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1)*1e3)
    ts.sort(); return round(ts[len(ts)//2],2), round(sum(ts)/len(ts),2)
print('empty-ish torch kernel (x.add_)', t(lambda: x.add_(1)))
print('tiny splat fused', t(lambda: S.splat_sparse_mhsa(a,Q,K,V,O,0.125)))
print('no flush: tiny', end=' ')
ts=[]
for i in range(50):
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); S.splat_sparse_mhsa(a,Q,K,V,O,0.125); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1)*1e3)
ts.sort(); print(round(ts[25],2))
