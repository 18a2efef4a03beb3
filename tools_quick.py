import time, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2601_12784_b200 import workload as W
from paper_2601_12784_b200.staleflow import StaleFlow
p = W.preset("C5")
g = StaleFlow.from_preset(p)
n = len(p.scenarios)
prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
t=time.time(); assert g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs)) == 0; print("submit", time.time()-t)
g.step(5); torch.cuda.synchronize()
m0 = g.metrics()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record(); g.step(50); e.record(); torch.cuda.synchronize()
m1 = g.metrics()
ms = s.elapsed_time(e)
it = m1[2]-m0[2]
print(f"C5 50 windows: {ms:.2f} ms, traj_iters {it}, {it/ms*1e3/1e9:.2f} G/s, routes {m1[5]-m0[5]} batches {m1[9]}")
