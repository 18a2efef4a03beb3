"""Where the e2e window time goes (C5, 4096 scenarios): submit_many_ptr (host validation + H2D +
scatter), step(1) without stats, step(1) with stats (metric reductions + syncs)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_12784_b200 import workload as W
from paper_2601_12784_b200.staleflow import StaleFlow
p = W.preset("C5"); S = len(p.scenarios)
g = StaleFlow.from_preset(p)
first = 4 * p.batch_size
pr, tg = zip(*[W.draw_lengths(p, k, first) for k in range(S)])
assert g.submit_many(np.arange(S), np.full(S, first), np.concatenate(pr), np.concatenate(tg)) == 0
ng = p.batch_size // 8
chunks = []
for w in range(40):
    pr, tg = zip(*[W.draw_lengths(p, k, ng, first + ng * w) for k in range(S)])
    chunks.append([torch.from_numpy(np.arange(S, dtype=np.int32)).pin_memory(), torch.from_numpy(np.full(S, ng, np.int32)).pin_memory(),
                   torch.from_numpy(np.concatenate(pr)).pin_memory(), torch.from_numpy(np.concatenate(tg)).pin_memory()])
g.step(5); torch.cuda.synchronize()
ts, tn, tst = [], [], []
for w in range(30):
    t0 = time.perf_counter(); assert g.submit_many_ptr(S, *(x.data_ptr() for x in chunks[w])) == 0; torch.cuda.synchronize(); t1 = time.perf_counter()
    if w % 2: g.step(1); torch.cuda.synchronize(); t2 = time.perf_counter(); tn.append(t2 - t1)
    else: g.step(1, stats=True); t2 = time.perf_counter(); tst.append(t2 - t1)
    ts.append(t1 - t0)
print("submit %.3f ms, step(1)+sync %.3f ms, step(1, stats) %.3f ms" % (np.median(ts) * 1e3, np.median(tn) * 1e3, np.median(tst) * 1e3))
