"""SF_TIMING + SF_TIMING_ROUTE build: cycles per routing sub-step for the slowest scenarios
(0 prefetch, 1 item + candidates, 2 dT + waterfall reduction, 3 state update / Reserve,
4 Route writes + command hash, 5 group batch)."""
import ctypes as C, sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_12784_b200 import workload as W
from paper_2601_12784_b200.staleflow import StaleFlow
p = W.preset("C5")
g = StaleFlow.from_preset(p)
n = len(p.scenarios)
prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs))
f = g.L.sf_debug_coord_cycles
f.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
out = np.zeros((n, 8), np.int64)
rows = []
for w in range(100):
    g.step(1)
    torch.cuda.synchronize()
    f(g.h, out.ctypes.data_as(C.POINTER(C.c_int64)))
    if w >= 5:
        rows.append(out.copy())
a = np.concatenate(rows)
print("cols: total routes [rep path: gather+init, waterfall+bcast, update, divisions, records, hash] (route_steps)")
for t in np.argsort(-a[:, 0])[:10]:
    r = a[t]
    print(r.tolist(), "per route:", (r[2:] / max(r[1], 1)).round(0).tolist())
