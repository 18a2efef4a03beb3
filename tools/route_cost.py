"""SF_TIMING build: cycles per routing decision in the real routing pass (C5 bench workload)."""
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
routes, rp, tot = a[:, 1], a[:, 7], a[:, 0]
m = routes >= 100
print("heavy (>=100 routes): n", m.sum(), "cycles/route in pass: median", np.median(rp[m] / routes[m]), "total coord cycles median", np.median(tot[m]))
m2 = (routes >= 5) & (routes < 100)
print("normal (5..99 routes): cycles/route median", np.median(rp[m2] / routes[m2]), "pass share of coord", np.median(rp[m2] / tot[m2]))
m3 = routes == 0
print("no routes: coord cycles median", np.median(tot[m3]), "pass cycles median", np.median(rp[m3]))
per_window_max = np.stack(rows)[:, :, 0].max(1)
print("per-window max coord cycles: median", np.median(per_window_max), "p90", np.percentile(per_window_max, 90))
