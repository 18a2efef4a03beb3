"""SF_TIMING build: what makes a scenario's coordinator slow (C5 bench workload)."""
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
for w in range(60):
    g.step(1)
    torch.cuda.synchronize()
    f(g.h, out.ctypes.data_as(C.POINTER(C.c_int64)))
    if w >= 5:
        rows.append(out.copy())
a = np.concatenate(rows)          # (windows*n, 8): cycles routes interrupts pulls valid n_v n_vl tent
cyc = a[:, 0]
print("cycles p50 %.0f p90 %.0f p99 %.0f max %.0f" % tuple(np.percentile(cyc, [50, 90, 99, 100])))
top = np.argsort(-cyc)[:15]
print("slowest: cycles routes interrupts pulls valid n_v n_vl tentative")
for t in top: print(a[t].tolist())
for name, col in (("routes", 1), ("tentative", 7), ("n_v", 5), ("n_vl", 6)):
    for lo, hi in ((0, 0), (1, 5), (6, 20), (21, 80), (81, 10**9)):
        m = (a[:, col] >= lo) & (a[:, col] <= hi)
        if m.sum(): print(f"{name} in [{lo},{hi}]: n={m.sum()} median cycles {np.median(cyc[m]):.0f} p99 {np.percentile(cyc[m], 99):.0f}")
