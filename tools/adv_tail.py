"""SF_TIMING build: per-instance advance cycles and event counts (C5 bench workload)."""
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
f = g.L.sf_debug_adv_cycles
f.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
NI = 4 * n
out = np.zeros((NI, 8), np.int64)
rows = []
for w in range(100):
    g.step(1)
    torch.cuda.synchronize()
    f(g.h, out.ctypes.data_as(C.POINTER(C.c_int64)))
    if w >= 5: rows.append(out.copy())
a = np.concatenate(rows)
cyc = a[:, 0]
print("cycles p50 %.0f p90 %.0f p99 %.0f max %.0f" % tuple(np.percentile(cyc, [50, 90, 99, 100])))
print("cols: cycles ticks comps arrivals preempts run_n wait_n iters")
for t in np.argsort(-cyc)[:10]: print(a[t].tolist())
for lo, hi in ((0, 0), (1, 10), (11, 40), (41, 100), (101, 10**9)):
    m = (a[:, 3] >= lo) & (a[:, 3] <= hi)
    if m.sum(): print(f"arrivals in [{lo},{hi}] n={m.sum()} median cycles {np.median(cyc[m]):.0f}")
per_win_max = np.stack(rows)[:, :, 0].max(1)
print("per-window max: median", np.median(per_win_max), "mean of medians", np.median(np.stack(rows)[:, :, 0], 1).mean())
