"""SF_TIMING build: per-phase cycle checkpoints of the coordinator for the slowest scenarios."""
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
        o = out.copy(); o = np.concatenate([o, np.full((n, 1), w), np.arange(n)[:, None]], 1)
        rows.append(o)
a = np.concatenate(rows)
print("cols: total routes ck0(pre-sync) ck1(sync) ck2(migr) ck3(mlq2) ck4(route) ck5(arrivals) window scen")
for t in np.argsort(-a[:, 0])[:12]: print(a[t].tolist(), "eta", p.scenarios[a[t, 9]].eta)
# typical scenario: median cycles of each phase over all scenario-windows
ph = np.diff(np.concatenate([np.zeros((len(a), 1)), a[:, 2:8]], 1), axis=1)   # ck0, ck1-ck0, ..., ck5-ck4
tot = a[:, 0]
print("median total %.0f; median per phase [pre-sync, sync, migr, mlq2, route, arrivals]:" % np.median(tot),
      np.median(ph, 0).round(0).tolist(), "post (total - ck5):", np.median(tot - a[:, 7]))
# share of the total coordinator cycles (all scenario-windows) spent in each phase
sums = ph.sum(0)
post = (tot - a[:, 7]).sum()
allc = sums.sum() + post
print("share of all cycles [pre-sync, sync, migr, mlq2, route, arrivals, post]:",
      [round(float(x) / allc, 3) for x in list(sums) + [post]])
big = a[:, 1] > 128
print("scenario-windows with > 128 routes: %.3f, their share of cycles %.3f" % (big.mean(), tot[big].sum() / tot.sum()))
