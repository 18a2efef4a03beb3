"""Where the cycles go, per scenario-window, on an instrumented build (B200).

Build the variant once (it lands next to the product library and travels with gpurun):
  python -m paper_2601_12784_b200.build --out paper_2601_12784_b200/libstaleflow_timing.so -DSF_TIMING
Then:
  SF_LIB=paper_2601_12784_b200/libstaleflow_timing.so python tools/timing_profile.py [--from 150 --to 300]

Coordinator (clock64 checkpoints per warp, coord.cuh SF_CK): total cycles and phases [pre-sync, sync,
migration, MLQ rebuild, routing, arrival ordering, post]; advance (per instance-window, advance.cuh
SF_TIMING): cycles, ticks, completions, arrivals, preemptions, run/wait sizes, traj-iters.
Windows run one per sf_step call (the kernels of one window are what is being dissected).
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_12784_b200 import workload as W  # noqa: E402
from paper_2601_12784_b200.staleflow import StaleFlow  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--from", dest="w0", type=int, default=150)
ap.add_argument("--to", dest="w1", type=int, default=300)
ap.add_argument("--preset", default="C5")
ap.add_argument("--scenarios", type=int, default=None, help="C5 only (default 4096)")
a = ap.parse_args()
p = W.preset(a.preset, n_scenarios=a.scenarios or 4096) if a.preset == "C5" else W.preset(a.preset)
n = len(p.scenarios)
n_inst = sum(sc.instances for sc in p.scenarios)
prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
g = StaleFlow.from_preset(p)
g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs))
fc, fa = g.L.sf_debug_coord_cycles, g.L.sf_debug_adv_cycles
fc.argtypes = fa.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
co = np.zeros((n, 8), np.int64)
ad = np.zeros((n_inst, 8), np.int64)
g.step(a.w0)
crow, arow = [], []
for w in range(a.w0, a.w1):
    g.step(1)
    torch.cuda.synchronize()
    fc(g.h, co.ctypes.data_as(C.POINTER(C.c_int64)))
    fa(g.h, ad.ctypes.data_as(C.POINTER(C.c_int64)))
    crow.append(np.concatenate([co, np.full((n, 1), w), np.arange(n)[:, None]], 1))
    arow.append(ad.copy())
c = np.concatenate(crow)
tot = c[:, 0]
if os.environ.get("SF_ROUTE_STEPS") == "1":
    # library built with -DSF_TIMING -DSF_TIMING_ROUTE: columns 2..7 are the routing sub-steps
    # (coord.cuh SF_RT): [item prefetch, candidates, decision, route/Reserve, issue+log, group batch]
    r = c[:, 1]
    names = ["prefetch", "candidates", "decision", "route+reserve", "issue+log", "group-batch"]
    for lo, hi in ((1, 64), (65, 10 ** 9)):
        m = (r >= lo) & (r <= hi)
        if m.sum():
            per = c[m, 2:8].sum(0) / r[m].sum()
            print(f"routes in [{lo},{hi}]: {int(r[m].sum())} routes, cycles per route by sub-step:",
                  {k: round(float(v)) for k, v in zip(names, per)}, "total", round(float(per.sum())))
    sys.exit(0)
ph = np.diff(np.concatenate([np.zeros((len(c), 1)), c[:, 2:8]], 1), axis=1)
post = tot - c[:, 7]
print(f"== coordinator, windows {a.w0}..{a.w1 - 1}, {n} scenarios")
print("cycles per scenario-window: p50 %.0f p90 %.0f p99 %.0f p99.9 %.0f max %.0f" % tuple(np.percentile(tot, [50, 90, 99, 99.9, 100])))
allc = ph.sum() + post.sum()
print("share of all cycles [pre-sync, sync, migr, mlq2, route, arrivals, post]:",
      [round(float(x) / allc, 3) for x in list(ph.sum(0)) + [post.sum()]])
print("median per phase:", np.median(ph, 0).round(0).tolist(), "post", float(np.median(post)))
print("per-window max (the window's coordinator critical path): median %.0f p90 %.0f" % tuple(
    np.percentile(np.stack([r[:, 0] for r in crow]).max(1), [50, 90])))
print("12 slowest: total routes ck0..ck5 window scen eta")
for t in np.argsort(-tot)[:12]:
    print(c[t].tolist(), "eta", p.scenarios[int(c[t, 9])].eta, "I", p.scenarios[int(c[t, 9])].instances)
r = c[:, 1]
for lo, hi in ((0, 0), (1, 8), (9, 64), (65, 200), (201, 10 ** 9)):
    m = (r >= lo) & (r <= hi)
    if m.sum():
        print(f"routes in [{lo},{hi}]: {m.mean():.3f} of scenario-windows, {tot[m].sum() / tot.sum():.3f} of cycles, "
              f"median {np.median(tot[m]):.0f} cycles, {np.median(ph[m, 4] / np.maximum(r[m], 1)):.0f} routing cycles/route")
ad = np.concatenate(arow)
if os.environ.get("SF_ADVANCE", "") == "lanes":
    # one-lane-per-instance kernel (advance_lanes.cuh): loop, stage, coordinator wait, tail cycles,
    # warp iterations, arrival-window refills, wait heads read from HBM, arrivals per lane
    print(f"== advance (lanes), {n_inst} instances per window")
    for k, name in enumerate(["loop", "stage", "wait", "tail", "iterations", "refills", "head_hbm", "arrivals"]):
        v = ad[:, k]
        print(f"  {name:10s} p50 {np.percentile(v, 50):9.0f} p90 {np.percentile(v, 90):9.0f} max {v.max():9.0f} mean {v.mean():9.1f}")
    X = np.stack([np.ones(len(ad)), ad[:, 4]], 1).astype(np.float64)
    print("  loop cycles ~ %.0f + %.0f per warp iteration" % tuple(np.linalg.lstsq(X, ad[:, 0].astype(np.float64), rcond=None)[0]))
    sys.exit(0)
cyc = ad[:, 0]
print(f"== advance, {n_inst} instances per window")
print("cycles per instance-window: p50 %.0f p90 %.0f p99 %.0f max %.0f; mean %.0f" % (
    *np.percentile(cyc, [50, 90, 99, 100]), cyc.mean()))
print("means: ticks %.1f comps %.2f arrivals %.2f preempts %.3f run_n %.1f wait_n %.2f iters %.0f" % tuple(ad[:, 1:8].mean(0)))
for col, name in ((2, "comps"), (3, "arrivals")):
    for lo, hi in ((0, 0), (1, 3), (4, 10), (11, 10 ** 9)):
        m = (ad[:, col] >= lo) & (ad[:, col] <= hi)
        if m.sum():
            print(f"  {name} in [{lo},{hi}]: {m.mean():.3f} of instance-windows, median {np.median(cyc[m]):.0f} cycles")
X = np.stack([np.ones(len(ad)), ad[:, 1], ad[:, 2], ad[:, 3]], 1).astype(np.float64)
coef = np.linalg.lstsq(X, cyc.astype(np.float64), rcond=None)[0]
print("least squares cycles ~ %.0f + %.0f/tick + %.0f/completion + %.0f/arrival" % tuple(coef))

if len({sc.instances for sc in p.scenarios}) > 1:
    # mixed family (C4): per instance count, the coordinator's and the advance's cycles per
    # scenario-window (the advance summed over the scenario's instances: the work one block does)
    inst_of = np.repeat(np.arange(n), [sc.instances for sc in p.scenarios])
    nw = len(arow)
    adv_s = np.stack([np.bincount(inst_of, weights=r[:, 0], minlength=n) for r in arow])
    co_s = np.stack([r[:, 0] for r in crow])
    print("== per instance count: scenarios, coordinator p50/max, advance summed over instances p50/max (cycles per window)")
    for I in sorted({sc.instances for sc in p.scenarios}):
        m = np.array([sc.instances == I for sc in p.scenarios])
        print(f"  I={I:4d} n={m.sum():3d} coord {np.median(co_s[:, m]):9.0f} {co_s[:, m].max():9.0f}  "
              f"adv-sum {np.median(adv_s[:, m]):9.0f} {adv_s[:, m].max():9.0f}")
