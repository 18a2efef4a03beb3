"""How many C5 scenarios are idle per trainer-period call over a complete run (B200): a scenario is
idle in a call if its metric vector changed only in the window / valid-snapshot / simulated-time
counters (nothing routed, advanced, rewarded, consumed or published).  Measures the share of the
complete run's scenario-windows that do no work -- the ceiling for skipping finished scenarios.

  python tools/dormancy_probe.py [--per-call 15]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_12784_b200 import workload as W  # noqa: E402
from paper_2601_12784_b200.staleflow import StaleFlow  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--per-call", type=int, default=15)
a = ap.parse_args()
p = W.preset("C5")
n = len(p.scenarios)
windows = p.full_run_windows
prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
g = StaleFlow.from_preset(p)
assert g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs)) == 0
IGNORE = {0, 10, 26, 30}            # windows, valid snapshots, simulated time, max time
keep = [k for k in range(32) if k not in IGNORE]
prev = g.all_metrics()
rows = []
for w0 in range(0, windows, a.per_call):
    g.step(min(a.per_call, windows - w0))
    torch.cuda.synchronize()
    m = g.all_metrics()
    idle = ~(m[:, keep] != prev[:, keep]).any(1)
    rows.append((w0, int(idle.sum()), int((m[:, 2] - prev[:, 2]).sum())))
    prev = m
tot = len(rows) * n
print(f"C5, {n} scenarios, {windows} windows in calls of {a.per_call}: idle scenario-calls "
      f"{sum(r[1] for r in rows)} of {tot} ({sum(r[1] for r in rows) / tot:.3f})")
for w0, idle, it in rows[:: max(1, len(rows) // 28)]:
    print(f"  windows {w0:5d}+: idle scenarios {idle:5d}  traj-iters {it}")
