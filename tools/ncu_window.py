"""Driver for ncu captures of one window kernel in steady state (B200): C5 (4096 scenarios) stepped
one window per sf_step call up to --windows.  Use with ncu's -k / --launch-skip / --launch-count, e.g.
  ncu --set full --import-source on --clock-control none -k regex:k_advance_lanes --launch-skip 160 \
      --launch-count 1 -o gpurun_out/adv -f python tools/ncu_window.py --windows 162
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
ap.add_argument("--windows", type=int, default=162)
ap.add_argument("--scenarios", type=int, default=4096)
a = ap.parse_args()
p = W.preset("C5", n_scenarios=a.scenarios)
n = len(p.scenarios)
prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
g = StaleFlow.from_preset(p)
assert g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs)) == 0
for _ in range(a.windows):
    g.step(1)
torch.cuda.synchronize()
print("windows", a.windows, "traj_iters", int(g.metrics()[2]))
