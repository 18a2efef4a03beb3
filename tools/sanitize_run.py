"""Small run for compute-sanitizer (memcheck / synccheck / racecheck) on a B200: C1 (1 scenario,
4 instances) for --windows windows, plus a few C5 scenarios and a redundancy (C5R) scenario, in
the default launch mode (three kernels, PDL).  The run must finish with the oracle's metrics.
  compute-sanitizer --tool memcheck python tools/sanitize_run.py --windows 120
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import OracleSim  # noqa: E402  (checking tool: compares with the oracle)
from paper_2601_12784_b200 import workload as W  # noqa: E402
from paper_2601_12784_b200.staleflow import StaleFlow  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--windows", type=int, default=120)
a = ap.parse_args()
for name, n in (("C1", None), ("C5", 4), ("C5R", 2)):
    p = W.preset(name, n) if n else W.preset(name)
    g = StaleFlow.from_preset(p, command_log_capacity=10_000)
    o = OracleSim.from_preset(p)
    for k in range(len(p.scenarios)):
        pr, tg = W.draw_lengths(p, k, p.pool_groups)
        assert g.submit(k, pr, tg) == 0 and o.submit(k, pr, tg) == 0
        if p.filter_prob > 0:
            f = W.draw_filter_flags(p, k, p.pool_groups)
            g.mark_filtered(k, 0, f)
            assert o.mark_filtered(k, 0, f) == 0
    g.step(a.windows, stats=True)
    assert o.step(a.windows, 4) == 0
    for k in range(len(p.scenarios)):
        assert (o.metrics(k) == g.metrics(k)).all(), (name, k)
    print(name, "ok:", int(g.metrics()[2]), "trajectory-iterations,", int(g.metrics()[9]), "batches")
