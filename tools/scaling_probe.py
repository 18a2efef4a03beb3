"""Throughput of the C5 family vs the number of scenarios on one GPU (B200): steady-state windows
(pre-advanced untimed), sf_step calls of --per-call windows, L2 flushed between calls.  Flat ms per
window as scenarios grow = latency-bound per-scenario chains; linear = throughput-bound.

  python tools/scaling_probe.py [--counts 64,512,4096,16384] [--start 150] [--windows 300]
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
ap.add_argument("--counts", default="64,256,1024,2048,4096,8192,16384")
ap.add_argument("--start", type=int, default=150)
ap.add_argument("--windows", type=int, default=300)
ap.add_argument("--per-call", type=int, default=15)
a = ap.parse_args()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for n in [int(x) for x in a.counts.split(",")]:
    p = W.preset("C5", n_scenarios=n)
    prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
    g = StaleFlow.from_preset(p, stream=torch.cuda.current_stream())
    assert g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs)) == 0
    g.step(a.start)
    m0 = g.metrics()
    ms = 0.0
    for w0 in range(0, a.windows, a.per_call):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.step(min(a.per_call, a.windows - w0))
        e.record()
        torch.cuda.synchronize()
        ms += s.elapsed_time(e)
    it = int(g.metrics()[2] - m0[2])
    print(f"scenarios {n:6d}: {ms / a.windows:.4f} ms/window  {it / ms / 1e6:7.1f} G traj-iters/s  "
          f"{ms / a.windows / n * 1e6:.2f} ns per scenario-window", flush=True)
    g.close()
