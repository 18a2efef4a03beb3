"""Roofline sweep beyond L2: the C5 family replicated to 4096 .. 65536
scenarios on one B200, steady-state windows (150.. after an untimed advance) in sf_step calls of one
trainer period, L2 flushed before each call.  Per size: G traj-iters/s, ms per window, running
slots per window (traj-iters / ticks ...), the per-window working set of the hot arrays, and the
algorithmic-byte roofline fraction (8 B per traj-iter / time / HBM peak).

  python tools/l2_sweep.py [--counts 4096,8192,16384,32768,65536] [--windows 60] [--out gpurun_out/l2_sweep.json]
  python tools/l2_sweep.py --counts 65536 --windows 2 --ncu      (short run under ncu: DRAM bytes per kernel)
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_12784_b200 import workload as W  # noqa: E402
from paper_2601_12784_b200.staleflow import StaleFlow  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--counts", default="4096,8192,16384,32768,65536")
ap.add_argument("--start", type=int, default=150)
ap.add_argument("--windows", type=int, default=60)
ap.add_argument("--ncu", action="store_true")
ap.add_argument("--out", default="gpurun_out/l2_sweep.json")
a = ap.parse_args()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
l2 = torch.cuda.get_device_properties(0).L2_cache_size
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
rows = []
for n in [int(x) for x in a.counts.split(",")]:
    p = W.preset("C5", n_scenarios=n)
    prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
    g = StaleFlow.from_preset(p, stream=torch.cuda.current_stream())
    assert g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs)) == 0
    g.step(a.start)
    torch.cuda.synchronize()
    m0 = g.metrics()
    ms = 0.0
    for w0 in range(0, a.windows, p.auto_train_windows):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.step(min(p.auto_train_windows, a.windows - w0))
        e.record()
        torch.cuda.synchronize()
        ms += s.elapsed_time(e)
    m1 = g.metrics()
    it = int(m1[2] - m0[2])
    ticks = int(m1[1] - m0[1])
    # hot per-window working set: every instance's run list (rem, id, T, p+T) is read at window start
    # and written back at window end, plus instance state; the running slots per window
    running = it / max(1, a.windows)
    ws = running / max(1.0, ticks / max(1, a.windows) / (4 * n)) * 16 * 2      # slots x 16 B x (read+write)
    r = {"scenarios": n, "G_traj_iters_per_s": it / ms / 1e6, "ms_per_window": ms / a.windows,
         "traj_iters_per_window": running, "running_slots": running / max(1.0, ticks / max(1, a.windows) / (4 * n)),
         "hot_bytes_per_window": ws, "l2_bytes": l2, "ws_over_l2": ws / l2,
         "algo_gbs": 8 * it / (ms / 1e3) / 1e9, "frac_of_peak": 8 * it / (ms / 1e3) / 1e9 / peak}
    rows.append(r)
    print(json.dumps(r), flush=True)
    g.close()
    del g
    torch.cuda.empty_cache()
if not a.ncu:
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(rows, open(a.out, "w"), indent=1)
