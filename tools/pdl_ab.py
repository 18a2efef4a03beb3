"""ms per C5 window (L2 flushed between windows, profiling off) with and without PDL."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_12784_b200 import workload as W
from paper_2601_12784_b200.staleflow import StaleFlow

p = W.preset("C5")
n = len(p.scenarios)
prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
res = {}
for mode in sys.argv[1:] or ["1", "0"]:
    os.environ["SF_PDL"] = mode
    g = StaleFlow.from_preset(p)
    g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs))
    g.step(5)
    torch.cuda.synchronize()
    m0 = g.metrics()
    evs = []
    for _ in range(100):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); g.step(1); e.record(); evs.append((s, e))
    torch.cuda.synchronize()
    ms = sum(s.elapsed_time(e) for s, e in evs)
    m1 = g.metrics()
    res[mode] = (ms / 100, (m1 - m0).copy())
    print(f"SF_PDL={mode}: {ms / 100:.4f} ms/window, {(m1[2] - m0[2]) / ms * 1e3 / 1e9:.1f} G traj-iters/s")
    # multi-window call (PDL pipelines windows across scenarios)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0 = g.metrics()[2]
    s.record(); g.step(100); e.record(); torch.cuda.synchronize()
    print(f"   one call of 100 windows: {s.elapsed_time(e) / 100:.4f} ms/window, "
          f"{(g.metrics()[2] - k0) / s.elapsed_time(e) * 1e3 / 1e9:.1f} G/s")
    g.close()
if len(res) == 2:
    a, b = list(res.values())
    print("metrics identical:", bool((a[1] == b[1]).all()))
