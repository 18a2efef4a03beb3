"""Per-window ms (L2 flushed between windows, PDL on) of the C5 bench windows 5..104, plus the
routes / interrupts / pulls of each window: where the time goes across windows."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_12784_b200 import workload as W
from paper_2601_12784_b200.staleflow import StaleFlow
p = W.preset("C5")
n = len(p.scenarios)
prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
g = StaleFlow.from_preset(p)
g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs))
g.step(5)
rows = []
for w in range(5, 105):
    m0 = g.metrics()
    flush.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.step(1); e.record(); torch.cuda.synchronize()
    m1 = g.metrics()
    d = m1 - m0
    rows.append((w, s.elapsed_time(e), d[5], d[6], d[7], d[2]))
a = np.array(rows)
print("ms per window: mean %.4f median %.4f p90 %.4f max %.4f" % (a[:, 1].mean(), np.median(a[:, 1]), np.percentile(a[:, 1], 90), a[:, 1].max()))
print("share of time in windows above the median: %.2f" % (a[a[:, 1] > np.median(a[:, 1]), 1].sum() / a[:, 1].sum()))
print("window ms routes interrupts pulls traj_iters (slowest 15)")
for r in a[np.argsort(-a[:, 1])][:15]: print(int(r[0]), round(r[1], 4), int(r[2]), int(r[3]), int(r[4]), int(r[5]))
print("fastest 5:")
for r in a[np.argsort(a[:, 1])][:5]: print(int(r[0]), round(r[1], 4), int(r[2]), int(r[3]), int(r[4]), int(r[5]))

# serialized per-kernel times per window (profiling on -> launches serialized)
g2 = StaleFlow.from_preset(p)
g2.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs))
g2.step(5)
g2.profile(True)
prev = np.zeros(4)
per = []
for w in range(5, 105):
    flush.zero_()
    g2.step(1)
    torch.cuda.synchronize()
    ms, cnt = g2.profile_read()                     # events since the previous read
    per.append(ms.copy())
per = np.array(per)
print("serialized kernel ms per window: coord mean %.4f (min %.4f max %.4f) advance mean %.4f (min %.4f max %.4f) ledger mean %.4f" % (
    per[:, 0].mean(), per[:, 0].min(), per[:, 0].max(), per[:, 1].mean(), per[:, 1].min(), per[:, 1].max(), per[:, 2].mean()))
for w in (7, 43, 62, 94, 104):
    print("window", w, "coord %.4f advance %.4f ledger %.4f" % tuple(per[w - 5, :3]))
