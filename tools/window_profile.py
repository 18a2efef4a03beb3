"""Per-window profile of the C5 bench workload over the whole 10-train-step run (B200).

For each window: device ms (CUDA events on the context stream, L2 flushed before the window) and the
window's metric deltas (traj-iters, routes, interrupts, pulls, batches); then the same run replayed
with per-kernel events (launches serialized) for each kernel's ms per window.  Prints per-bucket
summaries and writes the rows as JSON (used for bench.py's timed-range choice).

  python tools/window_profile.py [--windows 1260] [--bucket 60] [--out gpurun_out/window_profile.json]
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


def make(p, prs, tgs):
    n = len(p.scenarios)
    g = StaleFlow.from_preset(p, stream=torch.cuda.current_stream())
    assert g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs)) == 0
    return g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--windows", type=int, default=1260)
    ap.add_argument("--bucket", type=int, default=60)
    ap.add_argument("--out", default="gpurun_out/window_profile.json")
    ap.add_argument("--per-call", type=int, default=15, help="windows per sf_step call in the second run")
    a = ap.parse_args()
    p = W.preset("C5")
    n = len(p.scenarios)
    prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    g = make(p, prs, tgs)
    rows = []
    m_prev = g.metrics()
    for w in range(a.windows):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.step(1)
        e.record()
        torch.cuda.synchronize()
        m = g.metrics()
        d = m - m_prev
        m_prev = m
        rows.append({"w": w, "ms": s.elapsed_time(e), "iters": int(d[2]), "routes": int(d[5]), "ints": int(d[6]),
                     "pulls": int(d[7]), "batches": int(d[9]), "invalid": int(d[11])})
    g.close()
    g = make(p, prs, tgs)
    g.profile(True)
    for w in range(a.windows):
        flush.zero_()
        g.step(1)
        torch.cuda.synchronize()
        ms, _ = g.profile_read()
        rows[w].update({"coord_ms": float(ms[0]), "adv_ms": float(ms[1]), "led_ms": float(ms[2])})
    g.close()
    # the same run in calls of --per-call windows (one sf_step call each, L2 flushed between calls):
    # within a call a scenario starts its next window as soon as its own previous one is done
    g = make(p, prs, tgs)
    calls = []
    m_prev = g.metrics()
    for w0 in range(0, a.windows, a.per_call):
        k = min(a.per_call, a.windows - w0)
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.step(k)
        e.record()
        torch.cuda.synchronize()
        m = g.metrics()
        calls.append({"w0": w0, "windows": k, "ms": s.elapsed_time(e), "iters": int(m[2] - m_prev[2])})
        m_prev = m
    g.close()
    tot_it = sum(r["iters"] for r in calls)
    tot_ms = sum(r["ms"] for r in calls)
    print(f"calls of {a.per_call} windows: full run {tot_it / tot_ms / 1e6:.1f} G traj-iters/s, "
          f"{tot_ms / a.windows:.4f} ms/window")
    per = max(1, a.bucket // a.per_call)
    for c0 in range(0, len(calls), per):
        r = calls[c0:c0 + per]
        it, ms = sum(x["iters"] for x in r), sum(x["ms"] for x in r)
        print(f"  windows {r[0]['w0']:5d}+: {it / ms / 1e6:6.1f} G/s  {ms / sum(x['windows'] for x in r):.4f} ms/window")
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(rows, open(a.out, "w"))
    tot_it = sum(r["iters"] for r in rows)
    tot_ms = sum(r["ms"] for r in rows)
    print(f"full run windows 0..{a.windows - 1}: {tot_it / tot_ms / 1e6:.1f} G traj-iters/s, {tot_ms / a.windows:.4f} ms/window")
    print("bucket  G/s    ms/win  coord  adv    led    routes/w  ints/w  pulls/w  batches/w")
    for b0 in range(0, a.windows, a.bucket):
        r = rows[b0:b0 + a.bucket]
        it, ms = sum(x["iters"] for x in r), sum(x["ms"] for x in r)
        f = lambda k: sum(x[k] for x in r) / len(r)
        print(f"{b0:5d} {it / ms / 1e6:6.1f} {ms / len(r):7.4f} {f('coord_ms'):6.4f} {f('adv_ms'):6.4f} {f('led_ms'):6.4f} "
              f"{f('routes'):9.0f} {f('ints'):7.0f} {f('pulls'):7.1f} {f('batches'):7.1f}")


if __name__ == "__main__":
    main()
