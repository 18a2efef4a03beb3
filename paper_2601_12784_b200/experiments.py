"""Simulated experiments of the paper, run on the B200 library.

* ablation    -- fig:ablation: the 2^3 combinations of StaleFlow vs vanilla routing (R),
                 synchronization (S) and migration (M) strategies; throughput = tokens / time to
                 finish K training steps, mean over seeds, relative to all-vanilla.
* staleness   -- fig:buffer: staleness V_buf - V_traj of every consumed group, per
                 buffer (no value may exceed eta).
* timeline    -- fig:case: per-instance load (running + waiting) over time.

Every scenario is an independent simulation (one warp on the GPU), so a whole ablation grid
runs as ONE context.  Usage:
  python -m paper_2601_12784_b200.experiments ablation [--seeds 16 --steps 8]
  python -m paper_2601_12784_b200.experiments staleness [--eta 3]
  python -m paper_2601_12784_b200.experiments timeline [--windows 600]
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import sys
from typing import Dict, List

import numpy as np

from . import workload as W

COMBOS = [(r, s, m) for r in (0, 1) for s in (0, 1) for m in (0, 1)]   # 1 = StaleFlow strategy


def combo_bits(r: int, s: int, m: int) -> int:
    return (W.STRAT_R if r else 0) | (W.STRAT_S if s else 0) | (W.STRAT_M if m else 0)


def combo_name(r: int, s: int, m: int) -> str:
    return "".join(("R" if r else "r", "S" if s else "s", "M" if m else "m"))


def skewed_preset(n_seeds: int, eta: int = 3, instances: int = 4, steps: int = 6, sigma: float = 1.0,
                  kprefill_ps: int = 10_000_000, pull_lat_ps: int = 2 * W.PS_PER_S, train_windows: int = 5) -> W.Preset:
    """A §6.5-shaped workload scaled down (B=128, G=16, 40K, eta=3 on 128 GPUs): long-tailed
    group-correlated lengths, every R/S/M combination for every seed.  kprefill_ps is the
    prefill stall per re-admitted context token (reading A20) -- the KV recomputation an Interrupt
    costs -- and pull_lat_ps the Pull duration q."""
    sc = []
    for seed in range(n_seeds):
        for (r, s, m) in COMBOS:
            sc.append(W.Scenario(eta, instances, combo_bits(r, s, m), 9000 + seed, None))
    # KV-pressured (M = 64K tokens) and trainer faster than rollout (5 windows), so that
    # instance skew builds up (the rollout phase is the step time)
    return W.Preset("ablation", sc, 32, 8, W.LengthDist("uniform", 64, 1024),
                    W.LengthDist("lognormal", median=1024, sigma_g=sigma / np.sqrt(2), sigma_m=sigma / np.sqrt(2),
                                 cap=16_384),
                    65_536, train_windows, steps, kprefill_ps=kprefill_ps, pull_lat_ps=pull_lat_ps)


def scenario_inputs(p: W.Preset, k: int, ng: int):
    """(prompt, target) of scenario k: seeds, not scenario indices, decide the lengths so that all 8
    combos of a seed share inputs."""
    return W.draw_lengths(dataclasses.replace(p, scenarios=[p.scenarios[k]]), 0, ng)


def _draw_all(p: W.Preset, ng: int):
    prs, tgs = zip(*[scenario_inputs(p, k, ng) for k in range(len(p.scenarios))])
    return np.concatenate(prs), np.concatenate(tgs)


def run_to_steps(ctx, n_scen: int, steps: int, max_windows: int):
    """Advance until every scenario consumed `steps` batches; per scenario, the simulated time
    (ps) and tokens at the window where it reached `steps` batches."""
    t_done = np.full(n_scen, -1, np.int64)
    tok_done = np.zeros(n_scen, np.int64)
    for w in range(max_windows):
        ctx.step(1)
        m = ctx.all_metrics()
        hit = (m[:, 9] >= steps) & (t_done < 0)
        t_done[hit] = m[hit, 26]
        tok_done[hit] = m[hit, 3]
        if (t_done >= 0).all():
            break
    return t_done, tok_done


def ablation(n_seeds: int = 16, steps: int = 6, eta: int = 3, instances: int = 4, max_windows: int = 6000,
             sigma: float = 1.0, kprefill_ps: int = 10_000_000, pull_lat_ps: int = 2 * W.PS_PER_S,
             train_windows: int = 5) -> Dict:
    from .staleflow import StaleFlow
    p = skewed_preset(n_seeds, eta, instances, steps, sigma, kprefill_ps, pull_lat_ps, train_windows)
    n = len(p.scenarios)
    ctx = StaleFlow.from_preset(p)
    pr, tg = _draw_all(p, p.pool_groups)
    assert ctx.submit_many(np.arange(n), np.full(n, p.pool_groups), pr, tg) == 0
    t_done, tok = run_to_steps(ctx, n, steps, max_windows)
    thr = np.where(t_done > 0, tok / np.maximum(t_done, 1) * 1e12, np.nan)      # tokens per simulated s
    per = thr.reshape(n_seeds, len(COMBOS))
    base = per[:, 0]                                                              # rsm = all vanilla
    rows = []
    for c, (r, s, m) in enumerate(COMBOS):
        rel = per[:, c] / base
        rows.append({"combo": combo_name(r, s, m), "tokens_per_s": float(np.nanmean(per[:, c])),
                     "vs_all_vanilla": float(np.nanmean(rel)), "seeds_done": int(np.isfinite(per[:, c]).sum())})
    m = ctx.all_metrics()
    ints = m[:, 6].reshape(n_seeds, len(COMBOS)).mean(0)
    pulls = m[:, 7].reshape(n_seeds, len(COMBOS)).mean(0)
    for c, row in enumerate(rows):
        row["interrupts_per_seed"] = float(ints[c])
        row["pulls_per_seed"] = float(pulls[c])
    return {"workload": {"instances": instances, "eta": eta, "B": p.batch_size, "G": p.group_size,
                         "sigma": sigma, "steps": steps, "seeds": n_seeds, "kprefill_ps": kprefill_ps,
                         "pull_lat_ps": pull_lat_ps, "train_windows": train_windows}, "rows": rows}


def staleness_by_buffer(ctx, scen: int, B: int) -> List[List[int]]:
    """Per consumed buffer (in order): histogram of V_buf - v_g over its B groups."""
    b = ctx.batches(scen).reshape(-1, 1 + 2 * B)
    out = []
    for row in b:
        st = row[0] - row[2::2]
        out.append(np.bincount(st, minlength=int(st.max()) + 1).tolist())
    return out


def staleness(eta: int = 3, n_scen: int = 64, windows: int = 600) -> Dict:
    from .staleflow import StaleFlow
    p = W.preset("C5", n_scenarios=16 * ((n_scen + 15) // 16))
    idx = [k for k in range(len(p.scenarios)) if p.scenarios[k].eta == eta][:n_scen]
    q = W.preset_scenario_slice(p, idx)
    ctx = StaleFlow.from_preset(q)
    prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in idx])
    assert ctx.submit_many(np.arange(len(idx)), np.full(len(idx), p.pool_groups), np.concatenate(prs),
                           np.concatenate(tgs)) == 0
    ctx.step(windows)
    per_buffer = {}
    for a in range(len(idx)):
        for bi, h in enumerate(staleness_by_buffer(ctx, a, p.batch_size)):
            acc = per_buffer.setdefault(bi, [0] * (eta + 2))
            for s, c in enumerate(h):
                acc[min(s, eta + 1)] += c
    return {"eta": eta, "scenarios": len(idx), "per_buffer": per_buffer,
            "max_staleness": max((s for h in per_buffer.values() for s, c in enumerate(h) if c), default=0)}


def timeline(windows: int = 600, preset: str = "C3") -> Dict:
    """Per-instance load (running, waiting) after every window for one scenario."""
    from .staleflow import StaleFlow
    p = W.preset(preset)
    ctx = StaleFlow.from_preset(p)
    pr, tg = W.draw_lengths(p, 0, p.pool_groups)
    assert ctx.submit(0, pr, tg) == 0
    run, wait, ver = [], [], []
    for w in range(windows):
        ctx.step(1)
        inst = ctx.instances(0)
        run.append(inst[:, 2].tolist())
        wait.append(inst[:, 3].tolist())
        ver.append(inst[:, 0].tolist())
    return {"preset": preset, "run": run, "wait": wait, "version": ver}


def _print_ablation(res: Dict):
    print("| combo (upper = StaleFlow) | tokens/s (simulated) | vs all-vanilla | seeds | interrupts | pulls |")
    print("|---|---|---|---|---|---|")
    for r in res["rows"]:
        print(f"| {r['combo']} | {r['tokens_per_s']:.0f} | {r['vs_all_vanilla']:.3f} | {r['seeds_done']} | "
              f"{r['interrupts_per_seed']:.0f} | {r['pulls_per_seed']:.0f} |")


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["ablation", "staleness", "timeline"])
    ap.add_argument("--seeds", type=int, default=16)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--eta", type=int, default=3)
    ap.add_argument("--instances", type=int, default=4)
    ap.add_argument("--sigma", type=float, default=1.0)
    ap.add_argument("--windows", type=int, default=600)
    ap.add_argument("--kprefill", type=int, default=10_000_000, help="ps per re-admitted context token (A20)")
    ap.add_argument("--pull", type=int, default=2 * W.PS_PER_S, help="Pull duration q (ps)")
    ap.add_argument("--train-windows", type=int, default=5)
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    if a.which == "ablation":
        res = ablation(a.seeds, a.steps, a.eta, a.instances, sigma=a.sigma, kprefill_ps=a.kprefill,
                       pull_lat_ps=a.pull, train_windows=a.train_windows)
        _print_ablation(res)
    elif a.which == "staleness":
        res = staleness(a.eta, windows=a.windows)
        print(json.dumps({k: v for k, v in res.items() if k != "per_buffer"}))
        for b, h in sorted(res["per_buffer"].items()):
            print(f"buffer {b}: {h}")
    else:
        res = timeline(a.windows)
        print("windows", len(res["run"]), "final run per instance", res["run"][-1])
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f)


if __name__ == "__main__":
    sys.exit(main())
