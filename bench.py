#!/usr/bin/env python
"""bench.py -- StaleFlow coordination step (arXiv 2601.12784) on B200.

Metric (BASELINE.json): trajectory-iterations per second (one running trajectory advanced by
one decode step of its instance) and the advance kernel's HBM roofline fraction.

Workload: the C5 configuration -- independent coordination scenarios (4 instances, B = 64,
G = 8, eta 0..3, lognormal lengths sigma 0.25..1.5, full SF strategies) -- 4096 scenarios per
GPU, weak scaling (rank r runs scenarios [r*4096, (r+1)*4096) of the same seeded family).  A
"step" is one sf_step window (W0-W9 of DESIGN.md §3.1) over every scenario on the GPU, i.e.
one pass of all of §8(a)'s rows.  L2 is flushed (512 MiB write) between timed windows.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU, NCCL)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "trajectory-iterations/sec per GPU and HBM GB/s fraction at 1/2/4/8 B200"
UNIT = "trajectory-iterations/s"
ALGO_BYTES_PER_ITER = 8          # read + write of the int32 remaining-length counter
FALLBACK_HBM_GBS = 6650.0        # B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="staleflow", choices=["staleflow", "reference"])
    ap.add_argument("--scenarios", type=int, default=4096, help="scenarios per GPU (C5 family)")
    ap.add_argument("--flush-mb", type=int, default=512)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--profile-run", action="store_true", help="short run for ncu (no e2e / cpu legs)")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)", {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 9 for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def pool_arrays(p, idx, n_groups, group0=0):
    import numpy as np
    from paper_2601_12784_b200 import workload as W
    prs, tgs = [], []
    for k in idx:
        pr, tg = W.draw_lengths(p, k, n_groups, group0)
        prs.append(pr)
        tgs.append(tg)
    return np.concatenate(prs), np.concatenate(tgs)


# ------------------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """The oracle, as it stands, on the host cores: same metric/config, bounded sample."""
    if rank != 0:
        return
    from paper_2601_12784_b200 import workload as W
    full = W.preset("C5", n_scenarios=args.scenarios)
    cpu = oracle_rate(full, list(range(args.scenarios)), args.warmup, args.steps, args.cpu_seconds)
    v = cpu["value"]
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "int32", "data": "synthetic",
           "config": {"workload": f"C5 ({cpu['sample']})", "windows_per_step": 1},
           "cpu_baseline": cpu,
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------ cpu baseline
def oracle_rate(full, idx, warmup, steps, target_s, n_first=64):
    """The oracle (as it stands) on host cores over the SAME window range as the timed GPU
    region (warm-up windows untimed), on a bounded sample of scenarios sized to ~target_s."""
    from oracle.oracle import OracleSim
    from paper_2601_12784_b200 import workload as W
    cores = os.cpu_count() or 1
    n = min(n_first, len(idx))
    while True:
        sample = idx[:n]
        o = OracleSim.from_preset(full, sample)
        for a, k in enumerate(sample):
            pr, tg = W.draw_lengths(full, k, full.pool_groups)
            assert o.submit(a, pr, tg) == 0
        o.step(warmup, cores)
        m0 = o.metrics()
        t0 = time.perf_counter()
        for _ in range(steps):
            o.step(1, cores)
        dt = time.perf_counter() - t0
        it = int(o.metrics()[2] - m0[2])
        if dt >= 0.3 * target_s or n >= len(idx):
            break
        n = min(len(idx), max(n + 1, int(n * target_s / max(dt, 1e-3))))
    return {"value": it / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{n} of {len(idx)} C5 scenarios, windows {warmup}..{warmup + steps - 1} "
                      f"(same range as the timed GPU steps), {dt:.1f} s on {cores} threads"}


def shard(n_per_rank: int, rank: int):
    """Weak scaling: rank r owns scenarios [r*S, (r+1)*S) of one seeded C5 family."""
    return list(range(rank * n_per_rank, (rank + 1) * n_per_rank))


def reduce_metrics(vec, world, dist):
    """All-reduce of the int64 metrics vector: sums, except slot 30 (max time)."""
    import torch
    if world > 1:
        mx = vec[30].clone()
        dist.all_reduce(vec, op=dist.ReduceOp.SUM)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        vec[30] = mx
    return vec


# ------------------------------------------------------------------------------ main arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2601_12784_b200 import workload as W
    from paper_2601_12784_b200.staleflow import StaleFlow

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    S = args.scenarios
    full = W.preset("C5", n_scenarios=S * world)
    idx = shard(S, rank)
    p = W.preset_scenario_slice(full, idx)
    ctx = StaleFlow.from_preset(p, stream=stream)
    pr, tg = pool_arrays(full, idx, full.pool_groups)
    assert ctx.submit_many(np.arange(S), np.full(S, full.pool_groups), pr, tg) == 0
    flush = torch.empty(args.flush_mb << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    ctx.step(args.warmup)
    barrier()
    m0 = ctx.metrics()
    l0 = ctx.kernel_launches
    clocks = ClockSampler(local)
    clocks.start()
    evs = []
    barrier()
    for _ in range(args.steps):
        flush.zero_()                                   # L2 flush, outside the timed events
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        ctx.step(1)
        e.record(stream)
        evs.append((s, e))
    barrier()
    ms = sum(s.elapsed_time(e) for s, e in evs)
    clk = clocks.stop()
    m1 = ctx.metrics()
    launches = ctx.kernel_launches - l0 - 1             # minus the metrics reduction at m1
    local_iters = int(m1[2] - m0[2])

    # per-kernel durations: the timed windows overlap their three kernels (programmatic dependent
    # launch), so CUDA events between the kernels would serialize them.  The simulation is
    # deterministic, so a second context replays exactly the same windows (same inputs, same work)
    # with events recorded around every launch; those give the dominant kernel and its duration.
    rctx = StaleFlow.from_preset(p, stream=stream)
    assert rctx.submit_many(np.arange(S), np.full(S, full.pool_groups), pr, tg) == 0
    rctx.step(args.warmup)
    barrier()
    rctx.profile(True)
    for _ in range(args.steps):
        flush.zero_()
        rctx.step(1)
    barrier()
    rctx.profile(False)
    kern_ms, kern_n = rctx.profile_read()
    replay_ok = bool((rctx.metrics() == m1).all())      # identical simulation (work and results)
    rctx.close()
    dm = torch.tensor((m1 - m0).astype(np.int64), device="cuda")
    tm = torch.tensor([ms], dtype=torch.float64, device="cuda")
    reduce_metrics(dm, world, dist)                     # the metrics all-reduce (NCCL over NVLink)
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    total_iters = int(dm[2].item())
    max_ms = float(tm.item())
    value = total_iters / (max_ms / 1e3)

    # ---------------- roofline of the dominant kernel from the replay's CUDA events
    hbm, peak_src, _ = peaks()
    kid = int(np.argmax(kern_ms))                       # dominant kernel of the step
    kname = ("k_begin_coord", "k_advance", "k_ledger", "k_window")[kid]
    adv_ms_per_launch = kern_ms[kid] / max(1, kern_n[kid])
    bytes_per_launch = ALGO_BYTES_PER_ITER * local_iters / max(1, kern_n[kid])
    achieved = bytes_per_launch / (adv_ms_per_launch / 1e3) / 1e9
    traffic = None                                      # ncu dram bytes per launch of that kernel
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            for k, v in json.load(open(tpath))["dram_bytes_per_launch"].items():
                if kname in k:
                    traffic = v
        except Exception:
            traffic = None
    share = {k: kern_ms[i] / max(1e-9, kern_ms.sum())
             for i, k in enumerate(("coordinate", "advance", "ledger", "fused_window")) if kern_n[i]}

    # ---------------- e2e: the same metric through the C ABI with host buffers
    e2e = None
    if not args.no_e2e and not args.profile_run:
        e2e = run_e2e(args, full, idx, stream, world, barrier)

    # ---------------- supplementary: the same K windows as ONE sf_step call (with programmatic
    # dependent launch a scenario starts its next window as soon as its own previous one is done,
    # so windows pipeline across scenarios; L2 not flushed between windows because there is no
    # host boundary).  Not the headline.
    multi = None
    if not args.profile_run and not args.no_e2e:
        ctx2 = StaleFlow.from_preset(p, stream=stream)
        assert ctx2.submit_many(np.arange(S), np.full(S, full.pool_groups), pr, tg) == 0
        ctx2.step(args.warmup)
        barrier()
        n0 = ctx2.metrics()[2]
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record(stream)
        ctx2.step(args.steps)
        e2.record(stream)
        barrier()
        it2 = torch.tensor([int(ctx2.metrics()[2] - n0)], dtype=torch.int64, device="cuda")
        ms2 = torch.tensor([s2.elapsed_time(e2)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(it2, op=dist.ReduceOp.SUM)
            dist.all_reduce(ms2, op=dist.ReduceOp.MAX)
        multi = {"value": int(it2.item()) / (float(ms2.item()) / 1e3), "unit": UNIT,
                 "windows_per_call": args.steps, "launch": "3 kernels per window with programmatic dependent launch, one sf_step call",
                 "ms_per_window": float(ms2.item()) / args.steps}
        ctx2.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile_run:
        cpu = oracle_rate(full, idx, args.warmup, args.steps, args.cpu_seconds)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": "C5: independent coordination scenarios (I=4, B=64, G=8, eta 0..3, "
                                   "lognormal skew 0.25..1.5, SF R/S/M), 1 step = 1 window over all",
                       "scenarios_per_gpu": S, "global_scenarios": S * world, "windows_per_step": 1,
                       "parallelism": f"scenario-sharded x{world}", "l2": f"flushed ({args.flush_mb} MiB write) "
                                                                          "between timed windows"},
            "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": hbm,
                         "peak_source": peak_src, "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                         "algorithmic_bytes_per_traj_iter": ALGO_BYTES_PER_ITER,
                         "launches": int(kern_n[kid]), "ms_per_launch": adv_ms_per_launch,
                         "step_share": share,
                         "timing": "CUDA events around each launch in a serialized replay of the timed windows "
                                   "(same inputs and work; the timed run overlaps kernels via PDL)",
                         "replay_identical": replay_ok},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "multi_window": multi,
            "gpu_launches": int(launches),
            "clocks": clk,
            "sim": {"routes": int(dm[5].item()), "completions": int(dm[4].item()), "batches": int(dm[9].item()),
                    "interrupts": int(dm[6].item()), "pulls": int(dm[7].item()),
                    "invalid_snapshots": int(dm[11].item()), "violations": int(dm[12].item())},
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, full, idx, stream, world, barrier):
    """Per step: H2D of that window's new prompts from pinned host memory through
    sf_submit_prompts_many, sf_step (one window), D2H of the step's metric deltas."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2601_12784_b200 import workload as W
    from paper_2601_12784_b200.staleflow import StaleFlow
    S = len(idx)
    p = W.preset_scenario_slice(full, idx)
    ctx = StaleFlow.from_preset(p, stream=stream)
    B = full.batch_size
    eta_max = max(s.eta for s in p.scenarios)
    first = (eta_max + 1) * B                              # the initial TS fill
    per_step = B // 8                                      # 8 groups/scenario/window keeps the TS fed
    total_windows = args.warmup + args.steps
    pool = full.pool_groups
    ctx_first = pool_arrays(full, idx, first)
    assert ctx.submit_many(np.arange(S), np.full(S, first), *ctx_first) == 0
    submitted = first
    chunks = []
    for w in range(total_windows):
        ng = min(per_step, pool - submitted)
        if ng <= 0:
            chunks.append(None)
            continue
        pr, tg = pool_arrays(full, idx, ng, submitted)
        hp = [torch.from_numpy(np.arange(S, dtype=np.int32)).pin_memory(),
              torch.from_numpy(np.full(S, ng, np.int32)).pin_memory(),
              torch.from_numpy(pr).pin_memory(), torch.from_numpy(tg).pin_memory()]
        chunks.append((ng, hp))
        submitted += ng
    iters = 0
    h2d = d2h = 0
    t_total = 0.0
    for w in range(total_windows):
        timed = w >= args.warmup
        if timed and w == args.warmup:
            barrier()
        t0 = time.perf_counter()
        if chunks[w] is not None:
            ng, hp = chunks[w]
            assert ctx.submit_many_ptr(S, *(x.data_ptr() for x in hp)) == 0
            if timed:
                h2d += sum(x.numel() * 4 for x in hp)
        st = ctx.step(1, stats=True)                       # syncs + D2H of the metric deltas
        t1 = time.perf_counter()
        if timed:
            t_total += t1 - t0
            iters += st["traj_iters"]
            d2h += 2 * 32 * 8
    tt = torch.tensor([t_total], dtype=torch.float64, device="cuda")
    it = torch.tensor([iters], dtype=torch.int64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dist.all_reduce(it, op=dist.ReduceOp.SUM)
    ctx.close()
    return {"value": int(it.item()) / float(tt.item()), "unit": UNIT,
            "h2d_bytes_per_step": h2d // max(1, args.steps), "d2h_bytes_per_step": d2h // max(1, args.steps),
            "note": "per window: pinned H2D of new prompts (sf_submit_prompts_many), sf_step, D2H of metrics; "
                    "host wall clock, max over ranks"}


if __name__ == "__main__":
    main()
