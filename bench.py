#!/usr/bin/env python
"""bench.py -- StaleFlow coordination step (arXiv 2601.12784) on B200.

Metric (BASELINE.json): trajectory-iterations per second -- one running trajectory advanced by one
decode step of its instance, counted identically by the oracle and the library --
and the dominant kernel's HBM roofline fraction (algorithmic 8 B per trajectory-iteration,
SURVEY §8(d)).

Workload (default C5, BASELINE.json configs[4]): independent coordination scenarios (I = 4, B = 64,
G = 8, eta 0..3, lognormal skew 0.25..1.5, StaleFlow R/S/M).  One bench STEP is one COMPLETE run of
the workload: every scenario of this GPU's shard from an empty state until every scenario has
consumed its train_steps batches (C5: 1,260 windows = 10 training steps; `full_run_windows`), issued
as sf_step calls of one trainer period (auto_train_windows windows) each.  Every §8(a) row runs in
every window, so the timed region holds the ramp, the steady state (Consume / Publish / Alg 3 pulls
/ Alg 4 migration) and the tail in their natural proportions.  Each step starts from a freshly
created context (sf_create and the pool upload are outside the device-timed region; the e2e leg
times the pool's host-to-device copy).  L2 is flushed (512 MiB write) before every step.

Multi-GPU: scenario s of the family belongs to rank s mod W.  --split weak (default):
the family has 4096 x W scenarios (4096 per GPU); --split strong: one 4096-scenario family (config 5
literally, 512 per GPU at 8 GPUs).  The only collective is the NCCL all-reduce of the int64 metric
vector plus the max-over-ranks of the timed duration.

  python bench.py [--gpus N --steps K --warmup W] [--workload C1..C5] [--split weak|strong] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU, NCCL)
"""
from __future__ import annotations

import argparse
import json
import os
import platform
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
KERNELS = ("k_begin_coord", "k_advance", "k_ledger", "k_window")
NCU_FILE = os.path.join(ROOT, "profiles", "r02", "ncu_kernels.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="staleflow", choices=["staleflow", "reference"])
    ap.add_argument("--workload", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--split", default="weak", choices=["weak", "strong"])
    ap.add_argument("--scenarios", type=int, default=4096, help="C5 scenarios per GPU (weak) / in the family (strong)")
    ap.add_argument("--windows", type=int, default=0, help="windows per step (default: the preset's full run)")
    ap.add_argument("--flush-mb", type=int, default=512)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the steady-state / replay supplementary legs")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--profile-run", action="store_true", help="short run for ncu (timed steps only)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)", {}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


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


# ------------------------------------------------------------------------------ workload + shard
def family(args, world):
    """(preset of the whole family, this rank's scenario indices, scaling mode)."""
    from paper_2601_12784_b200 import workload as W
    if args.workload == "C5":
        n = args.scenarios * world if args.split == "weak" else args.scenarios
        full = W.preset("C5", n_scenarios=n)
        return full, "weak" if args.split == "weak" else "strong"
    full = W.preset(args.workload)
    if len(full.scenarios) == 1:
        return full, "replicas"                        # a single scenario does not shard (§8(e))
    return full, "strong"


def shard(full, rank, world, mode):
    if mode == "replicas":
        return list(range(len(full.scenarios)))
    return [s for s in range(len(full.scenarios)) if s % world == rank]    # s mod W


def pool_arrays(full, idx):
    import numpy as np
    from paper_2601_12784_b200 import workload as W
    prs, tgs = zip(*[W.draw_lengths(full, k, full.pool_groups) for k in idx])
    return np.concatenate(prs), np.concatenate(tgs)


def workload_name(full, idx, mode, world):
    return (f"{full.name} complete run: {len(idx)} scenarios on this GPU ({len(full.scenarios)} in the family, "
            f"{mode}), {full.full_run_windows} windows = {full.train_steps} train steps each, "
            f"sf_step calls of {full.auto_train_windows} windows")


# ------------------------------------------------------------------------------ oracle timing
def oracle_run(full, idx, windows, threads):
    """The oracle, as it stands, over `windows` windows of scenarios idx: (traj_iters, seconds)."""
    from oracle.oracle import OracleSim
    from paper_2601_12784_b200 import workload as W
    o = OracleSim.from_preset(full, idx)
    for a, k in enumerate(idx):
        pr, tg = W.draw_lengths(full, k, full.pool_groups)
        assert o.submit(a, pr, tg) == 0
    t0 = time.perf_counter()
    assert o.step(windows, threads) == 0
    dt = time.perf_counter() - t0
    return int(o.metrics()[2]), dt


def oracle_sample(full, idx, target_s):
    """A bounded sample of the workload sized to ~target_s of host time: the first n scenarios of the
    shard over the full run (multi-scenario configs, all host threads), or one scenario over the
    first w windows (single-scenario configs, one thread: the oracle is sequential per scenario)."""
    cores = os.cpu_count() or 1
    W_full = full.full_run_windows
    if len(idx) == 1:
        w = min(W_full, 200)
        while True:
            it, dt = oracle_run(full, idx, w, 1)
            if dt >= 0.3 * target_s or w >= W_full:
                return {"n": 1, "windows": w, "threads": 1, "iters": it, "s": dt}
            w = min(W_full, max(w + 1, int(w * target_s / max(dt, 1e-3))))
    n = min(len(idx), max(1, cores))
    while True:
        it, dt = oracle_run(full, idx[:n], W_full, cores)
        if dt >= 0.3 * target_s or n >= len(idx):
            return {"n": n, "windows": W_full, "threads": cores, "iters": it, "s": dt}
        n = min(len(idx), max(n + 1, int(n * target_s / max(dt, 1e-3))))


def cpu_baseline_of(full, idx, smp, kind="oracle"):
    return {"value": smp["iters"] / smp["s"], "unit": UNIT, "cores": smp["threads"], "kind": kind,
            "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
            "sample": f"{smp['n']} of {len(idx)} {full.name} scenarios x windows 0..{smp['windows'] - 1} "
                      f"(the complete run is {full.full_run_windows}), {smp['s']:.1f} s on {smp['threads']} threads"}


def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands on the host cores, same workload / metric; each step
    a bounded sample of the workload (rank 0 only under torchrun)."""
    if rank != 0:
        return
    full, mode = family(args, world)
    idx = shard(full, 0, world, mode)
    per_step = max(1.0, args.cpu_seconds / max(1, args.steps + args.warmup))
    smp = oracle_sample(full, idx, per_step)
    sub = idx[:smp["n"]]
    for _ in range(args.warmup):
        oracle_run(full, sub, smp["windows"], smp["threads"])
    its, secs = 0, 0.0
    for _ in range(args.steps):
        it, dt = oracle_run(full, sub, smp["windows"], smp["threads"])
        its += it
        secs += dt
    v = its / secs
    smp_t = dict(smp, iters=its, s=secs)
    cpu = cpu_baseline_of(full, idx, smp_t)
    cpu["sample"] += f" per step, {args.steps} steps"
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": secs * 1e3 / args.steps, "higher_is_better": True,
           "scaling": "weak" if mode != "strong" else "strong", "vs_baseline": None, "dtype": "int32",
           "data": "synthetic", "config": {"workload": workload_name(full, idx, mode, world) + " (oracle sample)",
                                            "windows_per_step": smp["windows"]},
           "cpu_baseline": cpu,
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------ GPU arm
def reduce_metrics(vec, world, dist):
    """All-reduce of the int64 metrics vector: sums, except slot 30 (max time)."""
    if world > 1:
        mx = vec[30].clone()
        dist.all_reduce(vec, op=dist.ReduceOp.SUM)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        vec[30] = mx
    return vec


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
    full, mode = family(args, world)
    idx = shard(full, rank, world, mode)
    S = len(idx)
    p = W.preset_scenario_slice(full, idx)
    windows = args.windows or full.full_run_windows
    per_call = full.auto_train_windows
    pr, tg = pool_arrays(full, idx)
    hp = [torch.from_numpy(np.arange(S, dtype=np.int32)).pin_memory(),
          torch.from_numpy(np.full(S, full.pool_groups, np.int32)).pin_memory(),
          torch.from_numpy(pr).pin_memory(), torch.from_numpy(tg).pin_memory()]
    h2d_bytes = sum(x.numel() * x.element_size() for x in hp)
    flush = torch.empty(args.flush_mb << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def fresh(submit=True):
        ctx = StaleFlow.from_preset(p, stream=stream)
        if submit:
            assert ctx.submit_many_ptr(S, *(x.data_ptr() for x in hp)) == 0
        return ctx

    def run_windows(ctx, n):
        for w0 in range(0, n, per_call):
            ctx.step(min(per_call, n - w0))

    # ---------------- warm-up: W complete runs (untimed)
    for _ in range(args.warmup):
        ctx = fresh()
        run_windows(ctx, windows)
        ctx.close()
    barrier()

    # ---------------- timed: K complete runs, device time on the context stream
    clocks = ClockSampler(local)
    clocks.start()
    ms, launches = 0.0, 0
    dm = np.zeros(32, np.int64)
    for _ in range(args.steps):
        ctx = fresh()
        flush.zero_()                                   # L2 flush, outside the timed events
        barrier()
        m0 = ctx.metrics()
        l0 = ctx.kernel_launches
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        run_windows(ctx, windows)
        e.record(stream)
        barrier()
        ms += s.elapsed_time(e)
        launches += ctx.kernel_launches - l0
        m1 = ctx.metrics()
        dm += (m1 - m0).astype(np.int64)
        ctx.close()
    clk = clocks.stop()
    dmt = torch.tensor(dm, device="cuda")
    tm = torch.tensor([ms], dtype=torch.float64, device="cuda")
    reduce_metrics(dmt, world, dist)                    # the metrics all-reduce (NCCL over NVLink)
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    total_iters = int(dmt[2].item())
    max_ms = float(tm.item())
    value = total_iters / (max_ms / 1e3)
    assert int(dmt[12].item()) == 0 and int(dmt[29].item()) == 0, "protocol violation / poisoned scenario"

    # ---------------- roofline of the dominant kernel: one more complete run with CUDA events around
    # every launch (the library records them on the context stream, launches serialized); the
    # simulation is deterministic, so it is the same work as each timed step
    hbm, peak_src, _ = peaks()
    rctx = fresh()
    flush.zero_()
    barrier()
    rctx.profile(True)
    run_windows(rctx, windows)
    barrier()
    rctx.profile(False)
    kern_ms, kern_n = rctx.profile_read()
    replay_iters = int(rctx.metrics()[2])
    rctx.close()
    kid = int(np.argmax(kern_ms))
    kname = KERNELS[kid]
    ms_per_launch = kern_ms[kid] / max(1, kern_n[kid])
    bytes_per_launch = ALGO_BYTES_PER_ITER * replay_iters / max(1, kern_n[kid])
    achieved = bytes_per_launch / (ms_per_launch / 1e3) / 1e9
    ncu = {}
    if os.path.exists(NCU_FILE):
        try:
            ncu = json.load(open(NCU_FILE))
        except Exception:
            ncu = {}
    kn = ncu.get("kernels", {})
    traffic = kn.get(kname, {}).get("dram_bytes_per_launch")
    share = {KERNELS[i]: float(kern_ms[i] / max(1e-9, kern_ms.sum())) for i in range(4) if kern_n[i]}
    issue = {k: {"issue_active_frac": v.get("issue_active_frac"), "warps_per_sched": v.get("eligible_warps_per_sched"),
                 "achieved_occupancy": v.get("achieved_occupancy")} for k, v in kn.items() if k in share} or None

    # ---------------- e2e: the same complete runs through the C ABI with host buffers: per step the
    # pool's H2D from pinned memory (sf_submit_prompts_many), every window, the metrics' D2H
    e2e = None
    if not args.no_e2e and not args.profile_run:
        its, secs = 0, 0.0
        for k in range(max(1, args.steps)):
            ctx = fresh(submit=False)
            barrier()
            t0 = time.perf_counter()
            assert ctx.submit_many_ptr(S, *(x.data_ptr() for x in hp)) == 0
            run_windows(ctx, windows)
            m = ctx.metrics()                            # syncs the stream; D2H of the result
            secs += time.perf_counter() - t0
            its += int(m[2])
            ctx.close()
        it_t = torch.tensor([its], dtype=torch.int64, device="cuda")
        se_t = torch.tensor([secs], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(it_t, op=dist.ReduceOp.SUM)
            dist.all_reduce(se_t, op=dist.ReduceOp.MAX)
        e2e = {"value": int(it_t.item()) / float(se_t.item()), "unit": UNIT, "h2d_bytes_per_step": h2d_bytes,
               "d2h_bytes_per_step": 32 * 8,
               "note": "per step: pinned H2D of the whole prompt pool (sf_submit_prompts_many), every window "
                       "(sf_step per trainer period), D2H of the metric vector; host wall clock, max over ranks"}

    # ---------------- supplementary: steady state only (windows 150..449), as sf_step calls of one
    # window with L2 flushed before each (round 1's definition) and of one trainer period
    steady = None
    if not args.no_extra and not args.profile_run and full.name == "C5" and windows >= 450:
        steady = {}
        for label, pc in (("per_window_calls", 1), ("per_trainer_period_calls", per_call)):
            ctx = fresh()
            run_windows(ctx, 150)
            barrier()
            n0 = ctx.metrics()[2]
            t = 0.0
            for w0 in range(150, 450, pc):
                flush.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                ctx.step(pc)
                e.record(stream)
                e.synchronize()
                t += s.elapsed_time(e)
            it = int(ctx.metrics()[2] - n0)
            ctx.close()
            steady[label] = {"value": it / (t / 1e3), "ms_per_window": t / 300}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile_run:
        cpu = cpu_baseline_of(full, idx, oracle_sample(full, idx, args.cpu_seconds))

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if mode == "strong" else "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": workload_name(full, idx, mode, world), "windows_per_step": windows,
                       "windows_per_call": per_call, "scenarios_per_gpu": S, "global_scenarios": len(full.scenarios),
                       "split": mode, "parallelism": f"scenario-sharded x{world} (s mod W)" if mode != "replicas"
                       else f"replicas x{world}",
                       "l2": f"flushed ({args.flush_mb} MiB write) before every step"},
            "per_gpu": value / world,
            "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": hbm, "peak_source": peak_src,
                         "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                         "algorithmic_bytes_per_traj_iter": ALGO_BYTES_PER_ITER,
                         "launches": int(kern_n[kid]), "ms_per_launch": ms_per_launch, "step_share": share,
                         "timing": ("CUDA events around every launch in a serialized replay of one step "
                                    "(same inputs and work; the timed steps overlap kernels via PDL)") if kname != "k_window"
                                   else ("CUDA events around every window-kernel launch (block / cluster mode: one "
                                         "launch per sf_step call runs all its windows) in a replay of one step"),
                         "issue_slots_ncu": issue, "ncu_source": os.path.relpath(NCU_FILE, ROOT) if ncu else None},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "steady_state": steady,
            "gpu_launches": int(launches),
            "clocks": clk,
            "sim": {"routes": int(dmt[5].item()), "completions": int(dmt[4].item()), "batches": int(dmt[9].item()),
                    "interrupts": int(dmt[6].item()), "pulls": int(dmt[7].item()),
                    "invalid_snapshots": int(dmt[11].item()), "violations": int(dmt[12].item()),
                    "staleness_hist": [int(x) for x in dmt[16:25].tolist()]},
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
