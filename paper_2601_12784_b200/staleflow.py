"""Python binding of include/staleflow.h (argument marshalling only).

Every step of the coordination step runs in the sm_100a kernels of libstaleflow.so.  There is
no CPU fallback: constructing a `StaleFlow` without the library or without a CUDA device
raises.  PyTorch is used only to obtain the CUDA stream (and, in bench.py, for device memory
and torch.distributed).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from . import workload as W

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libstaleflow.so")
METRICS_LEN = 32

SF_OK, SF_NOT_READY = 0, 1
STATUS = {0: "SF_OK", 1: "SF_NOT_READY", -1: "SF_E_INVALID", -2: "SF_E_VERSION", -3: "SF_E_STATE",
          -4: "SF_E_NOMEM", -5: "SF_E_CUDA", -6: "SF_E_RANGE"}

EXPORTS = ["sf_create", "sf_destroy", "sf_submit_prompts", "sf_submit_prompts_many", "sf_step",
           "sf_publish_params", "sf_collect_batch", "sf_read_metrics", "sf_read_metrics_device",
           "sf_read_scenario_metrics", "sf_read_all_scenario_metrics", "sf_dump_lifecycles", "sf_dump_batches", "sf_dump_commands",
           "sf_dump_instances", "sf_kernel_launches", "sf_last_error", "sf_profile", "sf_profile_read",
           "sf_fit_cost_model", "sf_plan_comm", "sf_mark_filtered", "sf_filter_group",
           "sf_ps_lock_sim"]


class SfConfig(C.Structure):
    _fields_ = [
        ("batch_size", C.c_int32), ("n_scenarios", C.c_int32),
        ("scenario_eta", C.POINTER(C.c_int32)), ("scenario_instances", C.POINTER(C.c_int32)),
        ("scenario_strategy", C.POINTER(C.c_uint32)),
        ("k1_ps_per_tok", C.c_int64), ("k2_ps", C.c_int64), ("k3_ps", C.c_int64), ("k4_ps", C.c_int64),
        ("k5_tok", C.c_int32), ("kprefill_ps_per_tok", C.c_int64), ("kv_budget_tok", C.c_int64),
        ("mu", C.c_double), ("phi_throughput", C.c_double), ("phi_wait", C.c_int32),
        ("snap_period_ps", C.c_int64), ("route_lat_ps", C.c_int64), ("pull_lat_ps", C.c_int64),
        ("reward_lat_ps", C.c_int64), ("strategy", C.c_uint32), ("auto_train_windows", C.c_int32),
        ("pool_capacity_groups", C.c_int32), ("command_log_capacity", C.c_int32),
        ("extra_groups", C.c_int32), ("extra_members", C.c_int32), ("watchdog_windows", C.c_int32),
        ("device", C.c_int32), ("cuda_stream", C.c_void_p),
    ]


class SfStepStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("windows", "ticks", "traj_iters", "tokens", "completions", "routes",
                                         "interrupts", "pulls", "preemptions", "batches", "invalid_snapshots",
                                         "violations", "sim_time_ps")]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libstaleflow.so (built by paper_2601_12784_b200/build.py); raises if absent.
    SF_LIB overrides the path (A/B experiments between two builds of this library)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SF_LIB", path)
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run `python -m paper_2601_12784_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(path)
    P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
    pI32, pI64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64)
    sig = {
        "sf_create": (C.c_int, [I32, I32, I32, C.POINTER(SfConfig), C.POINTER(P)]),
        "sf_destroy": (None, [P]),
        "sf_submit_prompts": (C.c_int, [P, I32, I32, pI32, pI32]),
        "sf_submit_prompts_many": (C.c_int, [P, I32, pI32, pI32, pI32, pI32]),
        "sf_step": (C.c_int, [P, I32, C.POINTER(SfStepStats)]),
        "sf_publish_params": (C.c_int, [P, I32, I32]),
        "sf_collect_batch": (C.c_int, [P, I32, I32, pI32, pI32, pI32, pI32]),
        "sf_mark_filtered": (C.c_int, [P, I32, I32, I32, C.POINTER(C.c_uint8)]),
        "sf_filter_group": (C.c_int, [P, I32, I32]),
        "sf_read_metrics": (C.c_int, [P, pI64, I32]),
        "sf_read_metrics_device": (C.c_int, [P, C.c_void_p]),
        "sf_read_scenario_metrics": (C.c_int, [P, I32, pI64, I32]),
        "sf_read_all_scenario_metrics": (C.c_int, [P, pI64, I64]),
        "sf_dump_lifecycles": (C.c_int, [P, I32, pI64, I64, pI64]),
        "sf_dump_batches": (C.c_int, [P, I32, pI32, I64, pI64]),
        "sf_dump_commands": (C.c_int, [P, I32, pI64, I64, pI64]),
        "sf_dump_instances": (C.c_int, [P, I32, pI64, I64, pI64]),
        "sf_kernel_launches": (I64, [P]),
        "sf_last_error": (C.c_char_p, [P]),
        "sf_profile": (C.c_int, [P, I32]),
        "sf_fit_cost_model": (C.c_int, [I32, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]),
        "sf_ps_lock_sim": (C.c_int, [I32, pI32, pI64, pI64, pI32, I32, pI64, pI64, pI32, pI32]),
        "sf_plan_comm": (C.c_int, [I32, C.POINTER(C.c_double), I32, I32, C.POINTER(C.c_uint8),
                                   C.POINTER(C.c_double), C.POINTER(C.c_double), I32, pI32, pI32, pI32,
                                   C.POINTER(C.c_double)]),
        "sf_profile_read": (C.c_int, [P, C.POINTER(C.c_double), pI64, I32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class SfError(RuntimeError):
    pass


class StaleFlow:
    """A context of independent coordination scenarios on one GPU (include/staleflow.h)."""

    def __init__(self, instances: int, eta: int, group_size: int, batch_size: int, n_scenarios: int = 1, *,
                 scenario_eta: Optional[Sequence[int]] = None, scenario_instances: Optional[Sequence[int]] = None,
                 scenario_strategy: Optional[Sequence[int]] = None, k1: int = W.K1_PS, k2: int = W.K2_PS,
                 k3: int = W.K3_PS, k4: int = W.K4_PS, k5: int = 1, kprefill: int = 10_000_000,
                 kv_budget: int = 1 << 20, mu: float = W.MU, phi_throughput: float = W.PHI_TP,
                 phi_wait: int = W.PHI_WAIT, snap_period: int = W.PS_PER_S, route_lat: int = 10_000_000_000,
                 pull_lat: int = 2 * W.PS_PER_S, reward_lat: int = W.PS_PER_S, strategy: int = W.STRAT_SF,
                 auto_train_windows: int = 0, pool_capacity_groups: int = 1024, command_log_capacity: int = 0,
                 extra_groups: int = 0, extra_members: int = 0, watchdog_windows: int = 0,
                 device: Optional[int] = None, stream=None):
        import torch  # device + stream plumbing only
        if not torch.cuda.is_available():
            raise SfError("StaleFlow needs a CUDA device (no CPU fallback)")
        self.L = load_library()
        if device is None:
            device = torch.cuda.current_device()
        self.G, self.B, self.n_scen = group_size, batch_size, n_scenarios
        self.members = group_size + extra_members          # rolled out per group (App C)
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self._keep = []

        def arr(x, dt, ct):
            if x is None:
                return None
            a = np.ascontiguousarray(np.asarray(x, dtype=dt))
            if a.shape != (n_scenarios,):
                raise SfError(f"per-scenario array of shape {a.shape}, expected ({n_scenarios},)")
            self._keep.append(a)
            return _p(a, ct)

        cfg = SfConfig(batch_size=batch_size, n_scenarios=n_scenarios,
                       scenario_eta=arr(scenario_eta, np.int32, C.c_int32),
                       scenario_instances=arr(scenario_instances, np.int32, C.c_int32),
                       scenario_strategy=arr(scenario_strategy, np.uint32, C.c_uint32),
                       k1_ps_per_tok=k1, k2_ps=k2, k3_ps=k3, k4_ps=k4, k5_tok=k5, kprefill_ps_per_tok=kprefill,
                       kv_budget_tok=kv_budget, mu=mu, phi_throughput=phi_throughput, phi_wait=phi_wait,
                       snap_period_ps=snap_period, route_lat_ps=route_lat, pull_lat_ps=pull_lat,
                       reward_lat_ps=reward_lat, strategy=strategy, auto_train_windows=auto_train_windows,
                       pool_capacity_groups=pool_capacity_groups, command_log_capacity=command_log_capacity,
                       extra_groups=extra_groups, extra_members=extra_members, watchdog_windows=watchdog_windows,
                       device=device, cuda_stream=C.c_void_p(stream.cuda_stream))
        self.h = C.c_void_p()
        rc = self.L.sf_create(instances, eta, group_size, C.byref(cfg), C.byref(self.h))
        if rc != 0:
            raise SfError(f"sf_create failed: {STATUS.get(rc, rc)}")

    @classmethod
    def from_preset(cls, p: "W.Preset", scen_idx: Optional[Sequence[int]] = None, **kw):
        scs = p.scenarios if scen_idx is None else [p.scenarios[i] for i in scen_idx]
        return cls(scs[0].instances, scs[0].eta, p.group_size, p.batch_size, len(scs),
                   scenario_eta=[s.eta for s in scs], scenario_instances=[s.instances for s in scs],
                   scenario_strategy=[s.strategy for s in scs], k5=p.k5, kprefill=p.kprefill_ps,
                   kv_budget=p.kv_budget, mu=p.mu, phi_throughput=p.phi_tp, phi_wait=p.phi_wait,
                   snap_period=p.snap_period_ps, route_lat=p.route_lat_ps, pull_lat=p.pull_lat_ps,
                   reward_lat=p.reward_lat_ps, strategy=scs[0].strategy,
                   auto_train_windows=p.auto_train_windows, extra_groups=p.extra_groups,
                   extra_members=p.extra_members,
                   pool_capacity_groups=kw.pop("pool_capacity_groups", p.pool_groups), **kw)

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "h", None):
            self.L.sf_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what):
        if rc < 0:
            raise SfError(f"{what}: {STATUS.get(rc, rc)}: {self.L.sf_last_error(self.h).decode()}")
        return rc

    def _status(self, rc, what):
        """Calls whose documented failures leave the context usable (submit, publish, collect) return
        their sf_status for the caller to test; a poisoning status (SF_E_STATE, SF_E_NOMEM, SF_E_CUDA)
        raises, so a failure that ends the context cannot go unnoticed."""
        if rc in (-3, -4, -5):
            self._check(rc, what)
        return rc

    # ------------------------------------------------------------------ API
    def submit(self, scen: int, prompt, target) -> int:
        """sf_submit_prompts: prompt[n_groups], target[n_groups * members] (members = G + extra)."""
        prompt = np.ascontiguousarray(prompt, dtype=np.int32).reshape(-1)
        target = np.ascontiguousarray(target, dtype=np.int32).reshape(-1)
        if target.size != prompt.size * self.members:
            raise SfError(f"submit: {target.size} targets for {prompt.size} groups of {self.members} members")
        return self._status(self.L.sf_submit_prompts(self.h, scen, len(prompt), _p(prompt, C.c_int32),
                                                     _p(target, C.c_int32)), "sf_submit_prompts")

    def submit_many(self, scen_ids, n_groups, prompts, targets) -> int:
        """sf_submit_prompts_many: scen_ids[n], n_groups[n]; prompts[sum n_groups] and
        targets[sum n_groups * members] concatenated in scenario order."""
        a = np.ascontiguousarray(scen_ids, dtype=np.int32).reshape(-1)
        b = np.ascontiguousarray(n_groups, dtype=np.int32).reshape(-1)
        pr = np.ascontiguousarray(prompts, dtype=np.int32).reshape(-1)
        tg = np.ascontiguousarray(targets, dtype=np.int32).reshape(-1)
        tot = int(b.astype(np.int64).sum())
        if a.size != b.size or (b < 0).any() or pr.size != tot or tg.size != tot * self.members:
            raise SfError(f"submit_many: {a.size} scenario ids, {b.size} counts (sum {tot}), {pr.size} prompts, "
                          f"{tg.size} targets for {self.members} members per group")
        return self._status(self.L.sf_submit_prompts_many(self.h, len(a), _p(a, C.c_int32), _p(b, C.c_int32),
                                                          _p(pr, C.c_int32), _p(tg, C.c_int32)),
                            "sf_submit_prompts_many")

    def submit_many_ptr(self, n, scen_ptr, ng_ptr, prompt_ptr, target_ptr) -> int:
        """Raw host pointers (e.g. pinned torch tensors' data_ptr())."""
        c = C.POINTER(C.c_int32)
        return self.L.sf_submit_prompts_many(self.h, n, C.cast(scen_ptr, c), C.cast(ng_ptr, c),
                                             C.cast(prompt_ptr, c), C.cast(target_ptr, c))

    def step(self, n_windows: int = 1, stats: bool = False):
        if stats:
            st = SfStepStats()
            self._check(self.L.sf_step(self.h, n_windows, C.byref(st)), "sf_step")
            return {f: getattr(st, f) for f, _ in SfStepStats._fields_}
        self._check(self.L.sf_step(self.h, n_windows, None), "sf_step")
        return None

    def publish(self, scen: int, version: int) -> int:
        return self._status(self.L.sf_publish_params(self.h, scen, version), "sf_publish_params")

    def collect(self, scen: int):
        B = self.B
        vb = np.zeros(1, np.int32)
        g = np.zeros(B, np.int32)
        v = np.zeros(B, np.int32)
        n = np.zeros(1, np.int32)
        rc = self.L.sf_collect_batch(self.h, scen, B, _p(vb, C.c_int32), _p(g, C.c_int32), _p(v, C.c_int32),
                                     _p(n, C.c_int32))
        return self._status(rc, "sf_collect_batch"), int(vb[0]), g, v

    def mark_filtered(self, scen: int, first_group: int, flags) -> None:
        """Filtering (P:413 (2)): flags[a] != 0 drops group first_group + a when it completes."""
        f = np.ascontiguousarray(flags, dtype=np.uint8)
        self._check(self.L.sf_mark_filtered(self.h, scen, first_group, len(f), _p(f, C.c_uint8)), "sf_mark_filtered")

    def filter_group(self, scen: int, group: int) -> int:
        """Proactive filtering of a tracked group between windows; returns the sf_status
        (SF_E_INVALID = -1 if the group has no ledger entry)."""
        return self.L.sf_filter_group(self.h, scen, group)

    def metrics(self, scen: Optional[int] = None) -> np.ndarray:
        out = np.zeros(METRICS_LEN, np.int64)
        if scen is None:
            self._check(self.L.sf_read_metrics(self.h, _p(out, C.c_int64), METRICS_LEN), "sf_read_metrics")
        else:
            self._check(self.L.sf_read_scenario_metrics(self.h, scen, _p(out, C.c_int64), METRICS_LEN), "metrics")
        return out

    def all_metrics(self) -> np.ndarray:
        """(n_scenarios, 32) cumulative per-scenario metrics, one transfer."""
        out = np.zeros((self.n_scen, METRICS_LEN), np.int64)
        self._check(self.L.sf_read_all_scenario_metrics(self.h, _p(out, C.c_int64), out.size), "all metrics")
        return out

    def metrics_device(self, out_ptr: int):
        self._check(self.L.sf_read_metrics_device(self.h, C.c_void_p(out_ptr)), "sf_read_metrics_device")

    def _dump(self, fn, scen, width, dtype, ct):
        n = np.zeros(1, np.int64)
        fn(self.h, scen, None, 0, _p(n, C.c_int64))
        cnt = int(n[0])
        out = np.zeros(max(1, cnt * width), dtype)
        self._check(fn(self.h, scen, _p(out, ct), cnt, _p(n, C.c_int64)), "dump")
        return out[: cnt * width].reshape(-1, width) if width > 1 else out[:cnt]

    def lifecycles(self, scen: int) -> np.ndarray:
        return self._dump(self.L.sf_dump_lifecycles, scen, 13, np.int64, C.c_int64)

    def batches(self, scen: int) -> np.ndarray:
        return self._dump(self.L.sf_dump_batches, scen, 1, np.int32, C.c_int32)

    def commands(self, scen: int) -> np.ndarray:
        return self._dump(self.L.sf_dump_commands, scen, 4, np.int64, C.c_int64)

    def instances(self, scen: int) -> np.ndarray:
        return self._dump(self.L.sf_dump_instances, scen, 7, np.int64, C.c_int64)

    def profile(self, enable: bool = True):
        self._check(self.L.sf_profile(self.h, int(enable)), "sf_profile")

    def profile_read(self):
        """(ms[4], launches[4]) per window kernel: coordinate, advance, ledger, -."""
        ms = np.zeros(4, np.float64)
        n = np.zeros(4, np.int64)
        self._check(self.L.sf_profile_read(self.h, _p(ms, C.c_double), _p(n, C.c_int64), 4), "sf_profile_read")
        return ms, n

    @property
    def kernel_launches(self) -> int:
        return int(self.L.sf_kernel_launches(self.h))


# ---------------------------------------------------------------- host-side tools (f4)
def fit_cost_model(kv, n_run, latency):
    """sf_fit_cost_model: (k1, k2, k3, k4) of Eq 7 from profile samples."""
    L = load_library()
    kv = np.ascontiguousarray(kv, np.float64)
    n_run = np.ascontiguousarray(n_run, np.float64)
    latency = np.ascontiguousarray(latency, np.float64)
    out = np.zeros(4, np.float64)
    rc = L.sf_fit_cost_model(len(kv), _p(kv, C.c_double), _p(n_run, C.c_double), _p(latency, C.c_double),
                             _p(out, C.c_double))
    if rc != 0:
        raise SfError(f"sf_fit_cost_model: {STATUS.get(rc, rc)}")
    return out


def plan_comm(slice_bytes, holds, bandwidth, latency, req_slice, req_receiver):
    """sf_plan_comm: (sender per requirement, accumulated estimate per sender)."""
    L = load_library()
    sb = np.ascontiguousarray(slice_bytes, np.float64)
    h = np.ascontiguousarray(holds, np.uint8)
    bw = np.ascontiguousarray(bandwidth, np.float64)
    lt = np.ascontiguousarray(latency, np.float64)
    rs = np.ascontiguousarray(req_slice, np.int32)
    rr = np.ascontiguousarray(req_receiver, np.int32)
    n_senders, n_receivers = bw.shape
    out = np.zeros(max(1, len(rs)), np.int32)
    acc = np.zeros(n_senders, np.float64)
    rc = L.sf_plan_comm(len(sb), _p(sb, C.c_double), n_senders, n_receivers, _p(h, C.c_uint8), _p(bw, C.c_double),
                        _p(lt, C.c_double), len(rs), _p(rs, C.c_int32), _p(rr, C.c_int32), _p(out, C.c_int32),
                        _p(acc, C.c_double))
    if rc != 0:
        raise SfError(f"sf_plan_comm: {STATUS.get(rc, rc)}")
    return out[: len(rs)], acc


def ps_lock_sim(kind, t_issue, duration, push_version, v0: int = 0):
    """Parameter-server Push/Pull under the writer-preferring read-write lock (include/staleflow.h
    sf_ps_lock_sim).  Returns (t_start, t_end, version, status) int arrays."""
    L = load_library()
    k = np.ascontiguousarray(kind, dtype=np.int32)
    n = len(k)
    t = np.ascontiguousarray(t_issue, dtype=np.int64)
    d = np.ascontiguousarray(duration, dtype=np.int64)
    pv = np.ascontiguousarray(push_version, dtype=np.int32)
    ts, te = np.zeros(n, np.int64), np.zeros(n, np.int64)
    ver, st = np.zeros(n, np.int32), np.zeros(n, np.int32)
    rc = L.sf_ps_lock_sim(n, _p(k, C.c_int32), _p(t, C.c_int64), _p(d, C.c_int64), _p(pv, C.c_int32), v0,
                          _p(ts, C.c_int64), _p(te, C.c_int64), _p(ver, C.c_int32), _p(st, C.c_int32))
    if rc != 0:
        raise SfError(f"sf_ps_lock_sim: {STATUS.get(rc, rc)}")
    return ts, te, ver, st
