"""ctypes marshalling for the C++ oracle (TEST INFRASTRUCTURE ONLY).

Argument marshalling only: every step of the simulation runs in sf_oracle.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "sf_oracle.cpp")
HDR = os.path.join(HERE, "sf_oracle.h")
LIB = os.path.join(HERE, "libsforacle.so")

METRICS_LEN = 32
METRIC_NAMES = [
    "windows", "ticks", "traj_iters", "tokens", "completions", "routes", "interrupts", "pulls",
    "preemptions", "batches", "valid_snapshots", "invalid_snapshots", "violations", "publishes",
    "ingested_groups", "occupied_groups",
    "stale_0", "stale_1", "stale_2", "stale_3", "stale_4", "stale_5", "stale_6", "stale_7", "stale_8+",
    "command_hash", "sim_time_ps", "reserves", "relocations", "poisoned_scenarios", "max_sim_time_ps", "aborts",
]

_lock = threading.Lock()
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile the oracle with g++ (no FMA contraction, no fast-math)."""
    with _lock:
        if (not force and os.path.exists(LIB)
                and os.path.getmtime(LIB) >= max(os.path.getmtime(SRC), os.path.getmtime(HDR))):
            return LIB
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               SRC, "-o", tmp, "-lpthread"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, LIB)
        return LIB


class Config(C.Structure):
    _fields_ = [
        ("batch_size", C.c_int32), ("n_scenarios", C.c_int32),
        ("scenario_eta", C.POINTER(C.c_int32)), ("scenario_instances", C.POINTER(C.c_int32)),
        ("scenario_strategy", C.POINTER(C.c_uint32)),
        ("k1", C.c_int64), ("k2", C.c_int64), ("k3", C.c_int64), ("k4", C.c_int64),
        ("k5", C.c_int32), ("kp", C.c_int64), ("M", C.c_int64),
        ("mu", C.c_double), ("phi_tp", C.c_double), ("phi_wait", C.c_int32),
        ("delta", C.c_int64), ("r", C.c_int64), ("q", C.c_int64), ("R", C.c_int64),
        ("strategy", C.c_uint32), ("atw", C.c_int32), ("pool_capacity_groups", C.c_int32),
        ("extra_groups", C.c_int32), ("extra_members", C.c_int32), ("watchdog_windows", C.c_int32),
    ]


class Params(C.Structure):
    _fields_ = [("k1", C.c_int64), ("k2", C.c_int64), ("k3", C.c_int64), ("k4", C.c_int64),
                ("k5", C.c_int32), ("kp", C.c_int64), ("M", C.c_int64),
                ("mu", C.c_double), ("phi_tp", C.c_double), ("phi_wait", C.c_int32), ("eta", C.c_int32)]


class InstView(C.Structure):
    _fields_ = [("v", C.c_int32), ("kv", C.c_int64), ("n_run", C.c_int32), ("n_wait", C.c_int32)]


class TsItem(C.Structure):
    _fields_ = [("id", C.c_int32), ("g", C.c_int32), ("v", C.c_int32), ("l", C.c_int32)]


def load_oracle():
    global _lib
    if _lib is not None:
        return _lib
    override = os.environ.get("SFO_ORACLE_LIB")        # tests/test_oracle_mutants.py: a mutated build
    if override:
        L = C.CDLL(override)
    else:
        build_oracle()
        L = C.CDLL(LIB)
    P, I32, I64, U32, D = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_double
    pI32, pI64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64)
    sig = {
        "sfo_create": (C.c_int, [I32, I32, I32, C.POINTER(Config), C.POINTER(P)]),
        "sfo_destroy": (None, [P]),
        "sfo_submit_prompts": (C.c_int, [P, I32, I32, pI32, pI32]),
        "sfo_step": (C.c_int, [P, I32, I32]),
        "sfo_publish_params": (C.c_int, [P, I32, I32]),
        "sfo_collect_batch": (C.c_int, [P, I32, I32, pI32, pI32, pI32, pI32]),
        "sfo_read_metrics": (C.c_int, [P, pI64, I32]),
        "sfo_read_scenario_metrics": (C.c_int, [P, I32, pI64, I32]),
        "sfo_dump_lifecycles": (C.c_int, [P, I32, pI64, I64, pI64]),
        "sfo_dump_batches": (C.c_int, [P, I32, pI32, I64, pI64]),
        "sfo_dump_commands": (C.c_int, [P, I32, pI64, I64, pI64]),
        "sfo_dump_instances": (C.c_int, [P, I32, pI64, I64, pI64]),
        "sfo_ledger_new": (P, [I32, I32]),
        "sfo_ledger_new2": (P, [I32, I32, I32]),
        "sfo_ledger_consume2": (C.c_int, [P, pI32, pI32, pI32, pI32]),
        "sfo_ledger_free": (None, [P]),
        "sfo_ledger_clone": (P, [P]),
        "sfo_ledger_verify": (C.c_int, [P, I32]),
        "sfo_ledger_reserve": (C.c_int, [P, I32, I32, pI32, pI32]),
        "sfo_ledger_delete_relocate": (C.c_int, [P, I32]),
        "sfo_ledger_abort": (C.c_int, [P, I32, pI32]),
        "sfo_mark_filtered": (C.c_int, [P, I32, I32, I32, C.POINTER(C.c_uint8)]),
        "sfo_filter_group": (C.c_int, [P, I32, I32]),
        "sfo_ledger_occupy": (C.c_int, [P, I32, I32, pI32, pI32]),
        "sfo_ledger_state": (C.c_int, [P, I32]),
        "sfo_ledger_consume": (C.c_int, [P, pI32, pI32]),
        "sfo_ledger_get": (C.c_int, [P, I32, I32, pI32, pI32, pI32]),
        "sfo_ledger_cu": (I32, [P]),
        "sfo_tick_latency": (I64, [C.POINTER(Params), I64, I32, I64]),
        "sfo_throughput": (D, [C.POINTER(Params), I32, I64]),
        "sfo_marginal_gain": (D, [C.POINTER(Params), C.POINTER(InstView), I32]),
        "sfo_ideal_gain": (D, [C.POINTER(Params), I32]),
        "sfo_check_routable": (C.c_int, [C.POINTER(Params), C.POINTER(InstView), I32, P]),
        "sfo_mlq_order": (C.c_int, [C.POINTER(TsItem), I32, pI32]),
        "sfo_route": (C.c_int, [C.POINTER(Params), C.POINTER(InstView), I32, C.POINTER(TsItem), I32, P, I32, pI32]),
        "sfo_sync_select": (C.c_int, [C.POINTER(Params), C.POINTER(InstView), I32, C.POINTER(TsItem), I32, P, I32,
                                      I32, I32, pI32]),
        "sfo_migrate": (C.c_int, [C.POINTER(Params), C.POINTER(InstView), I32, pI32, pI32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def oracle_config_from_preset(p, scen_idx: Optional[Sequence[int]] = None):
    """(instances, eta, G, Config, keepalive) for a workload.Preset."""
    scs = p.scenarios if scen_idx is None else [p.scenarios[i] for i in scen_idx]
    eta = np.array([s.eta for s in scs], dtype=np.int32)
    inst = np.array([s.instances for s in scs], dtype=np.int32)
    strat = np.array([s.strategy for s in scs], dtype=np.uint32)
    cfg = Config(batch_size=p.batch_size, n_scenarios=len(scs),
                 scenario_eta=_ptr(eta, C.c_int32), scenario_instances=_ptr(inst, C.c_int32),
                 scenario_strategy=_ptr(strat, C.c_uint32),
                 k1=p_k(p, "k1"), k2=p_k(p, "k2"), k3=p_k(p, "k3"), k4=p_k(p, "k4"),
                 k5=p.k5, kp=p.kprefill_ps, M=p.kv_budget, mu=p.mu, phi_tp=p.phi_tp, phi_wait=p.phi_wait,
                 delta=p.snap_period_ps, r=p.route_lat_ps, q=p.pull_lat_ps, R=p.reward_lat_ps,
                 strategy=scs[0].strategy, atw=p.auto_train_windows,
                 pool_capacity_groups=getattr(p, "pool_capacity", None) or p.pool_groups,
                 extra_groups=getattr(p, "extra_groups", 0), extra_members=getattr(p, "extra_members", 0))
    return int(inst[0]), int(eta[0]), p.group_size, cfg, (eta, inst, strat)


def p_k(p, name):
    from paper_2601_12784_b200 import workload as W
    return getattr(p, name + "_ps", None) or {"k1": W.K1_PS, "k2": W.K2_PS, "k3": W.K3_PS, "k4": W.K4_PS}[name]


class OracleSim:
    """One oracle context holding independent scenarios."""

    def __init__(self, instances: int, eta: int, group_size: int, cfg: Config, keepalive=None):
        self.L = load_oracle()
        self._keep = keepalive
        self.cfg = cfg
        self.G = group_size
        self.B = cfg.batch_size
        self.h = C.c_void_p()
        rc = self.L.sfo_create(instances, eta, group_size, C.byref(cfg), C.byref(self.h))
        if rc != 0:
            raise RuntimeError(f"sfo_create failed: {rc}")

    @classmethod
    def from_preset(cls, p, scen_idx=None):
        inst, eta, G, cfg, keep = oracle_config_from_preset(p, scen_idx)
        return cls(inst, eta, G, cfg, keep)

    def close(self):
        if self.h:
            self.L.sfo_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def submit(self, scen: int, prompt: np.ndarray, target: np.ndarray) -> int:
        prompt = np.ascontiguousarray(prompt, dtype=np.int32)
        target = np.ascontiguousarray(target, dtype=np.int32)
        return self.L.sfo_submit_prompts(self.h, scen, len(prompt), _ptr(prompt, C.c_int32), _ptr(target, C.c_int32))

    def step(self, n_windows: int = 1, n_threads: int = 1) -> int:
        return self.L.sfo_step(self.h, n_windows, n_threads)

    def publish(self, scen: int, version: int) -> int:
        return self.L.sfo_publish_params(self.h, scen, version)

    def collect(self, scen: int):
        B = self.B
        vb = np.zeros(1, np.int32)
        g = np.zeros(B, np.int32)
        v = np.zeros(B, np.int32)
        n = np.zeros(1, np.int32)
        rc = self.L.sfo_collect_batch(self.h, scen, B, _ptr(vb, C.c_int32), _ptr(g, C.c_int32),
                                      _ptr(v, C.c_int32), _ptr(n, C.c_int32))
        return rc, int(vb[0]), g, v

    def mark_filtered(self, scen: int, first_group: int, flags) -> int:
        f = np.ascontiguousarray(flags, dtype=np.uint8)
        return self.L.sfo_mark_filtered(self.h, scen, first_group, len(f), _ptr(f, C.c_uint8))

    def filter_group(self, scen: int, group: int) -> int:
        return self.L.sfo_filter_group(self.h, scen, group)

    def metrics(self, scen: Optional[int] = None) -> np.ndarray:
        out = np.zeros(METRICS_LEN, np.int64)
        if scen is None:
            self.L.sfo_read_metrics(self.h, _ptr(out, C.c_int64), METRICS_LEN)
        else:
            self.L.sfo_read_scenario_metrics(self.h, scen, _ptr(out, C.c_int64), METRICS_LEN)
        return out

    def _dump(self, fn, scen, width, dtype, ct):
        n = np.zeros(1, np.int64)
        fn(self.h, scen, None, 0, _ptr(n, C.c_int64))
        out = np.zeros(max(1, int(n[0]) * width), dtype)
        rc = fn(self.h, scen, _ptr(out, ct), int(n[0]), _ptr(n, C.c_int64))
        if rc != 0:
            raise RuntimeError(f"dump failed {rc}")
        return out[: int(n[0]) * width].reshape(-1, width) if width > 1 else out[: int(n[0])]

    def lifecycles(self, scen: int) -> np.ndarray:
        return self._dump(self.L.sfo_dump_lifecycles, scen, 13, np.int64, C.c_int64)

    def batches(self, scen: int) -> np.ndarray:
        n = np.zeros(1, np.int64)
        self.L.sfo_dump_batches(self.h, scen, None, 0, _ptr(n, C.c_int64))
        out = np.zeros(max(1, int(n[0])), np.int32)
        self.L.sfo_dump_batches(self.h, scen, _ptr(out, C.c_int32), int(n[0]), _ptr(n, C.c_int64))
        return out[: int(n[0])]

    def commands(self, scen: int) -> np.ndarray:
        return self._dump(self.L.sfo_dump_commands, scen, 4, np.int64, C.c_int64)

    def instances(self, scen: int) -> np.ndarray:
        return self._dump(self.L.sfo_dump_instances, scen, 7, np.int64, C.c_int64)


class Ledger:
    """Wrapper over the oracle's staleness ledger (§4.2) for unit pins."""

    def __init__(self, eta: int, B: int, _h=None, capacity: int = None):
        self.L = load_oracle()
        self.eta, self.B = eta, B
        self.cap = capacity or B
        self.h = _h if _h is not None else self.L.sfo_ledger_new2(eta, self.cap, B)

    def __del__(self):
        try:
            if self.h:
                self.L.sfo_ledger_free(self.h)
        except Exception:
            pass

    def clone(self):
        return Ledger(self.eta, self.B, self.L.sfo_ledger_clone(self.h), capacity=self.cap)

    def verify(self, v: int) -> bool:
        return bool(self.L.sfo_ledger_verify(self.h, v))

    def reserve(self, g: int, v: int):
        b, s = C.c_int32(), C.c_int32()
        rc = self.L.sfo_ledger_reserve(self.h, g, v, C.byref(b), C.byref(s))
        return (rc, b.value, s.value)

    def delete_relocate(self, g: int) -> int:
        return self.L.sfo_ledger_delete_relocate(self.h, g)

    def abort(self, g: int):
        """abort a tracked entry; returns (rc, moves)."""
        m = C.c_int32()
        rc = self.L.sfo_ledger_abort(self.h, g, C.byref(m))
        return rc, m.value

    def occupy(self, g: int, v: int):
        b, s = C.c_int32(), C.c_int32()
        rc = self.L.sfo_ledger_occupy(self.h, g, v, C.byref(b), C.byref(s))
        return (rc, b.value, s.value)

    def complete(self, g: int, v: int):
        """mark_complete for a fully rewarded group: delete_and_relocate then Occupy."""
        self.delete_relocate(g)
        return self.occupy(g, v)

    def state(self, b: int) -> str:
        return ["Waiting", "Ready", "Stuck"][self.L.sfo_ledger_state(self.h, b)]

    def consume(self):
        g = np.zeros(self.B, np.int32)
        v = np.zeros(self.B, np.int32)
        rc = self.L.sfo_ledger_consume(self.h, _ptr(g, C.c_int32), _ptr(v, C.c_int32))
        return rc, g, v

    def consume_surplus(self):
        g = np.zeros(self.B, np.int32)
        v = np.zeros(self.B, np.int32)
        sp = np.zeros(self.cap, np.int32)
        n = C.c_int32()
        rc = self.L.sfo_ledger_consume2(self.h, _ptr(g, C.c_int32), _ptr(v, C.c_int32), _ptr(sp, C.c_int32), C.byref(n))
        return rc, g, v, sp[: n.value]

    def get(self, b: int, s: int):  # noqa: D401
        st, g, v = C.c_int32(), C.c_int32(), C.c_int32()
        self.L.sfo_ledger_get(self.h, b, s, C.byref(st), C.byref(g), C.byref(v))
        return (["Empty", "Reserved", "Occupied"][st.value], g.value, v.value)

    @property
    def cu(self) -> int:
        return self.L.sfo_ledger_cu(self.h)

    def entries(self, nbuf: int):
        return [[self.get(b, s) for s in range(self.cap)] for b in range(nbuf)]


def make_params(eta=1, k1=None, k2=None, k3=None, k4=None, k5=1, kp=0, M=1 << 40, mu=0.3, phi_tp=5.0,
                phi_wait=3) -> Params:
    from paper_2601_12784_b200 import workload as W
    return Params(k1=W.K1_PS if k1 is None else k1, k2=W.K2_PS if k2 is None else k2,
                  k3=W.K3_PS if k3 is None else k3, k4=W.K4_PS if k4 is None else k4,
                  k5=k5, kp=kp, M=M, mu=mu, phi_tp=phi_tp, phi_wait=phi_wait, eta=eta)


def views(rows) -> "C.Array":
    arr = (InstView * len(rows))()
    for i, (v, kv, n_run, n_wait) in enumerate(rows):
        arr[i] = InstView(v, kv, n_run, n_wait)
    return arr


def items(rows) -> "C.Array":
    arr = (TsItem * max(1, len(rows)))()
    for k, (id_, g, v, l) in enumerate(rows):
        arr[k] = TsItem(id_, g, v, l)
    return arr


def route(params: Params, S, mlq_rows, ledger: Ledger, vanilla=False) -> List[int]:
    Sarr = views(S) if not isinstance(S, C.Array) else S
    it = items(mlq_rows)
    out = np.zeros(max(1, len(mlq_rows)), np.int32)
    n = load_oracle().sfo_route(C.byref(params), Sarr, len(Sarr), it, len(mlq_rows), ledger.h, int(vanilla),
                                _ptr(out, C.c_int32))
    return [int(x) for x in out[:n]], [(s.v, s.kv, s.n_run, s.n_wait) for s in Sarr]


def sync_select(params: Params, S, mlq_rows, ledger: Ledger, ps: int, vanilla_sync=False, vanilla_route=False):
    Sarr = views(S)
    it = items(mlq_rows)
    out = np.zeros(len(S), np.int32)
    n = load_oracle().sfo_sync_select(C.byref(params), Sarr, len(S), it, len(mlq_rows), ledger.h, ps,
                                      int(vanilla_sync), int(vanilla_route), _ptr(out, C.c_int32))
    return [int(x) for x in out[:n]]


def migrate(params: Params, S):
    Sarr = views(S)
    k1 = np.zeros(len(S), np.int32)
    c2 = C.c_int32()
    load_oracle().sfo_migrate(C.byref(params), Sarr, len(S), _ptr(k1, C.c_int32), C.byref(c2))
    return [int(x) for x in k1], c2.value


def mlq_order(rows):
    it = items(rows)
    out = np.zeros(max(1, len(rows)), np.int32)
    load_oracle().sfo_mlq_order(it, len(rows), _ptr(out, C.c_int32))
    return [int(x) for x in out[: len(rows)]]
