"""Seeded synthetic workloads shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no cost model, no ledger, no
routing). It only draws prompt/target lengths and fills in configuration
presets; both implementations receive its arrays and config values as inputs
(DESIGN.md §5 "input recipe").

RNG: counter-based SplitMix64 keyed by (seed, scenario, group, member, stream)
(SURVEY §8(d)). Integer uniforms use Lemire's multiply-high. Lognormals use
Box-Muller in fp64 (numpy, same process for both sides), rounded half away
from zero and clamped to [1, cap]. Group correlation: a shared per-group
normal z_g plus a per-member z_m, so "trajectories within a group tend to be
either all long or all short".

Presets C1..C5 follow SURVEY §8(d) / BASELINE.json `configs`.  `full_run_windows` is the window
count by which every scenario of the preset has reached its train-step count (measured once on the
oracle; tests/test_gpu_fulllength.py asserts it), i.e. the length of one complete run. Time constants
are integer picoseconds (reading A1): Table 6 gives
k1 = 7.28e-8 s/token = 72,800 ps, k2 = 1.72e-3 s, k3 = 1.25e-4 s,
k4 = 1.07e-2 s.
"""
from __future__ import annotations

import dataclasses
import hashlib
import math
from typing import List, Optional

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)

# ---------------------------------------------------------------- constants
PS_PER_S = 1_000_000_000_000
K1_PS = 72_800                 # P:982  7.28e-8 s per KV token
K2_PS = 1_720_000_000          # P:983  1.72e-3 s
K3_PS = 125_000_000            # P:984  1.25e-4 s
K4_PS = 10_700_000_000         # P:985  1.07e-2 s
MU, PHI_WAIT, PHI_TP = 0.3, 3, 5.0

STRAT_R, STRAT_S, STRAT_M = 1, 2, 4  # bit = 1 -> StaleFlow strategy, 0 -> vanilla
STRAT_SF = STRAT_R | STRAT_S | STRAT_M

STREAM_PROMPT, STREAM_GROUP_Z, STREAM_MEMBER_Z, STREAM_TARGET, STREAM_FILTER = 1, 2, 3, 4, 5


def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & M64
    z = x
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & M64
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & M64
    return z ^ (z >> np.uint64(31))


def counter_u64(seed: int, scenario: int, group: np.ndarray, member: np.ndarray,
                stream: int, draw: int = 0) -> np.ndarray:
    """One 64-bit random word per (seed, scenario, group, member, stream, draw)."""
    with np.errstate(over="ignore"):
        g = np.asarray(group, dtype=np.uint64)
        m = np.asarray(member, dtype=np.uint64)
        k = _splitmix64(np.full(g.shape, np.uint64(seed & 0xFFFFFFFFFFFFFFFF)))
        k = _splitmix64(k ^ np.uint64(scenario & 0xFFFFFFFF))
        k = _splitmix64(k ^ g)
        k = _splitmix64(k ^ (m << np.uint64(8)) ^ np.uint64(stream))
        k = _splitmix64(k ^ np.uint64(draw))
        return k


def uniform_int(x: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """Lemire multiply-high: integer uniform on [lo, hi] from 32 random bits."""
    span = np.uint64(hi - lo + 1)
    top = x >> np.uint64(32)
    return (lo + ((top * span) >> np.uint64(32))).astype(np.int64)


def uniform_open01(x: np.ndarray) -> np.ndarray:
    """Double in (0, 1): 53 random bits, offset by half an ulp."""
    return ((x >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def std_normal(seed, scenario, group, member, stream) -> np.ndarray:
    u1 = uniform_open01(counter_u64(seed, scenario, group, member, stream, 0))
    u2 = uniform_open01(counter_u64(seed, scenario, group, member, stream, 1))
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)


@dataclasses.dataclass
class LengthDist:
    kind: str                   # "uniform" or "lognormal"
    lo: int = 1                 # uniform
    hi: int = 1
    median: float = 1.0         # lognormal
    sigma_g: float = 0.0
    sigma_m: float = 0.0
    cap: int = 1


@dataclasses.dataclass
class Scenario:
    """One independent coordination scenario (own ledger, TS, PS, instances)."""
    eta: int
    instances: int
    strategy: int
    seed: int
    skew: Optional[float] = None


@dataclasses.dataclass
class Preset:
    name: str
    scenarios: List[Scenario]
    batch_size: int              # B groups per training step
    group_size: int              # G
    prompt: LengthDist
    target: LengthDist
    kv_budget: int               # M, tokens (reading A2)
    auto_train_windows: int
    train_steps: int
    k5: int = 1
    kprefill_ps: int = 10_000_000         # 10 us / token (reading A20)
    snap_period_ps: int = PS_PER_S        # Delta = 1 s (reading A25)
    route_lat_ps: int = 10_000_000_000    # r = 10 ms
    pull_lat_ps: int = 2 * PS_PER_S       # q = 2 s
    reward_lat_ps: int = PS_PER_S         # R = 1 s
    mu: float = MU
    phi_wait: int = PHI_WAIT
    phi_tp: float = PHI_TP
    extra_groups: int = 0                 # batch-level redundant rollout (App C)
    extra_members: int = 0                # group-level redundant rollout (P:473 footnote)
    filter_prob: float = 0.0              # P(group carries no learning signal), filtered (P:413 (2))
    full_run_windows: int = 0             # windows until every scenario has train_steps batches

    @property
    def members(self) -> int:
        """Members rolled out per group, the redundant ones included."""
        return self.group_size + self.extra_members

    @property
    def pool_groups(self) -> int:
        """Groups submitted per scenario: enough for every train step plus the TS cap (a batch
        retires up to batch_size + extra_groups groups)."""
        etamax = max(s.eta for s in self.scenarios)
        return (self.batch_size + self.extra_groups) * (self.train_steps + etamax + 1)

    def max_inflight(self, eta: int) -> int:
        return (eta + 1) * (self.batch_size + self.extra_groups) * self.members


def draw_lengths(p: Preset, scen_index: int, n_groups: int, group0: int = 0):
    """(prompt_len[n_groups], target_len[n_groups*(G + extra_members)]) int32 for one scenario."""
    sc = p.scenarios[scen_index]
    G = p.members
    g = np.arange(group0, group0 + n_groups, dtype=np.int64)
    prompt = uniform_int(counter_u64(sc.seed, scen_index, g, np.zeros_like(g), STREAM_PROMPT),
                         p.prompt.lo, p.prompt.hi)
    gg = np.repeat(g, G)
    mm = np.tile(np.arange(G, dtype=np.int64), n_groups)
    t = p.target
    if sc.skew is not None:
        t = dataclasses.replace(t, sigma_g=sc.skew / math.sqrt(2.0), sigma_m=sc.skew / math.sqrt(2.0))
    if t.kind == "uniform":
        target = uniform_int(counter_u64(sc.seed, scen_index, gg, mm, STREAM_TARGET), t.lo, t.hi)
    else:
        zg = std_normal(sc.seed, scen_index, gg, np.zeros_like(gg), STREAM_GROUP_Z)
        zm = std_normal(sc.seed, scen_index, gg, mm, STREAM_MEMBER_Z)
        x = np.exp(math.log(t.median) + t.sigma_g * zg + t.sigma_m * zm)
        target = np.floor(x + 0.5)
        target = np.clip(target, 1, t.cap).astype(np.int64)
    return prompt.astype(np.int32), target.astype(np.int32)


def draw_filter_flags(p: Preset, scen_index: int, n_groups: int, group0: int = 0) -> np.ndarray:
    """uint8[n_groups]: 1 for a group whose rewards carry no learning signal (e.g. all identical,
    DAPO dynamic sampling, P:413 (2)), drawn with probability p.filter_prob."""
    sc = p.scenarios[scen_index]
    g = np.arange(group0, group0 + n_groups, dtype=np.int64)
    u = uniform_open01(counter_u64(sc.seed, scen_index, g, np.zeros_like(g), STREAM_FILTER))
    return (u < p.filter_prob).astype(np.uint8)


def sha256_arrays(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


# ---------------------------------------------------------------- presets

def preset(name: str, n_scenarios: Optional[int] = None) -> Preset:
    name = name.upper()
    if name == "C1":
        return Preset("C1", [Scenario(1, 4, STRAT_SF, 1)], 64, 8,
                      LengthDist("uniform", 64, 512), LengthDist("uniform", 128, 2048),
                      131_072, 15, 10, full_run_windows=600)
    if name == "C2":
        return Preset("C2", [Scenario(2, 16, STRAT_R, 2)], 512, 16,
                      LengthDist("uniform", 64, 1024),
                      LengthDist("lognormal", median=2048, sigma_g=0.8, sigma_m=0.6, cap=16_384),
                      1_048_576, 200, 10, full_run_windows=10_500)
    if name == "C3":
        return Preset("C3", [Scenario(3, 32, STRAT_R | STRAT_M, 3)], 128, 16,
                      LengthDist("uniform", 64, 2048),
                      LengthDist("lognormal", median=4096, sigma_g=0.8, sigma_m=0.6, cap=32_768),
                      1_048_576, 60, 10, full_run_windows=4_200)
    if name == "C4":
        sc = []
        for eta in range(5):
            for inst in (8, 16, 32, 64, 128):
                for pull_sf in (0, 1):
                    strat = STRAT_R | STRAT_M | (STRAT_S if pull_sf else 0)
                    sc.append(Scenario(eta, inst, strat, 4))
        if n_scenarios is not None:
            sc = sc[:n_scenarios]
        return Preset("C4", sc, 1024, 16, LengthDist("uniform", 64, 1024),
                      LengthDist("lognormal", median=2048, sigma_g=0.8, sigma_m=0.6, cap=16_384),
                      1_048_576, 120, 5, full_run_windows=22_600)
    if name == "C5":
        n = 4096 if n_scenarios is None else n_scenarios
        sc = []
        skews = (0.25, 0.5, 1.0, 1.5)
        for k in range(n):
            seed, rest = divmod(k, 16)
            eta, skew_i = divmod(rest, 4)
            sc.append(Scenario(eta, 4, STRAT_SF, 5000 + seed, skews[skew_i]))
        return Preset("C5", sc, 64, 8, LengthDist("uniform", 64, 512),
                      LengthDist("lognormal", median=768, cap=4096),
                      131_072, 15, 10, full_run_windows=1_260)
    if name == "C5R":
        # C5 with App C's redundancy ratios (+1/16 of the batch, +1/16 of the group,
        # rounded up to whole groups / members): 64 + 4 groups, 8 + 1 members; 1/16 of the groups
        # filtered at completion (P:413 (2))
        p = preset("C5", n_scenarios)
        return dataclasses.replace(p, name="C5R", extra_groups=4, extra_members=1, filter_prob=1 / 16)
    raise ValueError(f"unknown preset {name}")


def preset_scenario_slice(p: Preset, idx: List[int]) -> Preset:
    """A preset restricted to the given scenario indices (seeds follow the scenario)."""
    q = dataclasses.replace(p, scenarios=[p.scenarios[i] for i in idx])
    q._orig_index = list(idx)  # type: ignore[attr-defined]
    return q


def scenario_lengths(p: Preset, local_index: int, n_groups: int, group0: int = 0):
    orig = getattr(p, "_orig_index", None)
    gi = orig[local_index] if orig is not None else local_index
    sc_backup = p.scenarios
    # draw with the scenario's original index so slices reproduce full-run inputs
    full = dataclasses.replace(p, scenarios=[None] * (gi + 1))  # type: ignore[list-item]
    full.scenarios[gi] = sc_backup[local_index]
    return draw_lengths(full, gi, n_groups, group0)
