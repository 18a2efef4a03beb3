"""Pins for the oracle's cost model (Eq 2-4, Eq 7) and strategies (Alg 2-4).

Closed forms are SPEC.md's hand evaluations of Table 6, restated
in integer picoseconds (reading A1).  Strategy examples are SPEC's worked
examples.  Routing decisions are re-derived with exact rational
arithmetic (fractions.Fraction, a different arithmetic than the oracle's fp64)
and the "64/72/77 trajectories per empty instance" pin is solved exactly.
"""
import random
from fractions import Fraction

import pytest

from oracle import oracle as O
from paper_2601_12784_b200 import workload as W

P = O.make_params()
L = O.load_oracle()
PS = 10 ** 12


# ---------------------------------------------------------------- Eq 7 / Eq 2 / Eq 4
def test_tick_latency_table6():                          # 2.684e-2 s
    assert L.sfo_tick_latency(P, 50_000, 100, 0) == 26_840_000_000


def test_tick_latency_floor_and_flat_region():
    assert L.sfo_tick_latency(P, 0, 0, 0) == W.K2_PS + W.K4_PS
    assert L.sfo_tick_latency(P, 1000, 5, 0) == L.sfo_tick_latency(P, 1000, 13, 0)   # n < k2/k3
    assert L.sfo_tick_latency(P, 1000, 14, 0) > L.sfo_tick_latency(P, 1000, 13, 0)


def test_breakpoint():                                   # k2/k3 = 13.76
    assert Fraction(W.K2_PS, W.K3_PS) == Fraction(1376, 100)


def test_prefill_term_linear():                          # reading A20
    p = O.make_params(kp=10_000_000)
    assert L.sfo_tick_latency(p, 10, 1, 512) - L.sfo_tick_latency(p, 10, 1, 0) == 512 * 10_000_000


def test_throughput_table6():                            # 3725.8 tok/s
    t = L.sfo_throughput(P, 100, 50_000) * PS
    assert abs(t - 100 / 2.684e-2) < 1e-9 * t
    assert round(t, 1) == 3725.8
    assert L.sfo_throughput(P, 0, 123) == 0.0


def test_ideal_gain_table6():                            # 80.05 tok/s
    g = L.sfo_ideal_gain(P, 1000) * PS
    assert round(g, 2) == 80.05
    assert L.sfo_ideal_gain(P, 0) * PS == pytest.approx(1 / ((W.K2_PS + W.K4_PS) / PS))


def test_marginal_gain_cases():
    idle = O.InstView(0, 0, 0, 0)
    assert L.sfo_marginal_gain(P, idle, 1000) == L.sfo_ideal_gain(P, 1000)      # exact equality
    assert L.sfo_marginal_gain(P, O.InstView(0, 100, 3, 1), 1000) == 0.0          # wait non-empty
    small = O.make_params(M=1500)
    assert L.sfo_marginal_gain(small, O.InstView(0, 600, 1, 0), 1000) == 0.0      # over budget


def test_monotone_and_ideal_upper_bound():
    rng = random.Random(3)
    for _ in range(2000):
        n = rng.randint(1, 300)
        kv = rng.randint(0, 1_000_000)
        assert L.sfo_throughput(P, n, 2 * kv + 1) < L.sfo_throughput(P, n, kv) or kv == 0
        l = rng.randint(0, 40_000)
        mg = L.sfo_marginal_gain(P, O.InstView(0, kv, n, rng.choice([0, 0, 2])), l)
        assert mg <= L.sfo_ideal_gain(P, l)


# ---------------------------------------------------------------- exact re-derivation helpers
def T_exact(n, kv, p=P):
    if n == 0:
        return Fraction(0)
    return Fraction(n, p.k1 * kv + max(p.k2, p.k3 * n) + p.k4)


def dT_exact(s, l, p=P):
    v, kv, n, nw = s
    if not (kv + p.k5 * l <= p.M and nw == 0):
        return Fraction(0)
    return T_exact(n + 1, kv + p.k5 * l, p) - T_exact(n, kv, p)


def ideal_exact(l, p=P):
    return Fraction(1, p.k1 * p.k5 * l + max(p.k2, p.k3) + p.k4)


@pytest.mark.parametrize("prompt,expected", [(512, 64), (256, 72), (128, 77)])
def test_waterfall_fill_of_empty_instance(prompt, expected):
    """an empty instance accepts 64 / 72 / 77 initial trajectories (cf. ~100)."""
    mu = Fraction(3, 10)
    n, kv = 0, 0
    while dT_exact((0, kv, n, 0), prompt) >= mu * ideal_exact(prompt):
        n, kv = n + 1, kv + prompt
    assert n == expected                                  # exact rational solution
    led = O.Ledger(0, 10_000)
    rows = [(k, k, -1, prompt) for k in range(200)]       # G = 1: one group per trajectory
    routed, S = O.route(P, [(0, 0, 0, 0)], rows, led)
    assert len(routed) == expected                        # the oracle's fp64 waterfall agrees


# ---------------------------------------------------------------- Alg 2 routing
def test_routing_prefers_idle_over_full_wait():
    led = O.Ledger(1, 8)
    S = [(0, 900_000, 60, 5), (0, 0, 0, 0)]
    routed, _ = O.route(P, S, [(0, 0, -1, 500)], led)
    assert routed == [1]


def test_routing_withholds_below_threshold():            # S:280 [PAPER] "temporarily withheld"
    led = O.Ledger(1, 8)
    S = [(0, 5_000_000, 400, 0)]                          # heavily loaded: gain << mu * ideal
    p = O.make_params(M=10 ** 9)
    routed, _ = O.route(p, S, [(0, 0, -1, 500)], led)
    assert routed == []


def test_routing_stop_flag_skips_lower_queues():         # S:281 [PAPER] Alg 2 stop flag
    led = O.Ledger(1, 8)
    S = [(0, 0, 0, 0)]
    rows = [(5, 5, 3, 100), (0, 0, -1, 100)]              # v=3 partial head is unroutable on v=0
    routed, _ = O.route(P, S, rows, led)
    assert routed == []


def test_vanilla_routing_fewest():
    led = O.Ledger(1, 8)
    routed, _ = O.route(P, [(0, 0, 2, 1), (0, 0, 5, 0)], [(0, 0, -1, 10)], led, vanilla=True)
    assert routed == [0]


def test_group_members_pinned_to_first_version():        # reading A11
    led = O.Ledger(1, 8)
    S = [(0, 0, 0, 0), (1, 0, 0, 0)]
    rows = [(0, 0, -1, 100), (1, 0, -1, 100)]
    routed, _ = O.route(P, S, rows, led)
    assert len(routed) == 2                               # first member fixes v_g, second follows


def test_mlq_order():
    rows = [(9, 9, 1, 5), (4, 4, 0, 5), (2, 2, -1, 5), (7, 7, 0, 5)]
    order = O.mlq_order(rows)
    assert [rows[k][0] for k in order] == [4, 7, 9, 2]


@pytest.mark.parametrize("seed", range(8))
def test_routing_decisions_exact_arithmetic(seed):
    """Every fp64 waterfall decision equals the exact-rational decision (no near-ties)."""
    rng = random.Random(seed)
    for _ in range(40):
        I = rng.randint(1, 8)
        S = [(rng.randint(0, 2), rng.randint(0, 400_000), rng.randint(0, 150), rng.choice([0, 0, 0, 1]))
             for _ in range(I)]
        S = [(v, kv if n else 0, n, w) for (v, kv, n, w) in S]
        rows = [(k, k, rng.choice([-1, -1, 0, 1, 2]), rng.randint(64, 3000)) for k in range(30)]
        rows = [rows[k] for k in O.mlq_order(rows)]
        led = O.Ledger(2, 64)
        routed, _ = O.route(P, S, rows, led)
        # replay with Fractions (ledger never binds here: 3 x 64 slots, <= 30 reserves)
        cur = [list(s) for s in S]
        mu = Fraction(3, 10)
        for k, inst in enumerate(routed):
            _, _, v_tau, l = rows[k]
            cand = [i for i in range(I) if v_tau < 0 or cur[i][0] >= v_tau]
            thr = mu * ideal_exact(l)
            sel = None
            for ver in sorted({cur[i][0] for i in cand}):
                grp = [i for i in cand if cur[i][0] == ver]
                gains = [dT_exact(tuple(cur[i]), l) for i in grp]
                best = max(gains)
                # no near-ties between the best and another candidate or the threshold
                for gval in gains:
                    assert gval == best or abs(float(best - gval)) > 1e-12 * float(best or 1)
                if best >= thr:
                    sel = grp[gains.index(best)]
                    break
            assert sel == inst
            s = cur[sel]
            if s[1] + l <= P.M and s[3] == 0:
                s[2] += 1
                s[1] += l
            else:
                s[3] += 1


# ---------------------------------------------------------------- Alg 3 sync
def test_sync_up_to_date_never_selected():
    led = O.Ledger(1, 4)
    assert O.sync_select(P, [(2, 0, 0, 0)], [(0, 0, -1, 100)], led, 2) == []


def test_sync_not_selected_when_partial_routable():
    led = O.Ledger(1, 4)
    assert O.sync_select(P, [(1, 0, 0, 0)], [(0, 0, 1, 100)], led, 2) == []


def test_sync_selected_when_update_unlocks():
    led = O.Ledger(0, 1)
    assert led.reserve(99, 0)[1] == 0                     # buffer 0 full: verify(0) false
    sel = O.sync_select(P, [(0, 0, 0, 0)], [(0, 0, -1, 100)], led, 1)
    assert sel == [0]
    assert led.verify(1) and not led.verify(0)            # tentative routing used a scratch ledger
    assert led.get(1, 0)[0] == "Empty"


def test_vanilla_sync_all_stale():
    led = O.Ledger(1, 4)
    assert O.sync_select(P, [(0, 0, 0, 0), (1, 0, 0, 0), (0, 0, 0, 0)], [], led, 1, vanilla_sync=True) == [0, 2]


# ---------------------------------------------------------------- Alg 4 migration
def test_migration_case1_excess():
    k1, c2 = O.migrate(P, [(0, 1000, 10, 5), (0, 1000, 10, 0)])
    assert k1 == [2, 0] and c2 == -1


def test_migration_case2_drain_max():                    # ratio 6 > 5
    # T = n / (k1 kv + max(k2, k3 n) + k4): instance 0 has 60 running on little KV,
    # instance 1 has 1 running on a huge KV.
    S = [(0, 60 * 100, 60, 0), (0, 400_000, 1, 0)]
    T0 = L.sfo_throughput(P, 60, 6000)
    T1 = L.sfo_throughput(P, 1, 400_000)
    assert T0 / T1 > 5
    k1, c2 = O.migrate(P, S)
    assert c2 == 0


def test_migration_disabled_with_empty_instance():       # S:299, reading A6
    k1, c2 = O.migrate(P, [(0, 6000, 60, 0), (0, 0, 0, 0)])
    assert c2 == -1
