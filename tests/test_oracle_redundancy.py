"""Pins for redundant rollout + Abort (PAPER §4.3 P:413, P:473 footnote, App C
P:1085-1093).

* batch level: buffers hold B + extra slots; Ready at >= B Occupied; Consume returns the first B
  Occupied in slot order and aborts the surplus (136 entries -> 128 + 8 aborted);
* group level: groups of G + extra members complete at G rewarded members; the others are aborted
  at once (the 17th member of 16 + 1);
* App C arithmetic: 128 + 128/16 = 136 groups, 16 + 16/16 = 17 members, 2176 trajectories/step;
* invariant fuzz: staleness <= eta, each group consumed once or aborted, aborted trajectories never
  consumed, Abort only for in-flight members, no protocol violation.
"""
import random

import numpy as np
import pytest

from oracle.oracle import Config, Ledger, OracleSim
from tests.test_oracle_sim import IDX

CONSUMED, ABORTED = 6, 7


def test_app_c_arithmetic():
    B, G, ratio_num, ratio_den = 128, 16, 1, 16
    assert B + B * ratio_num // ratio_den == 136
    assert G + G * ratio_num // ratio_den == 17
    assert B * G * (ratio_den + ratio_num) // ratio_den == 2176 == 136 * 16 == 128 * 17


def test_batch_level_consume_136_returns_128():          # S:95 [PAPER] App C
    L = Ledger(0, 128, capacity=136)
    for g in range(136):
        assert L.reserve(g, 0)[0] == 0
    assert L.state(0) == "Stuck"
    done = [g for g in range(136) if g % 17 != 3][:128]   # complete 128 of them (skip 8)
    for g in done:
        L.complete(g, 0)
    assert L.state(0) == "Ready"
    rc, gs, vs, surplus = L.consume_surplus()
    assert rc == 0 and len(gs) == 128 and len(surplus) == 8
    assert sorted(set(gs.tolist()) | set(surplus.tolist())) == list(range(136))
    assert L.cu == 1


def test_batch_level_ready_before_full():
    """Ready as soon as B entries are Occupied, even with empty slots left."""
    L = Ledger(1, 2, capacity=3)
    for g in range(2):
        L.reserve(g, 0)
    for g in range(2):
        L.complete(g, 0)
    assert L.state(0) == "Ready"


def small(B, G, eb=0, em=0, eta=1, I=2, steps=3, seed=0, strategy=7, M=1 << 20, q=30):
    rng = random.Random(seed)
    cfg = Config(batch_size=B, n_scenarios=1, k1=1, k2=100, k3=10, k4=50, k5=1, kp=0, M=M, mu=0.3, phi_tp=5.0,
                 phi_wait=3, delta=1000, r=5, q=q, R=20, strategy=strategy, atw=1, pool_capacity_groups=64,
                 extra_groups=eb, extra_members=em)
    n_groups = (B + eb) * (steps + eta + 2)
    prompt = np.array([rng.randint(1, 40) for _ in range(n_groups)], np.int32)
    target = np.array([rng.randint(1, 60) for _ in range(n_groups * (G + em))], np.int32)
    s = OracleSim(I, eta, G, cfg)
    assert s.submit(0, prompt, target) == 0
    return s, n_groups


def run_batches(s, steps, max_windows=3000):
    for _ in range(max_windows):
        assert s.step(1) == 0
        if s.metrics()[IDX["batches"]] >= steps:
            return
    raise AssertionError("no progress")


def test_group_level_17th_member_aborted():              # S:77 [PAPER] App C: 16 + 16/16
    s, _ = small(B=2, G=16, em=1, eta=1, steps=2)
    run_batches(s, 2)
    lc = s.lifecycles(0)
    b = s.batches(0).reshape(-1, 1 + 2 * 2)
    for g in b[:, 1::2].ravel():
        mem = lc[lc[:, 1] == g]
        assert len(mem) == 17
        assert (mem[:, 6] == CONSUMED).sum() == 16 and (mem[:, 6] == ABORTED).sum() == 1
    m = s.metrics()
    assert m[IDX["aborts"]] >= 2 * 2
    # every Abort command targets an in-flight member of a completed group
    cmds = s.commands(0)
    for w, kind, inst, j in cmds[cmds[:, 1] == 4]:
        assert lc[j, 6] == ABORTED


def test_batch_level_surplus_groups_aborted():
    B, eb = 3, 1
    s, _ = small(B=B, G=2, eb=eb, eta=1, steps=3, seed=3)
    run_batches(s, 3)
    lc = s.lifecycles(0)
    b = s.batches(0).reshape(-1, 1 + 2 * B)
    consumed = b[:, 1::2].ravel().tolist()
    assert len(consumed) == len(set(consumed)) == 3 * B
    aborted_groups = sorted({int(r[1]) for r in lc if r[6] == ABORTED})
    assert not set(aborted_groups) & set(consumed)
    for g in consumed:                                    # consumed groups: all G members consumed
        assert (lc[lc[:, 1] == g][:, 6] == CONSUMED).all()


@pytest.mark.parametrize("seed", range(60))
def test_redundancy_fuzz_invariants(seed):
    """Seeds 30+ use long pulls (q = 1500 ps > Delta) so that aborts land on pulling instances
    (reading R-ABORT: removal at the end of the pull)."""
    rng = random.Random(7000 + seed)
    B, G = rng.randint(1, 5), rng.randint(1, 4)
    eb, em, eta = rng.randint(0, 2), rng.randint(0, 2), rng.randint(0, 3)
    steps = rng.randint(2, 4)
    s, n_groups = small(B, G, eb, em, eta, I=rng.randint(1, 3), steps=steps, seed=seed,
                        strategy=rng.randint(0, 7), M=rng.choice([200, 500, 1 << 20]),
                        q=30 if seed < 30 else 1500)
    run_batches(s, steps)
    m = s.metrics()
    assert m[IDX["violations"]] == 0
    lc = s.lifecycles(0)
    st = lc[:, 11] - lc[:, 5]
    cons = lc[:, 6] == CONSUMED
    assert ((st[cons] >= 0) & (st[cons] <= eta)).all()
    assert m[IDX["tokens"]] == lc[:, 4].sum()
    b = s.batches(0).reshape(-1, 1 + 2 * B)
    groups = b[:, 1::2].ravel()
    assert len(groups) == len(set(groups.tolist())) == steps * B
    for g in groups:
        mem = lc[lc[:, 1] == g]
        assert (mem[:, 6] == CONSUMED).sum() == G                  # exactly the required members
    # aborted trajectories are never consumed and carry no consumed V_buf of their own group batch
    ab = lc[lc[:, 6] == ABORTED]
    for r in ab:
        assert r[1] not in set(groups.tolist()) or em > 0
    assert m[IDX["aborts"]] == len(ab)


# ------------------------------------------------------------------ filtering (P:413 (2))
E_EMPTY, E_RES, E_OCC = "Empty", "Reserved", "Occupied"


def occupied_pair():
    """eta=1, B=1: g1 Occupied in buffer 0 and g0 Occupied (version 0) in buffer 1."""
    L = Ledger(1, 1)
    assert L.reserve(0, 0)[:2] == (0, 1)
    assert L.reserve(1, 0)[:2] == (0, 0)
    L.complete(1, 0)
    L.complete(0, 0)
    assert L.get(0, 0)[:2] == (E_OCC, 1) and L.get(1, 0)[:2] == (E_OCC, 0)
    return L


def test_abort_occupied_moves_later_entry_forward():      # SPEC S:101 example 1
    L = occupied_pair()
    assert L.abort(1) == (0, 1)
    assert L.get(0, 0) == (E_OCC, 0, 0) and L.get(1, 0)[0] == E_EMPTY
    assert L.state(0) == "Ready"


def test_abort_lone_occupied_no_movement():
    L = Ledger(1, 1)
    L.reserve(0, 0)
    L.complete(0, 0)
    b = [x for x in range(2) if L.get(x, 0)[0] == E_OCC][0]
    assert L.abort(0) == (0, 0)
    assert L.get(b, 0)[0] == E_EMPTY


def test_abort_reserved_runs_cascade():                   # Reserved -> delete_and_relocate
    L = Ledger(1, 1)
    L.reserve(0, 0)                                        # buffer 1
    L.reserve(1, 0)                                        # buffer 0
    assert L.abort(0) == (0, 1)                            # g1 (v0 + 1 >= 1) moves into buffer 1
    assert L.get(1, 0)[:2] == (E_RES, 1) and L.get(0, 0)[0] == E_EMPTY


def test_abort_respects_version_constraint():
    """A later Occupied entry whose version exceeds the hole's buffer does not move (v <= hole)."""
    L = Ledger(1, 1)
    L.reserve(0, 0)                                        # buffer 1 (latest)
    L.reserve(1, 0)                                        # buffer 0
    L.complete(1, 0)                                       # g1 Occupied in buffer 0
    assert L.delete_relocate(0) == 0
    assert L.reserve(2, 1)[:2] == (0, 2)                   # version 1 -> buffers 2..1, latest first
    L.complete(2, 1)                                       # occupies buffer 1 (earliest empty >= 0)
    assert L.get(1, 0)[:2] == (E_OCC, 2)
    assert L.abort(1) == (0, 0)                            # v = 1 > hole 0: stays in buffer 1
    assert L.get(1, 0)[:2] == (E_OCC, 2) and L.get(0, 0)[0] == E_EMPTY


def test_abort_unknown_key():
    L = Ledger(1, 2)
    assert L.abort(5)[0] == -1                              # UnknownKey


@pytest.mark.parametrize("seed", range(40))
def test_abort_fuzz_invariants(seed):
    """Random Reserve / complete / abort sequences: every entry keeps 0 <= V_buf - v <= eta and an
    abort removes exactly its own entry (the others are only moved)."""
    rng = random.Random(seed)
    eta, B = rng.randint(0, 3), rng.randint(1, 4)
    L = Ledger(eta, B)
    live = {}                                              # g -> version
    nxt = 0
    for _ in range(200):
        op = rng.random()
        if op < 0.45:
            v = rng.randint(max(0, L.cu - eta), L.cu)          # versions <= ps <= consumed
            rc = L.reserve(nxt, v)
            if rc[0] == 0:
                live[nxt] = v
            nxt += 1
        elif op < 0.75 and live:
            g = rng.choice(sorted(live))
            st = [L.get(b, s) for b in range(L.cu, L.cu + eta + 1) for s in range(B)]
            if any(x[0] == E_RES and x[1] == g for x in st):
                L.complete(g, live[g])
        elif live:
            g = rng.choice(sorted(live))
            before = {(x[1], x[2]) for b in range(L.cu, L.cu + eta + 1) for s in range(B)
                      for x in [L.get(b, s)] if x[0] != E_EMPTY}
            assert L.abort(g)[0] == 0
            del live[g]
            after = {(x[1], x[2]) for b in range(L.cu, L.cu + eta + 1) for s in range(B)
                     for x in [L.get(b, s)] if x[0] != E_EMPTY}
            assert after == {e for e in before if e[0] != g}
        for b in range(L.cu, L.cu + eta + 1):
            for s in range(B):
                st, g, v = L.get(b, s)
                if st != E_EMPTY:
                    assert 0 <= b - v <= eta


def filtered_sim(seed, prob, **kw):
    s, n_groups = small(seed=seed, **kw)
    rng = random.Random(seed + 17)
    flags = np.array([rng.random() < prob for _ in range(n_groups)], np.uint8)
    assert s.mark_filtered(0, 0, flags) == 0
    return s, flags


@pytest.mark.parametrize("seed", range(20))
def test_completion_filter_drops_flagged_groups(seed):
    rng = random.Random(9100 + seed)
    B, G, eta = rng.randint(1, 4), rng.randint(1, 3), rng.randint(0, 2)
    em, eb = rng.randint(0, 1), rng.randint(0, 1)
    s, flags = filtered_sim(seed, 0.3, B=B, G=G, eb=eb, em=em, eta=eta, I=rng.randint(1, 3), steps=8,
                            strategy=rng.randint(0, 7))                     # pool for 8 steps, 3 run
    run_batches(s, 3)
    m = s.metrics()
    assert m[IDX["violations"]] == 0
    b = s.batches(0).reshape(-1, 1 + 2 * B)
    groups = set(b[:, 1::2].ravel().tolist())
    assert len(groups) == 3 * B and not any(flags[g] for g in groups)
    lc = s.lifecycles(0)
    st = lc[:, 11] - lc[:, 5]
    cons = lc[:, 6] == CONSUMED
    assert ((st[cons] >= 0) & (st[cons] <= eta)).all()
    # no member of a flagged group is ever consumed; some flagged group was dropped whole
    fl = flags[lc[:, 1]].astype(bool)
    assert not (cons & fl).any()


def test_completion_filter_whole_group():
    """Group 0 flagged: when it completes its entry is aborted, all members dropped, and the
    batches are filled by later groups."""
    s, n_groups = small(B=2, G=2, eta=0, I=1, steps=3, seed=4)
    flags = np.zeros(n_groups, np.uint8)
    flags[0] = 1
    assert s.mark_filtered(0, 0, flags) == 0
    run_batches(s, 3)
    lc = s.lifecycles(0)
    assert (lc[lc[:, 1] == 0][:, 6] == ABORTED).all()
    b = s.batches(0).reshape(-1, 1 + 2 * 2)
    assert 0 not in set(b[:, 1::2].ravel().tolist()) and len(b) >= 3
    assert s.metrics()[IDX["violations"]] == 0 and s.metrics()[IDX["aborts"]] == 2


def test_proactive_filter_group():                       # SPEC S:96-103 through the simulator
    s, _ = small(B=3, G=2, eta=1, steps=4, seed=11)
    assert s.filter_group(0, 0) == -1                    # nothing routed yet: UnknownKey
    for _ in range(3):
        assert s.step(1) == 0
    lc = s.lifecycles(0)
    tracked = sorted({int(g) for g in lc[lc[:, 5] >= 0][:, 1]})
    assert tracked
    g = tracked[0]
    assert s.filter_group(0, g) == 0
    assert s.filter_group(0, g) == -1                    # already dropped
    lc = s.lifecycles(0)
    assert (lc[lc[:, 1] == g][:, 6] == ABORTED).all()
    run_batches(s, 4)
    b = s.batches(0).reshape(-1, 1 + 2 * 3)
    assert g not in set(b[:, 1::2].ravel().tolist())
    assert s.metrics()[IDX["violations"]] == 0
