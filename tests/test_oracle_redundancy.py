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
