"""GPU parity of redundant rollout + Abort (PAPER P:413, P:473 footnote, App C
P:1085-1093): the CUDA path against the oracle, element by element (metrics incl.
the command hash, command log with Abort records, lifecycles incl. the aborted state, batches,
instance state), in every launch / decode-step mode."""
import dataclasses
import random

import numpy as np
import pytest

from oracle.oracle import Config, OracleSim
from paper_2601_12784_b200 import workload as W
from tests.parity import compare, make_pair, run_lockstep, submit_both
from tests.test_gpu_parity import launch_mode  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu

ABORTS = 31


def gpu_from_config(I, eta, G, cfg, cmdlog=100_000):
    from paper_2601_12784_b200.staleflow import StaleFlow
    return StaleFlow(I, eta, G, cfg.batch_size, 1, k1=cfg.k1, k2=cfg.k2, k3=cfg.k3, k4=cfg.k4, k5=cfg.k5,
                     kprefill=cfg.kp, kv_budget=cfg.M, mu=cfg.mu, phi_throughput=cfg.phi_tp, phi_wait=cfg.phi_wait,
                     snap_period=cfg.delta, route_lat=cfg.r, pull_lat=cfg.q, reward_lat=cfg.R,
                     strategy=cfg.strategy, auto_train_windows=cfg.atw, pool_capacity_groups=cfg.pool_capacity_groups,
                     command_log_capacity=cmdlog, extra_groups=cfg.extra_groups, extra_members=cfg.extra_members)


def pair(I, eta, G, B, eb, em, *, seed, M=1 << 20, q=30, strategy=7, atw=1, steps=4, kp=0, delta=1000, R=20,
         plen=(1, 40), tlen=(1, 60), cmdlog=100_000):
    rng = random.Random(seed)
    cfg = Config(batch_size=B, n_scenarios=1, k1=1, k2=100, k3=10, k4=50, k5=1, kp=kp, M=M, mu=0.3, phi_tp=5.0,
                 phi_wait=3, delta=delta, r=5, q=q, R=R, strategy=strategy, atw=atw,
                 pool_capacity_groups=(B + eb) * (steps + eta + 2), extra_groups=eb, extra_members=em)
    n_groups = cfg.pool_capacity_groups
    prompt = np.array([rng.randint(*plen) for _ in range(n_groups)], np.int32)
    target = np.array([rng.randint(*tlen) for _ in range(n_groups * (G + em))], np.int32)
    o = OracleSim(I, eta, G, cfg)
    g = gpu_from_config(I, eta, G, cfg, cmdlog)
    assert o.submit(0, prompt, target) == 0 and g.submit(0, prompt, target) == 0
    return o, g


@pytest.mark.parametrize("seed", range(40))
def test_redundancy_fuzz(seed, launch_mode):
    rng = random.Random(7000 + seed)
    B, G = rng.randint(1, 5), rng.randint(1, 4)
    eb, em, eta = rng.randint(0, 2), rng.randint(0, 2), rng.randint(0, 3)
    if eb == em == 0:
        eb = 1
    o, g = pair(rng.randint(1, 3), eta, G, B, eb, em, seed=seed, M=rng.choice([200, 500, 1 << 20]),
                q=30 if seed < 20 else 1500, strategy=rng.randint(0, 7))
    run_lockstep(o, g, [0], 150)
    assert g.metrics()[ABORTS] > 0 or seed % 7 == 0     # aborts actually happen in (almost) every case


def test_app_c_17th_member(launch_mode):                 # 16 + 1 members, the last one aborted
    o, g = pair(2, 1, 16, 2, 0, 1, seed=5, steps=3)
    run_lockstep(o, g, [0], 200, every=5)
    lc = g.lifecycles(0)
    b = g.batches(0).reshape(-1, 1 + 2 * 2)
    assert len(b) >= 3
    for grp in b[:, 1::2].ravel():
        st = lc[lc[:, 1] == grp][:, 6]
        assert (st == 6).sum() == 16 and (st == 7).sum() == 1


@pytest.mark.parametrize("seed", range(6))
def test_redundancy_preemption_and_global_path(seed, launch_mode):
    """Tight KV budget (aborts of running and waiting members, KV release at the boundary) and
    instances holding more than 128 run + wait + arrival entries (the global-memory advance path)."""
    rng = random.Random(300 + seed)
    I = 1 if seed % 2 == 0 else 2
    o, g = pair(I, rng.randint(1, 2), 8, 12, rng.randint(1, 3), rng.randint(1, 2), seed=seed, M=rng.choice([900, 3000]),
                q=3000, strategy=rng.choice([7, 6, 3]), atw=2, steps=3, kp=1, delta=30000, R=5000, plen=(5, 60),
                tlen=(20, 200), cmdlog=400_000)
    run_lockstep(o, g, [0], 300, every=10)
    m = g.metrics()
    assert m[ABORTS] > 0 and m[9] >= 4


def test_external_trainer_with_surplus(launch_mode):
    """atw = 0: sf_collect_batch returns the first B Occupied groups and aborts the surplus."""
    p = dataclasses.replace(W.preset("C1"), auto_train_windows=0, extra_groups=4, extra_members=1)
    o, g = make_pair(p)
    submit_both(o, g, p)
    n_batches = 0
    for w in range(300):
        o.step(1)
        g.step(1)
        ro, vo, go, vvo = o.collect(0)
        rg, vg, gg, vvg = g.collect(0)
        assert ro == rg
        if ro == 0:
            n_batches += 1
            assert len(gg) == p.batch_size
            assert vo == vg and (go == gg).all() and (vvo == vvg).all()
            assert o.publish(0, vo + 1) == 0 and g.publish(0, vg + 1) == 0
        compare(o, g, [0], where=f"external window {w}")
    assert n_batches >= 2 and g.metrics()[ABORTS] > 0


def test_c5r_subset_lockstep(launch_mode):
    """C5 with App C's redundancy ratios, 16 scenarios (all eta / skew combinations of one seed)."""
    p = W.preset("C5R", n_scenarios=16)
    o, g = make_pair(p)
    submit_both(o, g, p)
    run_lockstep(o, g, list(range(16)), 160, every=20)
    m = g.metrics()
    assert m[ABORTS] > 0 and m[9] >= 30


def test_c5r_full_size_sampled():
    """C5R at full size (4096 scenarios); a seeded sample recomputed by the oracle."""
    from paper_2601_12784_b200.staleflow import StaleFlow
    p = W.preset("C5R")
    g = StaleFlow.from_preset(p, command_log_capacity=0)
    n = len(p.scenarios)
    prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
    assert g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs)) == 0
    flags = [W.draw_filter_flags(p, k, p.pool_groups) for k in range(n)]
    for k in range(n):
        g.mark_filtered(k, 0, flags[k])
    g.step(130)
    sample = sorted(random.Random(2027).sample(range(n), 32))
    o = OracleSim.from_preset(p, sample)
    for a, k in enumerate(sample):
        assert o.submit(a, prs[k], tgs[k]) == 0
        assert o.mark_filtered(a, 0, flags[k]) == 0
    assert o.step(130, 8) == 0
    for a, k in enumerate(sample):
        mo, mg = o.metrics(a), g.metrics(k)
        assert (mo == mg).all(), f"scenario {k}: {np.nonzero(mo != mg)}"
        assert (o.lifecycles(a) == g.lifecycles(k)).all()
        assert (o.batches(a) == g.batches(k)).all()


@pytest.mark.parametrize("seed", range(24))
def test_completion_filter_fuzz(seed, launch_mode):
    """Groups flagged as carrying no learning signal are dropped when they complete (P:413 (2)):
    entry aborted, later Occupied entries moved forward, members aborted."""
    rng = random.Random(9100 + seed)
    B, G, eta = rng.randint(1, 4), rng.randint(1, 3), rng.randint(0, 2)
    em, eb = rng.randint(0, 1), rng.randint(0, 1)
    o, g = pair(rng.randint(1, 3), eta, G, B, eb, em, seed=seed, steps=8, strategy=rng.randint(0, 7),
                M=rng.choice([300, 1 << 20]))
    n_groups = (B + eb) * (8 + eta + 2)
    fr = random.Random(seed + 17)
    flags = np.array([fr.random() < 0.3 for _ in range(n_groups)], np.uint8)
    assert o.mark_filtered(0, 0, flags) == 0
    g.mark_filtered(0, 0, flags)
    run_lockstep(o, g, [0], 200, every=2)


@pytest.mark.parametrize("seed", range(12))
def test_proactive_filter_fuzz(seed, launch_mode):
    """sf_filter_group between windows on random tracked (and untracked) groups, in lockstep."""
    rng = random.Random(5500 + seed)
    B, G, eta = rng.randint(1, 4), rng.randint(1, 3), rng.randint(0, 2)
    o, g = pair(rng.randint(1, 3), eta, G, B, rng.randint(0, 1), rng.randint(0, 1), seed=seed, steps=8,
                strategy=rng.randint(0, 7))
    n_filtered = 0
    for w in range(150):
        assert o.step(1) == 0
        g.step(1)
        if rng.random() < 0.3:
            lc = o.lifecycles(0)
            tracked = sorted({int(x) for x in lc[lc[:, 5] >= 0][:, 1]})      # routed groups
            cand = tracked if tracked and rng.random() < 0.8 else sorted({int(x) for x in lc[:, 1]})
            grp = rng.choice(cand)
            ro, rg = o.filter_group(0, grp), g.filter_group(0, grp)
            assert ro == rg, (w, grp, ro, rg)
            n_filtered += ro == 0
        compare(o, g, [0], where=f"window {w}")
    assert n_filtered > 0
