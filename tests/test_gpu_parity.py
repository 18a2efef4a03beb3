"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Bar: bit-exact on every integer observable (DESIGN.md §2 makes the fp64 cost-model decisions
identical too): per-scenario metric vectors (incl. the order-sensitive command checksum), the full command log,
every trajectory's lifecycle record, every batch composition and every instance's state.
"""
import random

import numpy as np
import pytest

from oracle.oracle import Config, OracleSim
from paper_2601_12784_b200 import workload as W
from tests.parity import compare, make_pair, run_lockstep, submit_both

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["auto", "split", "lanes", "fused", "block", "step", "dyn", "nopdl"])
def launch_mode(request, monkeypatch):
    """Every launch / decode-step mode must give identical results: the default (a block per
    scenario -- a thread-block cluster for many instances -- when every block gets an SM, else the
    split), the split (three kernels with programmatic dependent launch, one warp per instance and
    closed-form quiet steps in the advance), the one-lane-per-instance advance, the fused window
    kernel, the block / cluster-per-scenario window kernel, one-by-one decode steps, the dataflow
    window kernel, and three fully serialized kernels."""
    monkeypatch.delenv("SF_LAUNCH", raising=False)
    monkeypatch.delenv("SF_ADVANCE", raising=False)
    monkeypatch.delenv("SF_PDL", raising=False)
    if request.param == "dyn":
        monkeypatch.setenv("SF_LAUNCH", "dyn")
    if request.param == "nopdl":
        monkeypatch.setenv("SF_PDL", "0")
    if request.param == "fused":
        monkeypatch.setenv("SF_LAUNCH", "fused")
    if request.param == "block":
        monkeypatch.setenv("SF_LAUNCH", "block")
    if request.param in ("split", "lanes", "step", "nopdl"):
        monkeypatch.setenv("SF_LAUNCH", "split")
    if request.param == "step":
        monkeypatch.setenv("SF_ADVANCE", "step")
    if request.param == "lanes":
        monkeypatch.setenv("SF_ADVANCE", "lanes")
    return request.param


def gpu_from_config(I, eta, G, cfg, cmdlog=100_000):
    from paper_2601_12784_b200.staleflow import StaleFlow
    return StaleFlow(I, eta, G, cfg.batch_size, 1, k1=cfg.k1, k2=cfg.k2, k3=cfg.k3, k4=cfg.k4, k5=cfg.k5,
                     kprefill=cfg.kp, kv_budget=cfg.M, mu=cfg.mu, phi_throughput=cfg.phi_tp, phi_wait=cfg.phi_wait,
                     snap_period=cfg.delta, route_lat=cfg.r, pull_lat=cfg.q, reward_lat=cfg.R,
                     strategy=cfg.strategy, auto_train_windows=cfg.atw, pool_capacity_groups=cfg.pool_capacity_groups,
                     command_log_capacity=cmdlog)


def test_T1_on_gpu(launch_mode):
    cfg = Config(batch_size=1, n_scenarios=1, k1=1, k2=100, k3=10, k4=50, k5=1, kp=0, M=1000, mu=0.3,
                 phi_tp=5.0, phi_wait=3, delta=1000, r=5, q=30, R=20, strategy=7, atw=1, pool_capacity_groups=4)
    o = OracleSim(1, 0, 2, cfg)
    g = gpu_from_config(1, 0, 2, cfg)
    pr, tg = np.array([10, 10], np.int32), np.array([2, 3, 1, 1], np.int32)
    assert o.submit(0, pr, tg) == 0 and g.submit(0, pr, tg) == 0
    run_lockstep(o, g, [0], 4)
    assert g.kernel_launches > 0


def _fuzz_config(rng):
    from tests.test_oracle_sim import small_config
    return small_config(rng)


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_small_configs(seed, launch_mode):
    rng = random.Random(seed)
    I, eta, G, cfg, prompt, target, steps = _fuzz_config(rng)
    o = OracleSim(I, eta, G, cfg)
    g = gpu_from_config(I, eta, G, cfg)
    assert o.submit(0, prompt, target) == 0 and g.submit(0, prompt, target) == 0
    run_lockstep(o, g, [0], 120, every=1)


def test_empty_pool_and_no_work():
    """Degenerate: no prompts submitted -> nothing happens, all snapshots valid."""
    p = W.preset("C1")
    o, g = make_pair(p)
    run_lockstep(o, g, [0], 5)
    assert g.metrics()[2] == 0


def test_external_trainer_collect_publish(launch_mode):
    """External mode (atw = 0): the caller Consumes and Pushes."""
    import dataclasses
    p = dataclasses.replace(W.preset("C1"), auto_train_windows=0)
    o, g = make_pair(p)
    submit_both(o, g, p)
    for w in range(150):
        o.step(1)
        g.step(1)
        ro, vo, go, vvo = o.collect(0)
        rg, vg, gg, vvg = g.collect(0)
        assert ro == rg
        if ro == 0:
            assert vo == vg and (go == gg).all() and (vvo == vvg).all()
            assert o.publish(0, vo + 1) == 0 and g.publish(0, vg + 1) == 0
        assert g.publish(0, 99) == -2           # SF_E_VERSION
        compare(o, g, [0], where=f"external window {w}")


@pytest.mark.parametrize("name,windows,every", [("C1", 400, 25), ("C3", 120, 30), ("C2", 80, 40)])
def test_single_scenario_presets(name, windows, every, launch_mode):
    p = W.preset(name)
    o, g = make_pair(p)
    submit_both(o, g, p)
    run_lockstep(o, g, [0], windows, every=every)


def test_c4_subset(launch_mode):
    p = W.preset("C4")
    idx = [0, 1, 9, 12, 23, 31, 40, 49]                      # eta 0..4, I 8..128, both pull policies
    o, g = make_pair(p, idx)
    submit_both(o, g, p, idx)
    run_lockstep(o, g, list(range(len(idx))), 60, every=30)


def test_c5_full_size_sampled(launch_mode):
    """C5 at full size (4096 scenarios, bench launch configuration) on the GPU; a seeded sample
    of scenarios is recomputed one by one by the oracle (scenarios are independent)."""
    from paper_2601_12784_b200.staleflow import StaleFlow
    p = W.preset("C5")
    g = StaleFlow.from_preset(p, command_log_capacity=0)
    n = len(p.scenarios)
    prs, tgs = zip(*[W.draw_lengths(p, k, p.pool_groups) for k in range(n)])
    assert g.submit_many(np.arange(n), np.full(n, p.pool_groups), np.concatenate(prs), np.concatenate(tgs)) == 0
    g.step(130)
    sample = sorted(random.Random(2026).sample(range(n), 48))
    o = OracleSim.from_preset(p, sample)
    for a, k in enumerate(sample):
        assert o.submit(a, prs[k], tgs[k]) == 0
    assert o.step(130, 8) == 0
    for a, k in enumerate(sample):
        mo, mg = o.metrics(a), g.metrics(k)
        assert (mo == mg).all(), f"scenario {k}: {np.nonzero(mo != mg)}"
        assert (o.lifecycles(a) == g.lifecycles(k)).all()
        assert (o.batches(a) == g.batches(k)).all()


@pytest.mark.parametrize("seed", range(6))
def test_preemption_stress(seed, launch_mode):
    """Tight KV budget and many arrivals per instance: preemptions interleaved with arrival
    admissions inside one window (the register arrival-prefetch path of k_advance)."""
    rng = random.Random(900 + seed)
    I, eta, G, B = rng.randint(1, 2), rng.randint(0, 2), 4, 16
    cfg = Config(batch_size=B, n_scenarios=1, k1=1, k2=100, k3=10, k4=50, k5=1, kp=1, M=1500, mu=0.05,
                 phi_tp=50.0, phi_wait=1000, delta=30000, r=5, q=3000, R=5000, strategy=rng.choice([7, 6, 3]),
                 atw=2, pool_capacity_groups=B * 5)
    steps = 4
    prompt = np.array([rng.randint(1, 120) for _ in range(B * steps)], np.int32)
    target = np.array([rng.randint(1, 300) for _ in range(B * steps * G)], np.int32)
    o = OracleSim(I, eta, G, cfg)
    g = gpu_from_config(I, eta, G, cfg)
    assert o.submit(0, prompt, target) == 0 and g.submit(0, prompt, target) == 0
    run_lockstep(o, g, [0], 150, every=3)
    assert o.metrics()[8] > 0                  # preemptions happened


@pytest.mark.parametrize("seed", range(3))
def test_reward_bursts_beyond_staging(seed, launch_mode):
    """Reward bursts of 300-2048 events per window (mu = 0 routes the whole TS at once; k1 = 0 makes
    steps short, so a batch completes inside one window): the ledger's shared-memory bitonic sort
    (<= 512 events) and its global-scratch sort (more) must apply rewards in exactly the oracle's
    (t_reward, id) order (W8)."""
    rng = random.Random(4000 + seed)
    B, G, I, eta = 128, 8, 8, 1
    cfg = Config(batch_size=B, n_scenarios=1, k1=0, k2=100, k3=1, k4=50, k5=1, kp=0, M=1 << 20, mu=0.0,
                 phi_tp=50.0, phi_wait=1000, delta=6000, r=5, q=300, R=6000, strategy=rng.choice([7, 5]), atw=1,
                 pool_capacity_groups=B * 8)
    prompt = np.array([rng.randint(1, 20) for _ in range(B * 8)], np.int32)
    target = np.array([rng.randint(30, 40) for _ in range(B * 8 * G)], np.int32)
    o = OracleSim(I, eta, G, cfg)
    g = gpu_from_config(I, eta, G, cfg)
    assert o.submit(0, prompt, target) == 0 and g.submit(0, prompt, target) == 0
    run_lockstep(o, g, [0], 24, every=1)
    assert o.metrics()[9] >= 6                   # batches
