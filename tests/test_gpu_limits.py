"""GPU parity at the library's size limits and the ABI's error paths (include/staleflow.h).

Limits: 128 instances in one scenario (the 4-instances-per-lane coordinator, KS = 4), the largest
staleness bound the on-chip ledger view supports (eta = 15), groups far beyond the group-batched
routing (G = 1024), and the degenerate B = G = 1.  Error paths: every status code an entry point
documents, and that a failed call leaves the context usable (only SF_E_STATE / SF_E_CUDA poison)."""
import random

import numpy as np
import pytest

from oracle.oracle import Config, OracleSim
from tests.parity import run_lockstep
from tests.test_gpu_parity import gpu_from_config, launch_mode  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu

OK, NOT_READY, E_INVALID, E_VERSION, E_STATE, E_RANGE = 0, 1, -1, -2, -3, -6


def cfg_of(B, M=1 << 20, delta=1000, q=30, R=20, atw=1, pool=64, strategy=7, k1=1, k2=100, k3=10, k4=50):
    return Config(batch_size=B, n_scenarios=1, k1=k1, k2=k2, k3=k3, k4=k4, k5=1, kp=0, M=M, mu=0.3, phi_tp=5.0,
                  phi_wait=3, delta=delta, r=5, q=q, R=R, strategy=strategy, atw=atw, pool_capacity_groups=pool)


def lengths(seed, n_groups, G, plen=(1, 60), tlen=(1, 90)):
    rng = random.Random(seed)
    return (np.array([rng.randint(*plen) for _ in range(n_groups)], np.int32),
            np.array([rng.randint(*tlen) for _ in range(n_groups * G)], np.int32))


def pair(I, eta, G, cfg, prompt, target):
    o = OracleSim(I, eta, G, cfg)
    g = gpu_from_config(I, eta, G, cfg)
    assert o.submit(0, prompt, target) == 0 and g.submit(0, prompt, target) == 0
    return o, g


@pytest.mark.parametrize("strategy", [7, 0, 3])
def test_128_instances(strategy, launch_mode):
    """I = 128: four instances per coordinator lane; migration and sync over all of them."""
    B, G = 24, 8
    cfg = cfg_of(B, M=4000, delta=2000, q=400, pool=B * 8, strategy=strategy)
    o, g = pair(128, 2, G, cfg, *lengths(1, B * 8, G, tlen=(20, 400)))
    run_lockstep(o, g, [0], 120, every=4)
    assert g.metrics()[9] > 0


def test_eta_15(launch_mode):
    """The largest staleness bound of the on-chip ledger view (kMaxEta = 15)."""
    B, G = 3, 2
    cfg = cfg_of(B, pool=B * 24)
    o, g = pair(3, 15, G, cfg, *lengths(2, B * 24, G))
    run_lockstep(o, g, [0], 400, every=8)
    m = g.metrics()
    assert m[9] > 0 and m[12] == 0


def test_large_groups(launch_mode):
    """G = 1024 members per group: group-batched routing does not apply (G > 16), long ids."""
    B, G = 2, 1024
    cfg = cfg_of(B, M=1 << 22, pool=B * 4, k1=0, delta=200_000)
    o, g = pair(4, 1, G, cfg, *lengths(3, B * 4, G, tlen=(1, 40)))
    run_lockstep(o, g, [0], 300, every=20)
    assert g.metrics()[9] > 0


def test_single_group_single_member(launch_mode):
    cfg = cfg_of(1, pool=12)
    o, g = pair(1, 0, 1, cfg, *lengths(4, 12, 1))
    run_lockstep(o, g, [0], 200, every=5)
    assert g.metrics()[9] >= 10


# ------------------------------------------------------------------ ABI error paths
def make(**kw):
    from paper_2601_12784_b200.staleflow import StaleFlow
    args = dict(instances=2, eta=1, group_size=2, batch_size=2, n_scenarios=1, kv_budget=1000, pool_capacity_groups=4,
                snap_period=1000, k1=1, k2=100, k3=10, k4=50, kprefill=0, route_lat=5, pull_lat=30, reward_lat=20)
    args.update(kw)
    return StaleFlow(**args)


@pytest.mark.parametrize("bad", [dict(batch_size=0), dict(group_size=0), dict(group_size=5000), dict(eta=16),
                                 dict(instances=129), dict(kv_budget=1 << 30), dict(k1=1 << 31), dict(k5=0),
                                 dict(snap_period=0), dict(pool_capacity_groups=0), dict(extra_groups=-1),
                                 dict(extra_members=-1),
                                 # grp_of()'s 64-bit multiply-shift would wrap: G = 1 beyond 2^24
                                 # trajectories, G = 3 beyond ~3 * 2^24
                                 dict(group_size=1, pool_capacity_groups=(1 << 24) + 1),
                                 dict(group_size=3, pool_capacity_groups=(1 << 24) + 1),
                                 # per-scenario list offsets would pass 2^31 (cap = (eta+1) B G in int64)
                                 dict(eta=15, batch_size=1 << 16, group_size=4096, pool_capacity_groups=1)])
def test_create_rejects_invalid_config(bad):
    from paper_2601_12784_b200.staleflow import SfError
    with pytest.raises(SfError):
        make(**bad)


def test_call_errors_do_not_poison():
    ctx = make()
    L, h = ctx.L, ctx.h
    p = np.array([10, 10], np.int32)
    assert ctx.submit(0, p, np.array([0, 5, 5, 5], np.int32)) == E_INVALID        # target < 1
    assert ctx.submit(0, p, np.array([5, 2000, 5, 5], np.int32)) == E_INVALID     # k5 (p + T) > M (A27)
    assert ctx.submit(3, p, np.array([5, 5, 5, 5], np.int32)) == E_RANGE          # scenario index
    big = np.full(5, 10, np.int32)
    assert ctx.submit(0, big, np.full(10, 5, np.int32)) == E_RANGE                # pool capacity
    assert ctx.submit(0, p, np.array([5, 5, 5, 5], np.int32)) == OK
    assert ctx.publish(0, 5) == E_VERSION                                         # not ps + 1
    assert ctx.publish(0, 1) == E_VERSION                                         # > consumed batches
    assert ctx.collect(0)[0] == NOT_READY                                         # buffer 0 Waiting
    assert ctx.filter_group(0, 0) == E_INVALID                                    # group not tracked yet
    out = np.zeros(1, np.int32)
    import ctypes as C
    assert L.sf_collect_batch(h, 0, 1, None, None, None, out.ctypes.data_as(C.POINTER(C.c_int32))) == E_RANGE
    assert out[0] == 2                                                            # *n_out = B
    ctx.step(3)                                                                   # still usable
    assert ctx.metrics()[0] == 3


def test_binding_rejects_mismatched_shapes():
    """The binding checks array sizes before handing host pointers to the C ABI: a short
    target array would otherwise be over-read by sf_submit_prompts[_many]."""
    from paper_2601_12784_b200.staleflow import SfError
    ctx = make(extra_members=1)                          # 3 members per group
    p = np.array([10, 10], np.int32)
    with pytest.raises(SfError):
        ctx.submit(0, p, np.full(4, 5, np.int32))        # 2 groups x 2 members: one member short per group
    with pytest.raises(SfError):
        ctx.submit_many([0], [2], p, np.full(4, 5, np.int32))
    with pytest.raises(SfError):
        ctx.submit_many([0, 0], [2], p, np.full(6, 5, np.int32))
    assert ctx.submit(0, p, np.full(6, 5, np.int32)) == OK


def test_watchdog_deadlock_matches_oracle():
    """SPEC S:494 Deadlock: the hand-derived starved batch of tests/test_oracle_pins.py on the GPU: the
    library poisons the scenario in the same window as the oracle and sf_step returns SF_E_STATE."""
    from paper_2601_12784_b200.staleflow import SfError
    from tests.test_oracle_pins import watchdog_sim
    o = watchdog_sim(3)
    g2 = make(instances=1, eta=0, group_size=1, batch_size=2, kv_budget=1000, pool_capacity_groups=2,
              auto_train_windows=1, watchdog_windows=3)
    assert g2.submit(0, np.array([10], np.int32), np.array([2], np.int32)) == OK
    g2.step(3, stats=True)
    with pytest.raises(SfError, match="deadlock .* at window 4"):
        g2.step(1, stats=True)                  # a synchronizing call reports the poisoned scenario
    assert o.step(3) == 0 and o.step(1) == E_STATE
    assert o.metrics(0)[0] == 4                 # the oracle fails in the same window (4 windows run)
    with pytest.raises(SfError):                # the context is poisoned (include/staleflow.h)
        g2.metrics(0)
