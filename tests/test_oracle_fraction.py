"""The oracle against a second, independent transcription with exact rationals (SURVEY §4 item 2,
§8(c) "A tiny-config Python Fraction transcription is diffed against the oracle").

`tests/fraction_sim.py` re-implements SF-SIM-1 from DESIGN.md §3 with `fractions.Fraction` for
every cost-model comparison.  On >= 200 random tiny configurations (all 8 R/S/M strategy mixes,
eta 0..2, 1-3 instances, tight KV budgets, prefill stall k_p > 0, command delays up to and beyond
Delta) every observable must be identical: each trajectory's lifecycle record, the full command
log, the batch compositions, every instance's state and the metric vector (except the command
checksum, our own verification device).  Configurations on which the
transcription saw a comparison within 1e-9 relative of a tie are discarded (fp64 rounding could
legitimately decide those either way) and counted.
"""
import random

import numpy as np
import pytest

from oracle.oracle import Config, OracleSim
from tests.fraction_sim import FracSim

N_CONFIGS = 300
WINDOWS = 60


def tiny_config(rng):
    I, eta, G, B = rng.randint(1, 3), rng.randint(0, 2), rng.randint(1, 3), rng.randint(1, 3)
    kw = dict(k1=rng.choice([1, 2]), k2=rng.choice([60, 100]), k3=rng.choice([7, 10, 30]), k4=50,
              k5=rng.choice([1, 2]), kp=rng.choice([0, 1, 3]), M=rng.choice([150, 300, 2000]),
              mu=rng.choice([0.3, 0.1, 0.8]), phi_tp=rng.choice([5.0, 1.5, 1.2]), phi_wait=rng.choice([0, 1, 3]),
              delta=rng.choice([300, 700, 1500]), r=rng.choice([5, 400]), q=rng.choice([30, 900]),
              R=rng.choice([20, 800]), strategy=rng.randint(0, 7), atw=rng.randint(1, 3))
    steps = rng.randint(2, 4)
    n_groups = B * (steps + eta + 1)
    maxp = 40
    prompt = [rng.randint(1, maxp) for _ in range(n_groups)]
    cap = kw["M"] // kw["k5"] - maxp                         # A27: k5 (p + T) <= M
    target = [rng.randint(1, min(60, cap)) for _ in range(n_groups * G)]
    return I, eta, G, B, kw, np.array(prompt, np.int32), np.array(target, np.int32)


def run_pair(seed):
    rng = random.Random(seed)
    I, eta, G, B, kw, prompt, target = tiny_config(rng)
    cfg = Config(batch_size=B, n_scenarios=1, pool_capacity_groups=len(prompt), **kw)
    o = OracleSim(I, eta, G, cfg)
    assert o.submit(0, prompt, target) == 0
    f = FracSim(I, eta, G, B, **kw)
    f.submit(prompt, target)
    for w in range(WINDOWS):
        assert o.step(1) == 0, f"seed {seed}: oracle failed in window {w}"
        f.window_step()
        if f.ambiguous:
            return f, False
        where = f"seed {seed} window {w}"
        assert o.commands(0).tolist() == [list(c) for c in f.cmds], where
        assert o.lifecycles(0).tolist() == f.lifecycles(), where
        assert o.instances(0).tolist() == f.instances(), where
        assert o.batches(0).tolist() == f.batches, where
        mo = o.metrics(0).tolist()
        mf = f.metrics()
        assert [a for k, a in enumerate(mo) if k != 25] == [a for k, a in enumerate(mf) if k != 25], where
    return f, True


def test_fraction_transcription_matches_oracle():
    cov = dict.fromkeys(["forfeit", "tail", "drain", "held", "prefill"], 0)
    totals = np.zeros(32, np.int64)
    clean = discarded = 0
    for seed in range(N_CONFIGS):
        f, ok = run_pair(seed)
        if not ok:
            discarded += 1
            continue
        clean += 1
        for k in cov:
            cov[k] += f.cov[k]
        m = f.metrics()
        totals += np.array([0 if x is None else x for x in m], np.int64)
    assert clean >= 200, (clean, discarded)
    # the configurations must actually reach every rule the oracle implements
    assert totals[8] > 0 and totals[7] > 0 and totals[6] > 0 and totals[28] > 0 and totals[9] > 0, totals
    assert all(v > 0 for v in cov.values()), cov
