"""GPU parity on the heaviest coordinator windows of the C5 bench workload.

The slowest scenario-windows of the bench (profiles/r01b/coord_phases.txt) are
eta = 0 scenarios right after a training step: every instance pulls, every in-flight trajectory
is interrupted and ~300 of them are re-routed in one window.  Those windows take the versioned
routing fast path far beyond one 32-item batch, overflow the 128-record arrival staging
(kArrStage) and order arrivals from global memory.  This runs the scenarios the phase profile
named, window by window, checks that such a window occurs, and compares every observable with
the oracle (metrics, command log, lifecycles, batches)."""
import numpy as np
import pytest

from paper_2601_12784_b200 import workload as W
from tests.parity import compare, make_pair, submit_both
from tests.test_gpu_parity import launch_mode  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu

HEAVY = [977, 3121, 1681, 1136, 2545, 4018]          # C5 scenario indices (eta 0, 300+ re-routes)
K_ARR_STAGE = 128


def test_heavy_reroute_windows(launch_mode):
    p = W.preset("C5")
    o, g = make_pair(p, HEAVY)
    submit_both(o, g, p, HEAVY)
    n = len(HEAVY)
    prev = np.array([g.metrics(a)[5] for a in range(n)])
    most = 0
    for w in range(100):
        assert o.step(1, 8) == 0
        g.step(1)
        cur = np.array([g.metrics(a)[5] for a in range(n)])
        most = max(most, int((cur - prev).max()))
        prev = cur
        if w % 10 == 9:
            compare(o, g, list(range(n)), where=f"after window {w + 1}")
    assert most > K_ARR_STAGE, f"no heavy re-route window (max routes in a window: {most})"
