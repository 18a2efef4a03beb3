"""Round-2 pins for the parts of the oracle that round 1 held only by invariants.

* T3 (tests/golden/t3_timeline.txt): a hand-derived I=2, eta=1 timeline with the prefill stall, LIFO
  preemption (B4, A21), case-1 and case-2 migration (Alg 4), an Interrupt that forfeits
  the in-flight token (B1, A18), a relocation cascade with two Reserved candidates in one buffer
  (A13), a Sync with held arrivals (Alg 3) and staleness-1 batches.
* Eq 1 gatekeeping (SPEC S:624 acceptance 3, Fig 9a): with route and pull delays longer
  than the snapshot period every snapshot taken before the commands took effect is rejected, and no
  command is issued twice, under vanilla sync (which would re-Pull every stale instance on an
  accepted snapshot).
* delete-and-relocate (reading A13): a two-move cascade to a fixpoint whose candidates
  sit in two earlier buffers (earliest buffer first, version eligibility v + eta >= hole), and a
  choice between two Reserved entries of one buffer (lowest slot first).
"""
import os

import numpy as np

from oracle.oracle import Config, Ledger, OracleSim

GOLD = os.path.join(os.path.dirname(__file__), "golden", "t3_timeline.txt")
IDX = {n: k for k, n in enumerate(__import__("oracle").METRIC_NAMES)}
T3_AFTER = ["ticks", "traj_iters", "tokens", "completions", "routes", "interrupts", "pulls", "preemptions",
            "batches", "publishes", "relocations", "stale_0", "stale_1"]


def load_gold(path):
    g = {"traj": [], "batch": [], "cmd": [], "after": [], "inst": []}
    for line in open(path):
        if line.startswith("#") or not line.strip():
            continue
        k, *vals = line.split()
        g[k].append([int(x) for x in vals])
    return g


def t3_sim():
    cfg = Config(batch_size=2, n_scenarios=1, k1=1, k2=100, k3=10, k4=50, k5=1, kp=1, M=54, mu=0.3,
                 phi_tp=1.5, phi_wait=0, delta=1000, r=5, q=30, R=20, strategy=7, atw=1, pool_capacity_groups=6)
    s = OracleSim(2, 1, 1, cfg)
    assert s.submit(0, np.array([10, 10, 40, 10, 10, 10]), np.array([8, 9, 6, 7, 2, 2])) == 0
    return s


def test_T3_hand_timeline():
    g = load_gold(GOLD)
    s = t3_sim()
    insts = {}
    for row in g["inst"]:
        insts.setdefault(row[0], []).append(row[2:])
    for w in range(5):
        assert s.step(1) == 0
        m = s.metrics()
        assert [w] + [int(m[IDX[k]]) for k in T3_AFTER] == g["after"][w], f"after window {w}"
        assert s.instances(0).tolist() == insts[w], f"instances after window {w}"
        assert m[IDX["violations"]] == 0 and m[IDX["invalid_snapshots"]] == 0
    assert s.lifecycles(0).tolist() == g["traj"]
    b = s.batches(0).tolist()
    assert [b[0:5], b[5:10], b[10:15]] == g["batch"]
    assert s.commands(0).tolist() == g["cmd"]


def test_eq1_gatekeeping_delays_longer_than_delta():
    """Hand-derived (DESIGN.md §3.1 W2, reading R-EQ1).  I=1, eta=0, B=1, G=1, Delta=100, route delay
    r=250, pull delay q=350, vanilla sync (strategy R|M = 5), tick L = kv + 150.  g0 (p10,T2), g1 (p10,T1).
    w0 t=0: Route(0,j0), arrives 250.  w1, w2: the arrival is pending -> rejected (acc 1 vs 0 counted).
    250: admitted, tick to 410; w3, w4 valid; 571: j0 completes (T=2), reward 591 -> buffer 0 Ready.
    w6 t=600: Consume, publish due 700; j1 ingested, verify(0) over [1,0] empty -> not routed.
    w7 t=700: ps=1; vanilla sync Pulls inst0 (v0 < 1), P=(1,0); j1 routed (v1), arrives 950.
    The pull runs 700-1050: w8, w9, w10 rejected (instance still v0 and pulling; accepting them would
    re-issue the Pull every window).  1050: v=1, held j1 admitted, tick to 1210, complete, reward 1230.
    w11, w12 valid; w13 Consume (1; g1 v1).  Exactly three commands in total."""
    cfg = Config(batch_size=1, n_scenarios=1, k1=1, k2=100, k3=10, k4=50, k5=1, kp=0, M=1000, mu=0.3,
                 phi_tp=5.0, phi_wait=3, delta=100, r=250, q=350, R=20, strategy=5, atw=1, pool_capacity_groups=2)
    s = OracleSim(1, 0, 1, cfg)
    assert s.submit(0, np.array([10, 10]), np.array([2, 1])) == 0
    valid = []
    prev = 0
    for w in range(14):
        assert s.step(1) == 0
        v = int(s.metrics()[IDX["valid_snapshots"]])
        valid.append(v - prev)
        prev = v
    assert valid == [1, 0, 0, 1, 1, 1, 1, 1, 0, 0, 0, 1, 1, 1]
    assert s.commands(0).tolist() == [[0, 1, 0, 0], [7, 3, 0, -1], [7, 1, 0, 1]]
    assert s.batches(0).tolist() == [0, 0, 0, 1, 1, 1]
    m = s.metrics()
    assert m[IDX["violations"]] == 0 and m[IDX["pulls"]] == 1 and m[IDX["routes"]] == 2
    lc = s.lifecycles(0)
    assert lc[:, 12].tolist() == [571, 1210]        # t_complete
    assert lc[:, 8].tolist() == [1, 1]              # each trajectory routed exactly once


def test_cascade_fixpoint_across_earlier_buffers():
    """eta=2, B=1, cu=0.  Reserve a(v1) -> buf 3, c(v1) -> buf 2, p(v0) -> buf 1, x(v0) -> buf 0 (latest
    buffer first).  delete_and_relocate(a) at buf 3: x, p have v + eta = 2 < 3, c qualifies ->
    c moves to 3, hole at 2; then x (buf 0) and p (buf 1) both qualify (2 >= 2): the EARLIEST buffer
    wins -> x moves to 2, hole at 0; nothing earlier -> stop.  2 moves; p stays in buf 1."""
    L = Ledger(eta=2, B=1)
    a, c, p, x = 10, 11, 12, 13
    assert L.reserve(a, 1)[1:] == (3, 0)
    assert L.reserve(c, 1)[1:] == (2, 0)
    assert L.reserve(p, 0)[1:] == (1, 0)
    assert L.reserve(x, 0)[1:] == (0, 0)
    assert L.delete_relocate(a) == 2
    assert L.entries(4) == [[("Empty", -1, -1)], [("Reserved", p, 0)], [("Reserved", x, 0)], [("Reserved", c, 1)]]


def test_cascade_lowest_slot_within_buffer():
    """eta=1, B=2: g0 -> (1,1), g1 -> (1,0), g2 -> (0,1), g3 -> (0,0).  delete_and_relocate(g0): buffer 0
    holds two qualifying Reserved entries (g3 slot 0, g2 slot 1): the LOWEST slot moves -> g3 to (1,1),
    hole (0,0); 1 move (the T3 window-1 ledger step)."""
    L = Ledger(eta=1, B=2)
    for g, where in ((0, (1, 1)), (1, (1, 0)), (2, (0, 1)), (3, (0, 0))):
        assert L.reserve(g, 0)[1:] == where
    assert L.delete_relocate(0) == 1
    assert L.entries(2) == [[("Empty", -1, -1), ("Reserved", 2, 0)], [("Reserved", 1, 0), ("Reserved", 3, 0)]]


def watchdog_sim(wd):
    """Hand-derived: I=1, eta=0, B=2, G=1, one group (p10, T2) in the pool, auto trainer.  Window 0
    routes, decodes and completes it (Occupy buffer 0 slot 0); the batch needs a second group that
    never comes, so from window 1 on nothing progresses and nothing is pending while a live group
    remains: windows 1, 2, 3 are idle and the watchdog (wd = 3) fails the scenario at window 3."""
    cfg = Config(batch_size=2, n_scenarios=1, k1=1, k2=100, k3=10, k4=50, k5=1, kp=0, M=1000, mu=0.3,
                 phi_tp=5.0, phi_wait=3, delta=1000, r=5, q=30, R=20, strategy=7, atw=1, pool_capacity_groups=2,
                 watchdog_windows=wd)
    s = OracleSim(1, 0, 1, cfg)
    assert s.submit(0, np.array([10]), np.array([2])) == 0
    return s


def test_watchdog_deadlock_starved_batch():
    """SPEC S:494 Deadlock ("no events pending but steps unfinished")."""
    s = watchdog_sim(3)
    assert s.step(3) == 0
    assert s.metrics()[IDX["occupied_groups"]] == 1 and s.metrics()[IDX["batches"]] == 0
    assert s.step(1) == -3                                      # SFO_E_STATE in window 3
    m = s.metrics()
    assert m[IDX["poisoned_scenarios"]] == 1 and m[IDX["windows"]] == 4
    off = watchdog_sim(0)                                       # off: idles forever, no error
    assert off.step(50) == 0 and off.metrics()[IDX["poisoned_scenarios"]] == 0


def test_watchdog_never_fires_on_progressing_runs():
    """A watchdog of 1 window leaves every normal simulation alone: each window either progresses or
    has something pending until all work is consumed (transcription configs, full length)."""
    import random
    from tests.test_oracle_fraction import tiny_config
    for seed in range(60):
        rng = random.Random(seed)
        I, eta, G, B, kw, prompt, target = tiny_config(rng)
        # pool = whole batches only (a partial last batch would legitimately starve)
        cfg = Config(batch_size=B, n_scenarios=1, pool_capacity_groups=len(prompt), watchdog_windows=1, **kw)
        s = OracleSim(I, eta, G, cfg)
        assert s.submit(0, prompt, target) == 0
        assert s.step(200) == 0, f"seed {seed}: watchdog fired"
