"""§8(f) f4 host-side tools in the library vs their plain references (oracle/tools.py), pinned to
SPEC's worked examples: cost-coefficient fitting (acceptance 4 S:625) and the App A.2
communication planner (acceptance 9 S:630).  Host code only: runs without a GPU."""
import random

import numpy as np
import pytest

from oracle import tools as OT
from paper_2601_12784_b200 import staleflow as SF

K = np.array([7.28e-8, 1.72e-3, 1.25e-4, 1.07e-2])          # Table 6, seconds


def eq7(kv, n, k=K):
    return k[0] * kv + np.maximum(k[1], k[2] * n) + k[3]


def samples(rng, m=200, noise=0.0, kv_max=1e6):
    """A profiling design spanning both latency regimes: half the samples below the
    k2/k3 = 13.76 crossover (the only ones that identify k2), half above."""
    kv = rng.uniform(0, kv_max, m)
    n = np.where(np.arange(m) % 2 == 0, rng.integers(1, 14, m), rng.integers(14, 300, m)).astype(np.float64)
    lat = eq7(kv, n)
    if noise:
        lat = lat * (1 + noise * rng.standard_normal(m))
    return kv, n, lat


def test_fit_noise_free_round_trip():                    # S:198, acceptance 4
    kv, n, lat = samples(np.random.default_rng(0))
    got = SF.fit_cost_model(kv, n, lat)
    assert np.allclose(got, K, rtol=1e-6, atol=0)
    assert np.allclose(OT.fit_cost_model(kv, n, lat), K, rtol=1e-6, atol=0)


def test_fit_breakpoint():                                # k2/k3 = 13.76
    kv, n, lat = samples(np.random.default_rng(1))
    k = SF.fit_cost_model(kv, n, lat)
    assert abs(k[1] / k[2] - 13.76) < 1e-5


def test_fit_degenerate_single_regime():
    rng = np.random.default_rng(2)
    kv = rng.uniform(0, 1e6, 50)
    n = rng.integers(1, 10, 50).astype(np.float64)        # all memory-bound: k3 unidentifiable
    with pytest.raises(SF.SfError):
        SF.fit_cost_model(kv, n, eq7(kv, n))
    with pytest.raises(ValueError):
        OT.fit_cost_model(kv, n, eq7(kv, n))


def test_fit_one_percent_noise():                         # within 5% over 30 seeded trials
    for seed in range(30):
        kv, n, lat = samples(np.random.default_rng(100 + seed), m=1000, noise=0.01, kv_max=2e5)
        got = SF.fit_cost_model(kv, n, lat)
        assert np.all(np.abs(got / K - 1) < 0.05), (seed, got)
        assert np.allclose(got, OT.fit_cost_model(kv, n, lat), rtol=1e-6)


def plan(sizes, holds, bw, lat, reqs):
    rs = [k for k, _ in reqs]
    rr = [r for _, r in reqs]
    a, acc = SF.plan_comm(sizes, holds, bw, lat, rs, rr)
    b, acc2 = OT.plan_comm(sizes, holds, bw, lat, rs, rr)
    assert list(a) == b and np.allclose(acc, acc2)
    return list(a), list(acc)


def test_plan_equal_slices_two_senders():
    out, acc = plan([1.0] * 4, [[1] * 4, [1] * 4], [[1.0], [1.0]], [[0.0], [0.0]], [(k, 0) for k in range(4)])
    assert out.count(0) == 2 and out.count(1) == 2


def test_plan_single_sender():
    out, _ = plan([1.0, 2.0], [[1, 1]], [[1.0]], [[0.0]], [(0, 0), (1, 0)])
    assert out == [0, 0]


def test_plan_greedy_balances_4321():                     # loads 4+1 vs 3+2
    out, acc = plan([4.0, 3.0, 2.0, 1.0], [[1] * 4, [1] * 4], [[1.0], [1.0]], [[0.0], [0.0]],
                    [(k, 0) for k in range(4)])
    assert sorted(acc) == [5.0, 5.0]


def test_plan_uncoverable():
    with pytest.raises(SF.SfError):
        SF.plan_comm([1.0], [[0]], [[1.0]], [[0.0]], [0], [0])


def test_plan_coverage_and_greedy_bound():                # acceptance 9
    rng = random.Random(9)
    for _ in range(100):
        n_sl, n_s, n_r = rng.randint(1, 12), rng.randint(1, 5), rng.randint(1, 4)
        sizes = [rng.uniform(1, 100) for _ in range(n_sl)]
        holds = [[0] * n_sl for _ in range(n_s)]
        for k in range(n_sl):
            for s in rng.sample(range(n_s), rng.randint(1, n_s)):
                holds[s][k] = 1
        bw = [[1.0] * n_r for _ in range(n_s)]
        lat = [[0.0] * n_r for _ in range(n_s)]
        reqs = [(k, r) for k in range(n_sl) for r in range(n_r)]
        out, acc = plan(sizes, holds, bw, lat, reqs)
        assert len(out) == len(reqs) and all(holds[s][k] for s, (k, _) in zip(out, reqs))
        # round-robin over holders for comparison
        rr_acc, turn = [0.0] * n_s, 0
        for k, r in reqs:
            hs = [s for s in range(n_s) if holds[s][k]]
            s = hs[turn % len(hs)]
            turn += 1
            rr_acc[s] += sizes[k]
        if all(sum(h) == n_sl for h in holds):            # identical senders: greedy is LPT-like
            assert max(acc) <= max(rr_acc) + 1e-9


# ------------------------------------------------------------------ PS read-write lock
def lock(kind, t, d, pv, v0=0):
    a = [np.asarray(x).tolist() for x in SF.ps_lock_sim(kind, t, d, pv, v0)]
    b = [list(x) for x in OT.ps_lock_sim(kind, t, d, pv, v0)]
    assert a == b, (a, b)
    return a


def test_push_no_readers():
    s, e, v, st = lock([1], [0], [10], [1])
    assert (s, e, v, st) == ([0], [10], [1], [0])
    s, e, v, st = lock([1, 0], [0, 10], [10, 1], [1, 0])  # a later Pull sees version 1
    assert v[1] == 1


def test_push_waits_for_active_pulls():                  # write begins after both complete
    s, e, v, st = lock([0, 0, 1], [0, 1, 2], [5, 8, 3], [0, 0, 1])
    assert s[2] == max(e[0], e[1]) == 9 and e[2] == 12


def test_push_version_skip():
    s, e, v, st = lock([1, 1], [0, 1], [1, 1], [1, 3])
    assert st == [0, -2] and s[1] == -1


def test_pulls_share_the_lock():                         # both complete after their own duration
    s, e, v, st = lock([0, 0], [0, 0], [4, 7], [0, 0], v0=5)
    assert s == [0, 0] and e == [4, 7] and v == [5, 5]


def test_pull_during_push_gets_new_version():
    s, e, v, st = lock([1, 0], [0, 2], [10, 3], [1, 0])
    assert s[1] == 10 and v[1] == 1


def test_writer_preference():                            # a waiting Push blocks new Pulls
    s, e, v, st = lock([0, 1, 0], [0, 1, 2], [10, 5, 1], [0, 1, 0])
    assert s[1] == 10 and s[2] == 15 and v[2] == 1


@pytest.mark.parametrize("seed", range(30))
def test_lock_fuzz_safety_and_parity(seed):
    """Library == reference on random traces; lock safety (no Push interval overlaps another
    interval), writer preference, version monotonicity."""
    rng = random.Random(4000 + seed)
    n = rng.randint(1, 60)
    kind = [1 if rng.random() < 0.3 else 0 for _ in range(n)]
    t = sorted(rng.randint(0, 200) for _ in range(n)) if seed % 2 else [rng.randint(0, 200) for _ in range(n)]
    d = [rng.randint(0, 30) for _ in range(n)]
    pv, nxt = [], 1
    for k in kind:
        if k == 1 and rng.random() < 0.9:
            pv.append(nxt)
            nxt += 1
        else:
            pv.append(rng.randint(0, 9) if k == 1 else 0)
    s, e, v, st = lock(kind, t, d, pv)
    ok = [k for k in range(n) if st[k] == 0]
    for a in ok:
        assert s[a] >= t[a]
        for b in ok:
            if a < b and (kind[a] == 1 or kind[b] == 1) and d[a] > 0 and d[b] > 0:
                assert not (s[a] < e[b] and s[b] < e[a]), (a, b)
    order = lambda k: (t[k], k)
    for w in ok:
        if kind[w] != 1:
            continue
        for r in ok:
            if kind[r] == 0 and order(w) < order(r) and s[r] < s[w]:
                assert s[r] < t[w] or (s[r] == t[w] and order(r) < order(w)), (w, r)   # granted before w arrived
    pulls = sorted((s[k], v[k]) for k in ok if kind[k] == 0)
    assert all(pulls[i][1] <= pulls[i + 1][1] for i in range(len(pulls) - 1))
