"""Pins for the oracle's staleness ledger (PAPER §4.2).

Worked examples are SPEC.md's (tagged PAPER/DERIVED there); T2 is
the hand example of SURVEY §8(c); placements are checked against brute force
over every slot (acceptance 2); fuzz checks the invariants of
S:116-122.
"""
import random

import pytest

from oracle.oracle import Ledger


def fill(L, b, n, st="R", v=None, g0=1000):
    """Fill n slots of buffer b via the public ops (reserve with v=b-eta..b window)."""
    out = []
    for k in range(n):
        vv = b if v is None else v
        rc, bb, ss = L.reserve(g0 + k, vv)
        assert rc == 0
        out.append((g0 + k, bb, ss))
    return out


# ---------------------------------------------------------------- verify
def test_verify_empty_ledger_true():                      # S:57 [TRIVIAL]
    assert Ledger(1, 4).verify(0)


def test_verify_full_buffers_false():                     # S:58 [DERIVED]
    L = Ledger(1, 2)
    for g in range(4):                                    # 2 buffers x 2 slots, v=0 -> buffers 1,1,0,0
        assert L.reserve(g, 0)[0] == 0
    assert not L.verify(0)


def test_verify_newer_buffer_open():                      # S:59 [DERIVED]
    L = Ledger(1, 2)
    for g in range(4):
        L.reserve(g, 0)
    assert L.verify(1)                                    # buffer 2 = v + eta is empty


# ---------------------------------------------------------------- reserve
def test_reserve_backward_scan_latest():                  # S:66 [PAPER] "backward scan"
    L = Ledger(1, 3)
    rc, b, s = L.reserve(7, 0)
    assert (rc, b, s) == (0, 1, 2)                        # latest buffer, highest slot


def test_reserve_eta0_single_buffer():
    L = Ledger(0, 2)
    rc, b, _ = L.reserve(1, 3)
    assert (rc, b) == (0, 3)


def test_reserve_skips_full_buffer():
    L = Ledger(2, 1)
    assert L.reserve(1, 0)[1] == 2                        # buffer 2 now full
    assert L.reserve(2, 0)[1] == 1                        # -> buffer 1


def test_reserve_no_capacity_and_duplicate():             # S:64 errors
    L = Ledger(0, 1)
    assert L.reserve(1, 0)[0] == 0
    assert L.reserve(2, 0)[0] != 0                        # NoCapacity
    assert L.reserve(1, 0)[0] != 0                        # DuplicateKey


# ---------------------------------------------------------------- mark_complete / relocate
def test_occupy_earliest():                               # S:75 [PAPER] "earliest available"
    L = Ledger(1, 1)
    assert L.reserve(5, 0)[1] == 1
    rc, b, s = L.complete(5, 0)
    assert (rc, b, s) == (0, 0, 0)
    assert L.get(1, 0)[0] == "Empty"


def test_delete_no_other_reserved():                      # S:84 [TRIVIAL]
    L = Ledger(1, 2)
    L.reserve(1, 0)
    assert L.delete_relocate(1) == 0
    assert all(e[0] == "Empty" for row in L.entries(2) for e in row)


def test_delete_moves_earlier_reserved():                 # S:85 [DERIVED]
    L = Ledger(1, 1)
    assert L.reserve(10, 0)[1] == 1                       # A in buffer 1
    assert L.reserve(11, 0)[1] == 0                       # B (V_B=0) in buffer 0
    assert L.delete_relocate(10) == 1
    assert L.get(1, 0) == ("Reserved", 11, 0)
    assert L.get(0, 0)[0] == "Empty"


def test_delete_respects_bound():                         # S:86 [DERIVED]
    L = Ledger(1, 1)
    # B with version 0 in buffer 0; A with version 1 in buffer 2 (0 + 1 < 2: B may not move).
    assert L.reserve(11, 0)[1] == 1
    assert L.reserve(12, 0)[1] == 0
    assert L.reserve(10, 1)[1] == 2
    assert L.delete_relocate(10) == 0
    assert L.get(0, 0) == ("Reserved", 12, 0)
    assert L.get(1, 0) == ("Reserved", 11, 0)


# ---------------------------------------------------------------- consume / state
def test_consume_exact_batch():
    L = Ledger(0, 4)
    for g in range(4):
        L.reserve(g, 0)
    for g in range(4):
        L.complete(g, 0)
    rc, gs, vs = L.consume()
    assert rc == 0 and sorted(gs.tolist()) == [0, 1, 2, 3] and L.cu == 1


def test_consume_stuck_not_ready():                       # S:94 [PAPER] "Stuck"
    L = Ledger(0, 2)
    L.reserve(0, 0)
    L.reserve(1, 0)
    L.complete(0, 0)
    assert L.state(0) == "Stuck"
    assert L.consume()[0] == 1                            # SF_NOT_READY


def test_states():
    L = Ledger(0, 2)
    L.reserve(0, 0)
    assert L.state(0) == "Waiting"
    L.reserve(1, 0)
    assert L.state(0) == "Stuck"
    L.complete(0, 0)
    L.complete(1, 0)
    assert L.state(0) == "Ready"


# ---------------------------------------------------------------- hand example T2
def test_T2_g0_first():
    L = Ledger(1, 1)
    assert L.reserve(0, 0)[1] == 1                        # backward scan -> buffer 1
    assert L.reserve(1, 0)[1] == 0
    assert not L.verify(0)
    assert L.complete(0, 0)[1] == 0                       # cascade moves g1 0 -> 1; g0 occupies 0
    assert L.get(1, 0) == ("Reserved", 1, 0)
    assert L.state(0) == "Ready"


def test_T2_g1_first():
    L = Ledger(1, 1)
    L.reserve(0, 0)
    L.reserve(1, 0)
    assert L.complete(1, 0)[1] == 0                       # delete at 0, no cascade, occupy 0
    assert L.complete(0, 0)[1] == 1                       # buffer 0 occupied (immovable) -> 1
    assert L.state(0) == "Ready" and L.state(1) == "Ready"


# ---------------------------------------------------------------- brute force
def _random_state(rng, eta, B):
    L = Ledger(eta, B)
    live = {}
    g = 0
    cu = 0
    for _ in range(rng.randint(0, 4 * (eta + 1) * B)):
        op = rng.random()
        if op < 0.55:
            v = rng.randint(max(0, cu - eta), cu)
            if L.verify(v):
                rc, b, s = L.reserve(g, v)
                assert rc == 0
                live[g] = v
                g += 1
        elif op < 0.9 and live:
            gg = rng.choice(sorted(live))
            st = None
            for b in range(cu, cu + eta + 2):
                for s in range(B):
                    e = L.get(b, s)
                    if e[1] == gg and e[0] == "Reserved":
                        st = e
            if st is not None:
                L.complete(gg, live[gg])
                del live[gg]
        else:
            rc, gs, vs = L.consume()
            if rc == 0:
                cu += 1
    return L, g, cu


def _snapshot(L, cu, eta, B):
    return {(b, s): L.get(b, s) for b in range(cu, cu + eta + 3) for s in range(B)}


@pytest.mark.parametrize("seed", range(10))
def test_placements_brute_force(seed):
    rng = random.Random(seed)
    checked = 0
    for _ in range(60):
        eta, B = rng.randint(0, 3), rng.randint(1, 4)
        L, gnext, cu = _random_state(rng, eta, B)
        snap = _snapshot(L, cu, eta, B)
        for v in range(max(0, cu - eta), cu + 1):
            feas = [(b, s) for (b, s), e in snap.items() if e[0] == "Empty" and max(v, cu) <= b <= v + eta]
            assert L.verify(v) == bool(feas)
            if feas:
                L2 = L.clone()
                rc, b, s = L2.reserve(gnext, v)
                assert rc == 0 and (b, s) == max(feas)           # latest buffer, highest slot
        feas_occ = [(b, s) for (b, s), e in snap.items() if e[0] == "Empty"]
        L3 = L.clone()
        rc, b, s = L3.occupy(gnext + 1, cu)
        assert rc == 0 and (b, s) == min(feas_occ)               # earliest buffer, lowest slot
        checked += 1
    assert checked == 60


# ---------------------------------------------------------------- fuzz invariants
@pytest.mark.parametrize("seed", range(20))
def test_ledger_fuzz_invariants(seed):
    rng = random.Random(1000 + seed)
    for _ in range(50):
        eta, B = rng.randint(0, 4), rng.randint(1, 8)
        L = Ledger(eta, B)
        cu, g = 0, 0
        live = {}
        consumed = []
        for _ in range(rng.randint(10, 120)):
            r = rng.random()
            if r < 0.5:
                v = rng.randint(max(0, cu - eta), cu)
                if L.verify(v):
                    assert L.reserve(g, v)[0] == 0
                    live[g] = v
                    g += 1
            elif r < 0.85 and live:
                gg = rng.choice(sorted(live))
                before = _snapshot(L, cu, eta, B)
                L.delete_relocate(gg)
                after = _snapshot(L, cu, eta, B)
                # relocation never moves an Occupied entry and never moves an entry later->earlier
                for k, e in before.items():
                    if e[0] == "Occupied":
                        assert after[k] == e
                pos_b = {e[1]: k[0] for k, e in before.items() if e[0] == "Reserved"}
                pos_a = {e[1]: k[0] for k, e in after.items() if e[0] == "Reserved"}
                assert set(pos_a) == set(pos_b) - {gg}
                for key in pos_a:
                    assert pos_a[key] >= pos_b[key]
                rc, b, s = L.occupy(gg, live.pop(gg))
                assert rc == 0
            else:
                rc, gs, vs = L.consume()
                if rc == 0:
                    consumed.append(cu)
                    for v in vs:
                        assert 0 <= cu - v <= eta                  # staleness safety at consume
                    cu += 1
            # staleness safety + in-flight bound after every op
            tracked = 0
            for (b, s), e in _snapshot(L, cu, eta, B).items():
                if e[0] != "Empty":
                    tracked += 1
                    assert e[2] <= b <= e[2] + eta
            assert tracked <= (eta + 1) * B
        assert consumed == list(range(len(consumed)))              # consume order 0,1,2,...
