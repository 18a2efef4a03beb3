"""Helpers that drive the oracle and the CUDA library with identical inputs and diff them.

Test infrastructure: imports the oracle (tests are allowed to) and the product binding.
"""
from __future__ import annotations

import numpy as np

from oracle.oracle import Config, OracleSim, METRIC_NAMES
from paper_2601_12784_b200 import workload as W


def make_pair(p: W.Preset, scen_idx=None, cmdlog=200_000, pool_capacity=None):
    from paper_2601_12784_b200.staleflow import StaleFlow
    kw = {}
    if pool_capacity is not None:
        kw["pool_capacity_groups"] = pool_capacity
        p.pool_capacity = pool_capacity  # type: ignore[attr-defined]
    o = OracleSim.from_preset(p, scen_idx)
    g = StaleFlow.from_preset(p, scen_idx, command_log_capacity=cmdlog, **kw)
    return o, g


def submit_both(o, g, p: W.Preset, scen_idx=None, n_groups=None):
    idx = list(range(len(p.scenarios))) if scen_idx is None else list(scen_idx)
    ng = p.pool_groups if n_groups is None else n_groups
    prs, tgs = [], []
    for a, k in enumerate(idx):
        pr, tg = W.draw_lengths(p, k, ng)
        assert o.submit(a, pr, tg) == 0
        prs.append(pr)
        tgs.append(tg)
    rc = g.submit_many(np.arange(len(idx)), np.full(len(idx), ng), np.concatenate(prs), np.concatenate(tgs))
    assert rc == 0
    if getattr(p, "filter_prob", 0.0) > 0:
        for a, k in enumerate(idx):
            f = W.draw_filter_flags(p, k, ng)
            assert o.mark_filtered(a, 0, f) == 0
            g.mark_filtered(a, 0, f)


def first_cmd_divergence(co, cg):
    n = min(len(co), len(cg))
    for k in range(n):
        if not (co[k] == cg[k]).all():
            return k, co[max(0, k - 3): k + 3].tolist(), cg[max(0, k - 3): k + 3].tolist()
    if len(co) != len(cg):
        return n, co[n: n + 3].tolist(), cg[n: n + 3].tolist()
    return None


def compare(o, g, scen_list, where="", check_cmds=True):
    """Element-by-element comparison of every observable of the listed scenarios."""
    for a in scen_list:
        mo, mg = o.metrics(a), g.metrics(a)
        if check_cmds:
            co, cg = o.commands(a), g.commands(a)
            d = first_cmd_divergence(co, cg)
            assert d is None, f"{where} scen {a}: first command divergence at record {d[0]}: oracle {d[1]} gpu {d[2]}"
        bad = [(METRIC_NAMES[k], int(mo[k]), int(mg[k])) for k in range(32) if mo[k] != mg[k]]
        assert not bad, f"{where} scen {a}: metrics differ {bad}"
        lo, lg = o.lifecycles(a), g.lifecycles(a)
        assert lo.shape == lg.shape
        diff = np.argwhere(lo != lg)
        assert len(diff) == 0, f"{where} scen {a}: lifecycle differs at {diff[:5].tolist()}: " \
                               f"oracle {lo[diff[0][0]].tolist()} gpu {lg[diff[0][0]].tolist()}"
        assert (o.batches(a) == g.batches(a)).all(), f"{where} scen {a}: batches differ"
        io, ig = o.instances(a), g.instances(a)
        assert (io == ig).all(), f"{where} scen {a}: instance state differs\n{io}\n{ig}"


def run_lockstep(o, g, scen_list, windows, every=1, check_cmds=True, threads=8):
    done = 0
    while done < windows:
        k = min(every, windows - done)
        assert o.step(k, threads) == 0, "oracle step failed"
        g.step(k)
        done += k
        compare(o, g, scen_list, where=f"after window {done}", check_cmds=check_cmds)
