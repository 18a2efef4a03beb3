"""TEST INFRASTRUCTURE ONLY: plain reference versions of the host-side tools.

* fit_cost_model -- Eq 7 least squares with iterated regime segmentation,
  solved with numpy.linalg.lstsq.
* plan_comm      -- App A.2 greedy min-accumulated-latency sender choice.
"""
import numpy as np


def fit_cost_model(kv, n_run, latency, max_rounds=50):
    kv, n_run, latency = (np.asarray(a, np.float64) for a in (kv, n_run, latency))
    compute = n_run > np.sort(n_run)[len(n_run) // 2]          # the upper median, as in the library
    x = None
    for _ in range(max_rounds):
        A = np.stack([kv, np.where(compute, 0.0, 1.0), np.where(compute, n_run, 0.0), np.ones_like(kv)], 1)
        if np.linalg.matrix_rank(A) < 4:
            raise ValueError("degenerate")
        x = np.linalg.lstsq(A, latency, rcond=None)[0]
        new = x[2] * n_run > x[1]
        if (new == compute).all():
            break
        compute = new
    return x


def plan_comm(slice_bytes, holds, bandwidth, latency, req_slice, req_receiver):
    n_senders = len(bandwidth)
    acc = [0.0] * n_senders
    out = []
    for k, r in zip(req_slice, req_receiver):
        cands = [s for s in range(n_senders) if holds[s][k]]
        if not cands:
            raise ValueError("uncoverable")
        best = min(cands, key=lambda s: (acc[s], s))
        acc[best] += slice_bytes[k] / bandwidth[best][r] + latency[best][r]
        out.append(best)
    return out, acc
