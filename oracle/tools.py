"""TEST INFRASTRUCTURE ONLY: plain reference versions of the host-side tools.

* fit_cost_model -- Eq 7 least squares with iterated regime segmentation,
  solved with numpy.linalg.lstsq.
* plan_comm      -- App A.2 greedy min-accumulated-latency sender choice.
"""
import numpy as np


def fit_cost_model(kv, n_run, latency, max_rounds=50):
    kv, n_run, latency = (np.asarray(a, np.float64) for a in (kv, n_run, latency))
    compute = n_run > np.median(n_run)                          # initial split (reading R-FIT)
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


def ps_lock_sim(kind, t_issue, duration, push_version, v0=0):
    """Parameter-server Push/Pull under a read-write lock, writer
    preference: a Pull is granted only if no Push is active or waiting; a Push only if
    nothing is active; on a release, a waiting Push goes first, else every waiting Pull.
    Requests are handled in (issue time, index) order; at equal times releases come first.
    A Pull delivers the version committed when its read starts; a Push commits its version when
    its write ends.  A Push whose version is not the last accepted version + 1 is rejected
    (VersionSkip, status -2) and takes no lock.  Returns (start, end, version, status) lists."""
    n = len(kind)
    start, end, ver, status = [-1] * n, [-1] * n, [-1] * n, [0] * n
    order = sorted(range(n), key=lambda k: (t_issue[k], k))
    accepted = v0
    committed = v0
    readers = []               # end times of active reads
    writer = None              # (end time, version) of the active write
    waiting = []               # request indices, arrival order
    releases = []              # pending release times (reads and the write)

    def grant(k, now):
        nonlocal writer
        start[k], end[k] = now, now + duration[k]
        if kind[k] == 1:
            writer = (end[k], push_version[k])
            ver[k] = push_version[k]
        else:
            readers.append(end[k])
            ver[k] = committed
        releases.append(end[k])

    def schedule(now):
        # after a change at `now`: a waiting Push first, else every waiting Pull
        if writer is not None:
            return
        w = [k for k in waiting if kind[k] == 1]
        if w:
            if not readers:
                waiting.remove(w[0])
                grant(w[0], now)
            return
        for k in list(waiting):
            waiting.remove(k)
            grant(k, now)

    def release_until(t):
        nonlocal writer, committed
        while releases and min(releases) <= t:
            now = min(releases)
            releases.remove(now)
            if writer is not None and writer[0] == now:
                committed = writer[1]
                writer = None
            elif now in readers:
                readers.remove(now)
            schedule(now)

    for k in order:
        now = t_issue[k]
        release_until(now)
        if kind[k] == 1:
            if push_version[k] != accepted + 1:
                status[k] = -2
                continue
            accepted = push_version[k]
            if writer is None and not readers and not any(kind[x] == 1 for x in waiting):
                grant(k, now)
            else:
                waiting.append(k)
        else:
            if writer is None and not any(kind[x] == 1 for x in waiting):
                grant(k, now)
            else:
                waiting.append(k)
    release_until(float("inf"))
    return start, end, ver, status
