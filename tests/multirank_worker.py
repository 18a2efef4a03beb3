"""Worker for tests/test_gpu_multirank.py (launched by torchrun, one process per GPU, NCCL).

Runs the C5 family's shard s mod W on this rank's GPU through libstaleflow.so, then (NCCL over
NVLink) all-reduces the metric vector exactly as bench.py does and sums the per-scenario rows
[32 metrics + a 63-bit lifecycle hash] into one table (each row has exactly one owner).  Rank 0
writes the result as JSON."""
import argparse
import hashlib
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2601_12784_b200 import workload as W  # noqa: E402
from paper_2601_12784_b200.staleflow import StaleFlow  # noqa: E402


def lifecycle_hash(lc: np.ndarray) -> int:
    return int.from_bytes(hashlib.blake2b(np.ascontiguousarray(lc).tobytes(), digest_size=8).digest(), "little") >> 1


def run(full, idx, windows, device):
    p = W.preset_scenario_slice(full, idx)
    g = StaleFlow.from_preset(p, device=device)
    prs, tgs = zip(*[W.draw_lengths(full, k, full.pool_groups) for k in idx])
    assert g.submit_many(np.arange(len(idx)), np.full(len(idx), full.pool_groups), np.concatenate(prs),
                         np.concatenate(tgs)) == 0
    for w0 in range(0, windows, full.auto_train_windows):
        g.step(min(full.auto_train_windows, windows - w0))
    rows = np.zeros((len(full.scenarios), 33), np.int64)
    am = g.all_metrics()
    for a, k in enumerate(idx):
        rows[k, :32] = am[a]
        rows[k, 32] = lifecycle_hash(g.lifecycles(a))
    return g.metrics(), rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenarios", type=int, default=256)
    ap.add_argument("--windows", type=int, default=300)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    full = W.preset("C5", n_scenarios=a.scenarios)
    idx = bench.shard(full, rank, world, "strong")
    m, rows = run(full, idx, a.windows, local)
    vec = torch.tensor(m, dtype=torch.int64, device="cuda")
    bench.reduce_metrics(vec, world, dist)                 # the NCCL all-reduce of the metric vector
    tab = torch.tensor(rows, device="cuda")
    dist.all_reduce(tab, op=dist.ReduceOp.SUM)             # each row has exactly one owner
    if rank == 0:
        json.dump({"world": world, "backend": dist.get_backend(), "nccl": ".".join(map(str, torch.cuda.nccl.version())),
                   "metrics": vec.cpu().tolist(), "rows": tab.cpu().tolist()}, open(a.out, "w"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
