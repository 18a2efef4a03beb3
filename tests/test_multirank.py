"""World-size-2 test of the multi-GPU host logic on CPU (gloo): scenario sharding (bench.shard,
weak scaling) and the metrics all-reduce (bench.reduce_metrics) must reproduce, bit for bit,
the metrics of one process running every scenario (integer sums, max time).
The per-rank simulation runs in the oracle here (no GPU on this box); on a GPU box bench.py
runs the same host logic over NCCL with the CUDA library."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from oracle.oracle import OracleSim
from paper_2601_12784_b200 import workload as W

S_PER_RANK = 6
WINDOWS = 40


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_rank(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = W.preset("C5", n_scenarios=S_PER_RANK * world)
    idx = bench.shard(S_PER_RANK, rank)
    o = OracleSim.from_preset(full, idx)
    for a, k in enumerate(idx):
        pr, tg = W.draw_lengths(full, k, full.pool_groups)
        assert o.submit(a, pr, tg) == 0
    assert o.step(WINDOWS, 2) == 0
    vec = torch.tensor(o.metrics(), dtype=torch.int64)
    bench.reduce_metrics(vec, world, dist)
    if rank == 0:
        np.save(out_path, vec.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_metrics_equal_single_process(tmp_path):
    world = 2
    out = str(tmp_path / "m.npy")
    mp.spawn(_run_rank, args=(world, _free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    full = W.preset("C5", n_scenarios=S_PER_RANK * world)
    o = OracleSim.from_preset(full)
    for k in range(S_PER_RANK * world):
        pr, tg = W.draw_lengths(full, k, full.pool_groups)
        assert o.submit(k, pr, tg) == 0
    assert o.step(WINDOWS, 4) == 0
    ref = o.metrics()
    assert (got == ref).all(), f"slots differ: {np.nonzero(got != ref)}"
    assert ref[2] > 0


def test_shards_partition_the_family():
    S, world = 4096, 8
    seen = sorted(k for r in range(world) for k in bench.shard(S, r))
    assert seen == list(range(S * world))
