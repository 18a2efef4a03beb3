"""World-size-2 test of the multi-GPU host logic on CPU (gloo): scenario sharding (bench.shard,
scenario s -> rank s mod W) and the metrics all-reduce (bench.reduce_metrics) must
reproduce, bit for bit, the metrics of one process running every scenario (integer
sums, max time).  The per-rank simulation runs in the oracle here (no GPU on this box);
tests/test_gpu_multirank.py runs the same host logic over NCCL with the CUDA library on 2 GPUs."""
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
    idx = bench.shard(full, rank, world, "weak")
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
    for S, world, mode in ((4096, 8, "weak"), (4096, 8, "strong"), (50, 4, "strong")):
        full = W.preset("C5", n_scenarios=S * (world if mode == "weak" else 1))
        parts = [bench.shard(full, r, world, mode) for r in range(world)]
        assert sorted(k for p in parts for k in p) == list(range(len(full.scenarios)))
        assert all(k % world == r for r, p in enumerate(parts) for k in p)            # s mod W
        assert max(map(len, parts)) - min(map(len, parts)) <= 1
    c3 = W.preset("C3")                                                             # replicas
    assert all(bench.shard(c3, r, 4, "replicas") == [0] for r in range(4))
