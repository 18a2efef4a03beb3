"""Two ranks over NCCL with the CUDA library: the C5 family split s mod W over
2 GPUs (torchrun, one process per GPU) must give, bit for bit, the all-reduced metric vector and
every scenario's metric row and lifecycle hash of one GPU running all scenarios (DESIGN.md §12:
integer sums, max time).  Needs 2 GPUs (gpurun --gpus 2); skipped on one."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_gpus_nccl_equal_one_gpu(tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    out = str(tmp_path / "two.json")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "multirank_worker.py"),
           "--scenarios", "256", "--windows", "300", "--out", out]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    two = json.load(open(out))
    assert two["world"] == 2 and two["backend"] == "nccl"
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from multirank_worker import run
    from paper_2601_12784_b200 import workload as W
    full = W.preset("C5", n_scenarios=256)
    m1, rows1 = run(full, list(range(256)), 300, 0)
    rows2 = np.array(two["rows"], np.int64)
    assert (rows2 == rows1).all(), f"scenario rows differ: {np.nonzero((rows2 != rows1).any(1))[0][:10]}"
    assert (np.array(two["metrics"], np.int64) == m1).all()
    assert m1[9] > 0 and m1[7] > 0                          # batches and pulls happened
