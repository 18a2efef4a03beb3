"""The library's branch-free division (sf_internal.cuh div_int_rn) equals __ddiv_rn bit for bit on
its operand domain (2^30 sampled integer pairs, denominators up to 2^62, incl. powers of two and
small numerators): the
cost-model decisions stay identical to the oracle's correctly rounded fp64 division."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_div_int_rn_matches_ddiv_rn(tmp_path):
    exe = str(tmp_path / "div_check")
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "-o", exe, os.path.join(HERE, "cuda", "div_check.cu")], check=True)
    out = subprocess.run([exe, str(1 << 30)], capture_output=True, text=True, check=True).stdout.split()
    assert int(out[0]) == 1 << 30 and int(out[1]) == 0, out
