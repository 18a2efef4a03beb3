"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/staleflow.h
declares; the Python binding names the same calls.  No compute calls (no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "staleflow.h")


def declared_functions():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sf_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2601_12784_b200 import build as B
    return B.build()


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for must in ("sf_create", "sf_submit_prompts", "sf_step", "sf_publish_params", "sf_collect_batch"):
        assert must in names


def test_library_exports_every_declared_symbol(lib_path):
    lib = C.CDLL(lib_path)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sf_[a-z_]+)", out))
    assert set(declared_functions()) <= exported


def test_sm100a_cubin_inside(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_binding_uses_the_same_names():
    from paper_2601_12784_b200 import staleflow
    assert set(staleflow.EXPORTS) == set(declared_functions())


def test_binding_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2601_12784_b200.staleflow import SfError, StaleFlow
    with pytest.raises(SfError):
        StaleFlow(4, 1, 8, 64)


def test_oracle_is_independent_of_the_product():
    """The oracle tree includes/imports nothing of the CUDA product and vice versa; the only shared
    module is the seeded input generator paper_2601_12784_b200/workload.py."""
    bad_in_oracle = ("staleflow.h", "libstaleflow", "csrc", "paper_2601_12784_b200.staleflow",
                     "paper_2601_12784_b200 import staleflow")
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".cpp", ".h")):
            src = open(os.path.join(ROOT, "oracle", f)).read()
            for b in bad_in_oracle:
                assert b not in src, f"oracle/{f} references {b}"
    bad_in_product = ("import oracle", "from oracle", "libsforacle", "sf_oracle", "sfo_")
    for dp, _, fs in os.walk(os.path.join(ROOT, "paper_2601_12784_b200")):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dp, f)).read()
                for b in bad_in_product:
                    assert b not in src, f"{f} references {b}"


def test_group_division_multiply_shift_exact():
    """grp_of() (sf_internal.cuh): id / G == (id * ceil(2^40/G)) >> 40 in 64-bit arithmetic for every id
    sf_create accepts: id < 2^27, id * m < 2^64 (G = 1 with 2^24 trajectories would wrap)."""
    import random
    rng = random.Random(7)
    for G in list(range(1, 65)) + [96, 100, 1000, 4095, 4096]:
        m = ((1 << 40) + G - 1) // G
        top = min(1 << 27, ((1 << 64) - 1) // m + 1)         # sf_create: pool_traj - 1 < top
        ids = list(range(5000)) + [rng.randrange(top) for _ in range(5000)] + [top - 1 - k for k in range(500)]
        assert all((i * m) < (1 << 64) and ((i * m) & ((1 << 64) - 1)) >> 40 == i // G for i in ids), G
    assert (((1 << 24) * (1 << 40)) & ((1 << 64) - 1)) >> 40 == 0   # the wrap sf_create now rejects (G = 1)


def test_window_kernels_use_strong_gpu_loads_only():
    """The window kernels hand data over per scenario through release/acquire flags while other
    scenarios' kernels run on the same SMs (programmatic dependent launch).  The
    library is built so that every global load is a .STRONG.GPU load served by L2 (-dlcm=cg); a
    build without it (weak, L1-cached LDG.E) fails here rather than running with L1 lines that may
    hold pre-release data."""
    import shutil
    import subprocess
    from paper_2601_12784_b200 import build as B
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    B.build()
    sass = subprocess.run([cuobjdump, "-sass", B.LIB], capture_output=True, text=True, check=True).stdout
    weak, func = {}, None
    for line in sass.splitlines():
        if "Function :" in line:
            func = line.split("Function :")[1].strip()
        elif func and "LDG." in line and ".STRONG.GPU" not in line:
            weak[func] = weak.get(func, 0) + 1
    window = [f for f in weak if any(k in f for k in ("k_begin_coord", "k_advance", "k_ledger", "k_window"))]
    assert not window, f"weak (L1-cached) global loads in window kernels: {[(f, weak[f]) for f in window]}"
