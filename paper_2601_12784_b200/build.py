"""Build the sm_100a CUDA library in-tree: paper_2601_12784_b200/libstaleflow.so."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libstaleflow.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -dlcm=cg: global loads are cached in L2 only.  With programmatic dependent launch the window
# kernels run concurrently and hand data over per scenario through release/acquire flags; an
# L1-cached load could return a line filled with pre-release data by another warp of the SM
# (measured: an SF_CHECK build diverged under PDL, bit-exact with L1 bypassed).
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-dlcm=cg", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2"]
if os.environ.get("SF_L1_LOADS") == "1":          # experiment only: L1-cached global loads
    FLAGS = [f for f in FLAGS if f not in ("-Xptxas", "-dlcm=cg")]
FLAGS += [f for f in os.environ.get("SF_NVCC_EXTRA", "").split() if f]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "staleflow.h")]
    return os.path.getmtime(LIB) < max(os.path.getmtime(d) for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, extra=()) -> str:
    """Compile every csrc/*.cu for sm_100a and link `out`.  `extra` nvcc flags (e.g. -DSF_TIMING)
    build an instrumented variant next to the product library (tools/timing_profile.py)."""
    if out == LIB and not extra and not force and not needs_build():
        return LIB
    objs = []
    bdir = os.path.join(HERE, "build" if out == LIB else "build_" + os.path.basename(out).replace(".", "_"))
    os.makedirs(bdir, exist_ok=True)
    procs = []
    for src in sources():
        obj = os.path.join(bdir, os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    for p, cmd in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    tmp = out + f".tmp{os.getpid()}"
    subprocess.run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs], check=True)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    # python -m paper_2601_12784_b200.build [--force] [-v] [--out lib.so -DFLAG ...]
    argv = sys.argv[1:]
    out = LIB
    if "--out" in argv:
        out = os.path.abspath(argv[argv.index("--out") + 1])
    extra = [a for a in argv if a.startswith("-D")]
    print(build(force="--force" in argv, verbose="-v" in argv, out=out, extra=extra))
