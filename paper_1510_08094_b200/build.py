"""Build the sm_100a shared library ``libsk_poisson.so`` in-tree with nvcc.

No JIT cache, no torch extension machinery: the built ``.so`` sits next to
this file, so it travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsk_poisson.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", f"-I{INCLUDE}"]
# coeff_kernels.cu and assemble_kernels.cu reproduce the reference's IEEE operation order: no FMA
# contraction anywhere in those translation units.
UNITS = [
    ("grid_kernels.cu", []),
    ("grid_large.cu", []),
    ("theta_sym.cu", []),
    ("theta_mp.cu", []),
    ("lambda_duo.cu", []),
    ("coeff_kernels.cu", ["--fmad=false"]),
    ("assemble_kernels.cu", ["--fmad=false"]),
    ("ge_kernels.cu", ["--fmad=false"]),
    ("transforms.cu", []),
    ("sk_poisson.cu", []),
]
HEADERS = ["sk_internal.h", "params.h", "fft_dev.cuh", "block_ops.cuh", "tma.cuh", "theta_common.cuh"]


def nvcc() -> str:
    exe = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(exe):
        raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libsk_poisson.so")
    return exe


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "sk_poisson.h"), __file__]
    objs = []
    jobs = []
    for src, extra in UNITS:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([nvcc(), *ARCH, *COMMON, *extra, "-c", s, "-o", o])
    # translation units compile side by side (one nvcc process each)
    procs = []
    for cmd in jobs:
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd)))
    failed = [cmd for cmd, pr in procs if pr.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    if force or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
