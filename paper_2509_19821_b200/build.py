"""Builds the engine library in-tree: paper_2509_19821_b200/libgmpea_b200.so.

One nvcc invocation for sm_100a (B200); no torch extension machinery, the
library is a plain C ABI (include/gmpea_b200.h).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libgmpea_b200.so")
SOURCES = [os.path.join(HERE, "csrc", "engine.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in
                  ("common.cuh", "kernels.cuh", "problems.cuh", "topology.cuh", "metrics.cuh", "fronts.cuh", "baselines.cuh")] + [
    os.path.join(ROOT, "include", "gmpea_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fno-builtin-sin", "-Xcompiler", "-fno-builtin-cos",
]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in DEPS if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-o", LIB + ".tmp", *SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
