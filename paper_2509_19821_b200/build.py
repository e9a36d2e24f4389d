"""Builds the engine library in-tree: paper_2509_19821_b200/libgmpea_b200.so.

Every translation unit of csrc/ is compiled for sm_100a (B200) in parallel
(the generation kernels are instantiated per problem family, vary_<family>.cu)
and linked into one shared library with a plain C ABI (include/gmpea_b200.h);
no torch extension machinery.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgmpea_b200.so")
OBJ = os.path.join(ROOT, "build", "obj")
SOURCES = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
HEADERS = sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "gmpea_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fno-builtin-sin", "-Xcompiler", "-fno-builtin-cos",
]
LINK_FLAGS = ["-shared", "-ldl"]


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _obj(src: str) -> str:
    return os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def up_to_date() -> bool:
    return not _stale(LIB, SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, jobs: int = 0) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    # every header may feed every TU: a header change rebuilds all objects
    todo = [s for s in SOURCES if force or _stale(_obj(s), [s] + HEADERS)]

    extra = os.environ.get("GMPEA_NVCC_EXTRA", "").split()  # A/B variants (-DGMPEA_...)

    def compile_one(src):
        cmd = [nvcc(), *NVCC_FLAGS, *extra, "-c", "-o", _obj(src) + ".tmp", src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr, flush=True)
        subprocess.run(cmd, check=True)
        os.replace(_obj(src) + ".tmp", _obj(src))

    # the heaviest TUs first
    todo.sort(key=lambda s: -os.path.getsize(s) if not os.path.basename(s).startswith("vary_") else -10**9)
    with cf.ThreadPoolExecutor(max_workers=jobs or max(1, os.cpu_count() or 1)) as ex:
        for f in [ex.submit(compile_one, s) for s in todo]:
            f.result()
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", *LINK_FLAGS, "-o", LIB + ".tmp",
           *[_obj(s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr, flush=True)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_variant(out: str, extra: str, only) -> str:
    """A/B helper: the library with the TUs `only` (basenames, e.g. engine.cu)
    recompiled with the extra flags and every other object as built."""
    build()
    objs = []
    for src in SOURCES:
        if os.path.basename(src) in only:
            o = os.path.join(OBJ, "variant_" + os.path.basename(src)[:-3] + ".o")
            subprocess.run([nvcc(), *NVCC_FLAGS, *extra.split(), "-c", "-o", o, src], check=True)
            objs.append(o)
        else:
            objs.append(_obj(src))
    subprocess.run([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", *LINK_FLAGS, "-o", out, *objs], check=True)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
