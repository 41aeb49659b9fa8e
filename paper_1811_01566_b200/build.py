"""Build the in-tree CUDA library ``_lib/libbmode200.so`` for sm_100a.

    python -m paper_1811_01566_b200.build          # or __graft_entry__.build()

nvcc cross-compiles without a GPU; the resulting .so travels with the repo
snapshot to the GPU box.
"""

from __future__ import annotations

import concurrent.futures
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "_lib", "libbmode200.so")
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
    f"-I{os.path.join(ROOT, 'include')}",
]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))  # noqa


def deps():
    return sources() + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [
        os.path.join(ROOT, "include", "bmode200.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


# Files whose results must be bitwise equal to the reference: no FMA
# contraction anywhere (ptxas would otherwise fuse mul.rn.f32x2 + add.rn.f32x2
# into FFMA2, changing the rounding of the DAS accumulation).
NO_FMAD = {"bm_das.cu", "bm_das_tma.cu", "bm_das_tma64.cu"}


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = os.path.join(HERE, "_lib", "obj")
    os.makedirs(objdir, exist_ok=True)
    jobs = []
    for src in sources():
        name = os.path.basename(src)
        obj = os.path.join(objdir, name + ".o")
        flags = [f for f in NVCC_FLAGS if f != "-shared"]
        if name in NO_FMAD:
            flags.append("-fmad=false")
        cmd = [nvcc, *flags, "-c", "-o", obj, src]
        hdrs = [p for p in deps() if not p.endswith(".cu")]
        if (not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(
                os.path.getmtime(p) for p in [src] + hdrs)):
            continue
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        jobs.append((obj, cmd))
    # one nvcc per translation unit, in parallel
    with concurrent.futures.ThreadPoolExecutor(max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for _ in ex.map(lambda j: subprocess.run(j[1], check=True), jobs):
            pass
    objs = [os.path.join(objdir, os.path.basename(s) + ".o") for s in sources()]
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB + ".tmp",
           *objs]
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
