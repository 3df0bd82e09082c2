"""Build libfsgpu.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

    python -m paper_2405_07989_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(HERE, "libfsgpu.so")
SOURCES = ["fs_host.cu", "fs_capi.cu", "fs_launch.cu", "fs_k_count.cu", "fs_k_hist.cu", "fs_k_any.cu", "fs_k_rows.cu", "fs_k_rowsany.cu", "fs_k_rowsb.cu", "fs_micro.cu"]
HEADERS = ["fs_core.cuh", "fs_internal.h", "fs_kernels.cuh", "fs_rows_batch.cuh"]
INCLUDE = [os.path.join(ROOT, "include", h) for h in ("fsgpu.h", "fsgpu_debug.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-Xcompiler", "-fvisibility=default"]
# experiments only (e.g. FS_NVCC_EXTRA="-DFS_CC_GROUP=8"); the shipped build sets none
FLAGS += os.environ.get("FS_NVCC_EXTRA", "").split()


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + INCLUDE + [__file__]
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest(deps):
        return LIB
    objs = []

    def compile_one(src):
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        cmd = [NVCC] + ARCH + FLAGS + (["-Xptxas", "-v"] if verbose else []) + [
            "-c", os.path.join(CSRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError("nvcc failed for %s:\n%s" % (src, res.stderr))
        if verbose:
            with open(os.path.join(BUILD, src + ".ptxas.log"), "w") as f:
                f.write(res.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("link failed:\n%s" % res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
