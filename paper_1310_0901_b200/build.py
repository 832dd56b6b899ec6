"""Builds the sm_100a C-ABI library ``libcgcheck.so`` in-tree with nvcc."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcgcheck.so")
SOURCES = [os.path.join(CSRC, f) for f in ("cg_kernels.cu", "cg_runtime.cu", "cg_conc.cu", "cg_shard.cu")]
HEADERS = [os.path.join(ROOT, "include", "cg.h"), os.path.join(CSRC, "cg_internal.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-shared", "-Xptxas", "-v",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-ldl"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        extra = os.environ.get("CG_NVCC_EXTRA", "").split()   # tuning experiments (-D...)
        cmd = [NVCC] + FLAGS + extra + ["-o", LIB] + SOURCES
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libcgcheck.so")
        if verbose:
            sys.stderr.write(r.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
