"""Builds libparadl.so in-tree for sm_100a with nvcc (no JIT, no torch extension cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libparadl.so")
SOURCES = [os.path.join(CSRC, "kernels.cu"), os.path.join(CSRC, "api.cpp")]
HEADERS = [os.path.join(CSRC, "paradl_internal.h"), os.path.join(ROOT, "include", "paradl.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off", "-shared",
    "-I", os.path.join(ROOT, "include"),
]


def nvcc() -> str:
    for p in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.isabs(p) and os.path.exists(p):
            return p
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-o", LIB + ".tmp", *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
