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


RECORD = LIB + ".build.json"   # sources' SHA-256 + flags of the build that produced LIB


def fingerprint() -> dict:
    import hashlib
    h = {os.path.relpath(p, ROOT): hashlib.sha256(open(p, "rb").read()).hexdigest() for p in SOURCES + HEADERS}
    return {"sources_sha256": h, "nvcc_flags": NVCC_FLAGS}


def up_to_date() -> bool:
    """LIB exists and was built from exactly these sources and flags (content hashes recorded
    by the build next to it; a library without a record is rebuilt)."""
    import json
    if not (os.path.exists(LIB) and os.path.exists(RECORD)):
        return False
    try:
        rec = json.load(open(RECORD))
    except Exception:
        return False
    fp = fingerprint()
    return rec.get("sources_sha256") == fp["sources_sha256"] and rec.get("nvcc_flags") == fp["nvcc_flags"]


def build(force: bool = False, verbose: bool = False) -> str:
    import json
    import time
    if not force and up_to_date():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-o", LIB + ".tmp", *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    t0 = time.time()
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    rec = fingerprint()
    rec.update({"built_utc": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), "seconds": round(time.time() - t0, 1),
                "nvcc": subprocess.run([nvcc(), "--version"], capture_output=True, text=True).stdout.strip().splitlines()[-1]})
    with open(RECORD, "w") as f:
        json.dump(rec, f, indent=1)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
