"""Builds the checked variant of libparadl (device bounds checks, PARADL_CHECKS=1) into
exp/libparadl_checked.so.  Run the GPU suite against it with
    PARADL_LIB=$PWD/exp/libparadl_checked.so python -m pytest tests -m gpu
(compute-sanitizer is not available on the GPU pool)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import importlib.util  # noqa: E402

spec = importlib.util.spec_from_file_location("_b", os.path.join(ROOT, "paper_2104_09075_b200", "build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
out = os.path.join(ROOT, "exp", "libparadl_checked.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
cmd = [b.nvcc(), *b.NVCC_FLAGS, "-DPARADL_CHECKS=1", "-o", out, *b.SOURCES]
subprocess.check_call(cmd)
print(out)
