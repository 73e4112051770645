"""Profiling driver for the SURVEY §8(f) next-row sweeps: python tools/prof_next.py gpipe|spatial_ag"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_09075_b200 as P
from workloads import sweeps as W

name = sys.argv[1] if len(sys.argv) > 1 else "gpipe"
sw = W.NEXT[name]()
ctx = P.Context(0)
spec = ctx.prepare(sw)
n = ctx.sweep_size(spec)
dh = torch.empty((64, 2), dtype=torch.int64, device="cuda")
dc = torch.zeros(1, dtype=torch.int64, device="cuda")
for i in range(2):
    ctx.topk_async(spec, 0, n, 0, 1, 64, dh.data_ptr(), dc.data_ptr())
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
ctx.topk_async(spec, 0, n, 0, 1, 64, dh.data_ptr(), dc.data_ptr())
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e)
print(f"{name}: {n} configs in {ms:.3f} ms = {n/ms/1e6:.1f} Gconfigs/s; count {int(dc.item())}")
