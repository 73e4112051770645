"""Times topk over a window of a BASELINE config's sweep: python tools/time_window.py CFG FIRST COUNT"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_09075_b200 as P
from workloads import sweeps as W
cfg, first, count = int(sys.argv[1]), int(float(sys.argv[2])), int(float(sys.argv[3]))
sw = W.CONFIGS[cfg]()
ctx = P.Context(0)
spec = ctx.prepare(sw)
n = ctx.sweep_size(spec)
first = min(first, n - 1); count = min(count, n - first)
dh = torch.empty((64, 2), dtype=torch.int64, device="cuda")
dc = torch.zeros(1, dtype=torch.int64, device="cuda")
ctx.topk_async(spec, first, count, 0, 1, 64, dh.data_ptr(), dc.data_ptr())
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    ctx.topk_async(spec, first, count, 0, 1, 64, dh.data_ptr(), dc.data_ptr())
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 3
print(f"cfg{cfg} [{first}, +{count}): {ms:.3f} ms = {count/ms*1e3:.4g} configs/s; feasible {int(dc.item())}")
