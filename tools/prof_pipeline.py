"""Profiling driver: the dominant cfg2 kernel (pipeline sub-sweep, reduce mode), a few launches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_09075_b200 as P
from workloads import sweeps as W

which = sys.argv[1] if len(sys.argv) > 1 else "pipeline"
fam = {"pipeline": W.PIPELINE, "data": W.DATA, "ds": W.DS, "df": W.DF, "spatial": W.SPATIAL,
       "filter": W.FILTER, "pd": W.PD, "all": -1}[which]
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sw = W.CONFIGS[cfg]()
ctx = P.Context(0)
spec = ctx.prepare(sw)
subs = [i for i, s in enumerate(sw.subs) if s.family == fam]
dspec = spec if fam < 0 else P.Spec([sw.subs[subs[0]]], [spec.c.sub[subs[0]].model_id])
n = ctx.sweep_size(dspec)
dh = torch.empty((64, 2), dtype=torch.int64, device="cuda")
dc = torch.zeros(1, dtype=torch.int64, device="cuda")
for i in range(3):
    ctx.topk_async(dspec, 0, n, 0, 1, 64, dh.data_ptr(), dc.data_ptr())
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
ctx.topk_async(dspec, 0, n, 0, 1, 64, dh.data_ptr(), dc.data_ptr())
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e)
print(f"{which}: {n} configs in {ms:.3f} ms = {n/ms/1e6:.1f} Gconfigs/s; count {int(dc.item())}")
