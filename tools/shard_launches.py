"""A few topk_async calls on shard 0 of N (for an ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_09075_b200 as P
from workloads import sweeps as W
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ctx = P.Context(0)
spec = ctx.prepare(W.config2())
n = ctx.sweep_size(spec)
rec = torch.zeros((65, 2), dtype=torch.int64, device="cuda")
for _ in range(6):
    ctx.topk_async(spec, 0, n, 0, ns, 64, rec.data_ptr(), rec[64].data_ptr())
torch.cuda.synchronize()
print("ok")
