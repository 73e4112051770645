"""Host-side enqueue time of paradl_topk_async (no synchronisation) vs device time.

    python tools/host_overhead.py [CFG] [SHARDS,...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_09075_b200 as P
from workloads import sweeps as W
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
shards = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 4, 8]
sw = W.CONFIGS[cfg]()
ctx = P.Context(0)
spec = ctx.prepare(sw)
n = ctx.sweep_size(spec)
rec = torch.zeros((65, 2), dtype=torch.int64, device="cuda")
for ns in shards:
    for _ in range(3):
        ctx.topk_async(spec, 0, n, 0, ns, 64, rec.data_ptr(), rec[64].data_ptr())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        ctx.topk_async(spec, 0, n, 0, ns, 64, rec.data_ptr(), rec[64].data_ptr())
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"shards {ns}: host enqueue {1e6*(t1-t0)/20:.1f} us/call, wall incl. device {1e6*(t2-t0)/20:.1f} us/call")
