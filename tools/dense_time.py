"""Dense-mode timing on a 2^28-config cfg2 window + a pure-write reference (torch fill)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_09075_b200 as P
from workloads import sweeps as W
ctx = P.Context(0)
spec = ctx.prepare(W.config2())
N = ctx.sweep_size(spec)
cnt = 1 << 28
t = torch.empty(cnt, dtype=torch.float64, device="cuda"); m = torch.empty_like(t)
bits = torch.empty(cnt // 32, dtype=torch.int32, device="cuda"); rs = torch.empty(cnt, dtype=torch.uint8, device="cuda")
first = (N // 3) // 32 * 32
def run():
    ctx.sweep_dense(spec, first, cnt, t.data_ptr(), m.data_ptr(), bits.data_ptr(), rs.data_ptr())
for _ in range(2): run()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); run(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
ms = statistics.median(ts)
print(f"dense {cnt} configs {ms:.3f} ms  {cnt*17.125/ms/1e6:.0f} GB/s")
buf = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
buf.fill_(1); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); buf.fill_(3); b.record(); torch.cuda.synchronize()
print(f"torch fill (write-only) {4*1.073741824/a.elapsed_time(b)*1e3:.0f} GB/s")
