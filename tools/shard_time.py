"""Device time of one shard of a BASELINE sweep on one GPU: topk_async(shard s of N) for
each s, CUDA events on the launching stream, L2 flushed before each call.

    python tools/shard_time.py CFG N [REPS]

Separates the per-shard sweep time (what each rank of an N-GPU step runs) from the
collective and merge that follow it in bench.py's multi-GPU step."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_09075_b200 as P  # noqa: E402
from workloads import sweeps as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
ctx = P.Context(0)
spec = ctx.prepare(W.CONFIGS[cfg]())
n = ctx.sweep_size(spec)
rec = torch.zeros((65, 2), dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for s in range(ns):
    ctx.topk_async(spec, 0, n, s, ns, 64, rec.data_ptr(), rec[64].data_ptr(), stream=st)
torch.cuda.synchronize()
for s in range(ns):
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        ctx.topk_async(spec, 0, n, s, ns, 64, rec.data_ptr(), rec[64].data_ptr(), stream=st)
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"cfg{cfg} shard {s}/{ns}: {statistics.median(ts):.3f} ms (min {min(ts):.3f})", flush=True)
