"""Per-rank breakdown of one multi-GPU top-k step (torchrun): sweep+local merge, all_gather,
record merge -- CUDA events on the current stream, averaged over steps."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2104_09075_b200 as P
from workloads import sweeps as W
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ws, rank = dist.get_world_size(), dist.get_rank()
ctx = P.Context(local)
spec = ctx.prepare(W.config2())
n = ctx.sweep_size(spec)
k = 64
rec = torch.zeros((k + 1, 2), dtype=torch.int64, device="cuda")
recs = torch.empty((ws, k + 1, 2), dtype=torch.int64, device="cuda")
out = torch.empty((k, 2), dtype=torch.int64, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
T = {"sweep": [], "gather": [], "merge": [], "step": []}
for it in range(40):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    dist.barrier()
    e[0].record(st)
    ctx.topk_async(spec, 0, n, rank, ws, k, rec.data_ptr(), rec[k].data_ptr(), stream=st)
    e[1].record(st)
    dist.all_gather_into_tensor(recs.view(ws, -1), rec.reshape(-1))
    e[2].record(st)
    ctx.merge_records(recs.data_ptr(), ws, k, out.data_ptr(), cnt.data_ptr(), stream=st)
    e[3].record(st)
    torch.cuda.synchronize()
    if it >= 10:
        T["sweep"].append(e[0].elapsed_time(e[1])); T["gather"].append(e[1].elapsed_time(e[2]))
        T["merge"].append(e[2].elapsed_time(e[3])); T["step"].append(e[0].elapsed_time(e[3]))
print(f"rank {rank}: " + ", ".join(f"{kk} {1e3*statistics.median(v):.1f} us" for kk, v in T.items()), flush=True)
dist.destroy_process_group()
