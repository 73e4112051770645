"""Multi-GPU sweep: tile shards per rank + one all_gather of fixed-size top-k records.

SURVEY §8(e): every rank runs paradl_topk_async on its tile shard (t % world == rank),
then the (k x 16 B) hit records and the feasible counts are all-gathered (NCCL over
NVLink on GPUs; gloo on CPU for tests) and every rank merges them with the device merge
kernel (paradl_merge_topk).  The merge is order-independent, so the result is bit-identical
to the 1-GPU result.  A hit record is two int64 words: (idx, key bits of the fp64 key).
"""
from __future__ import annotations

import contextlib

import torch
import torch.distributed as dist


def gather_topk(hits: torch.Tensor, count: torch.Tensor, group=None):
    """All-gathers per-rank [k, 2] int64 hit records and [1] int64 counts.
    Returns (lists [world, k, 2], counts [world])."""
    ws = dist.get_world_size(group)
    k = hits.shape[0]
    lists = torch.empty((ws, k, 2), dtype=torch.int64, device=hits.device)
    counts = torch.empty(ws, dtype=torch.int64, device=hits.device)
    if dist.get_backend(group) == "gloo":
        dist.all_gather(list(lists.unbind(0)), hits.contiguous(), group=group)
        dist.all_gather(list(counts.view(ws, 1).unbind(0)), count.view(1).contiguous(), group=group)
    else:
        dist.all_gather_into_tensor(lists.view(ws, -1), hits.reshape(-1).contiguous(), group=group)
        dist.all_gather_into_tensor(counts, count.view(1).contiguous(), group=group)
    return lists, counts


def sharded_topk(ctx, spec, first: int, count: int, k: int, out_hits: torch.Tensor, out_count: torch.Tensor,
                 my_rec: torch.Tensor, group=None, stream=None):
    """One multi-GPU top-k step on the current device: shard -> one all_gather -> device merge.
    my_rec: int64 [k + 1, 2] record (k hits, then the count in row k, column 0); out_hits
    [k, 2] and out_count [1] int64 on the ctx's device.  Returns (out_hits, out_count, stats)
    with this rank's H2D bytes and kernel launches.

    Stream order: the sweep, the collective and the merge all run on `stream` (default: the
    caller's current stream).  The collective is issued under `torch.cuda.stream(stream)`,
    so NCCL waits for the sweep that writes my_rec and the merge waits for the gather, even
    when `stream` is not torch's current stream."""
    ws = dist.get_world_size(group)
    rank = dist.get_rank(group)
    on_gpu = my_rec.is_cuda
    if stream is None and on_gpu:
        stream = torch.cuda.current_stream(my_rec.device)
    ctx.topk_async(spec, first, count, rank, ws, k, my_rec.data_ptr(), my_rec[k].data_ptr(), stream=stream)
    stats = {"h2d": ctx.stat(0), "launches": ctx.stat(2) + 1}
    with torch.cuda.stream(stream) if on_gpu else contextlib.nullcontext():
        recs = torch.empty((ws, k + 1, 2), dtype=torch.int64, device=my_rec.device)
        if dist.get_backend(group) == "gloo":
            dist.all_gather(list(recs.unbind(0)), my_rec.contiguous(), group=group)
        else:
            dist.all_gather_into_tensor(recs.view(ws, -1), my_rec.reshape(-1).contiguous(), group=group)
    ctx.merge_records(recs.data_ptr(), ws, k, out_hits.data_ptr(), out_count.data_ptr(), stream=stream)
    return out_hits, out_count, stats


def decode_hits(hits: torch.Tensor):
    """[k, 2] int64 records -> list of (idx, key) (host)."""
    h = hits.detach().cpu()
    idx = [int(v) & ((1 << 64) - 1) for v in h[:, 0].tolist()]
    keys = h[:, 1].contiguous().view(torch.float64).tolist()
    return list(zip(idx, keys))
