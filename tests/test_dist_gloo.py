"""World-size-2 gloo test of the multi-GPU exchange (CPU only): each rank computes the
top-k of its shard (with the oracle, standing in for the GPU sweep), the records go
through paper_2104_09075_b200.dist.gather_topk exactly as on NCCL, and the merged
result equals the whole-range top-k and count."""
from __future__ import annotations

import os
import socket
import struct

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import corpus

K = 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _records(hits):
    t = torch.empty((len(hits), 2), dtype=torch.int64)
    for i, (idx, key) in enumerate(hits):
        t[i, 0] = struct.unpack("<q", struct.pack("<Q", idx))[0]
        t[i, 1] = struct.unpack("<q", struct.pack("<d", key))[0]
    return t


def _worker(rank, ws, port, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from oracle import oracle as O
        from paper_2104_09075_b200 import dist as D
        sw = corpus.random_sweep(seed)
        osw = O.OracleSweep(sw)
        n = osw.size()
        # strided chunk shards, like the GPU tile shards
        chunk = max(1, n // 7)
        mine = []
        cnt = 0
        for c0 in range(rank * chunk, n, ws * chunk):
            hits, nf = osw.topk(c0, min(chunk, n - c0), K, nthreads=1)
            mine += [h for h in hits if h[0] != 2 ** 64 - 1]
            cnt += nf
        mine = sorted(mine, key=lambda h: (h[1], h[0]))[:K]
        mine += [(2 ** 64 - 1, float("inf"))] * (K - len(mine))
        lists, counts = D.gather_topk(_records(mine), torch.tensor([cnt], dtype=torch.int64))
        if rank == 0:
            allh = []
            for r in range(ws):
                allh += D.decode_hits(lists[r])
            merged = sorted([h for h in allh if h[0] != 2 ** 64 - 1], key=lambda h: (h[1], h[0]))[:K]
            ref, ref_n = osw.topk(0, n, K, nthreads=1)
            ref = [h for h in ref if h[0] != 2 ** 64 - 1]
            q.put((merged == ref, int(counts.sum()) == ref_n, lists.shape))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed", [1, 5, 9])
def test_gloo_world2_merge(oracle_mod, seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    ok_hits, ok_count, shape = q.get(timeout=5)
    assert ok_hits and ok_count
    assert tuple(shape) == (2, K, 2)
