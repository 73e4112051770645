"""Multi-process GPU test of the product's multi-GPU step (-m gpu): two ranks (gloo process
group, both on cuda:0) run paper_2104_09075_b200.dist.sharded_topk -- the tile-sharded
paradl_topk_async, the all_gather of the (k + 1) x 16 B records and paradl_merge_records on
the device -- exactly as bench.py does over NCCL, and the merged top-k and count equal the
oracle's whole-range reduction."""
from __future__ import annotations

import os
import socket

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist   # noqa: E402
import torch.multiprocessing as mp   # noqa: E402

K = 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sweep(name):
    from workloads import sweeps as W
    if name == "cfg2":
        return W.config2(n_alpha=8, n_beta=64, b_list=[2, 32, 256], pipe_smax=3)
    if name == "cfg5":
        return W.config5(s_max=3)
    return W.config4(n_alpha=4, n_beta=4)


def _worker(rank, ws, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        import paper_2104_09075_b200 as P
        from paper_2104_09075_b200 import dist as D
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        sw = _sweep(name)
        ctx = P.Context(0)
        spec = ctx.prepare(sw)
        n = ctx.sweep_size(spec)
        my_rec = torch.zeros((K + 1, 2), dtype=torch.int64, device=dev)
        out = torch.empty((K, 2), dtype=torch.int64, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        side = torch.cuda.Stream(dev)   # not the current stream: sharded_topk must order itself
        D.sharded_topk(ctx, spec, 0, n, K, out, cnt, my_rec, stream=side)
        side.synchronize()
        q.put((rank, D.decode_hits(out), int(cnt.item()), n))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg2", "cfg5", "cfg4"])
def test_sharded_topk_two_ranks_vs_oracle(oracle_mod, name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    osw = oracle_mod.OracleSweep(_sweep(name))
    n = osw.size()
    ohits, onf = osw.topk(0, n, K)
    for rank, hits, nf, ng in res:
        assert ng == n
        assert nf == onf, (rank, nf, onf)
        assert [h[0] for h in hits] == [h[0] for h in ohits]
        assert [h[1] for h in hits] == [h[1] for h in ohits]
