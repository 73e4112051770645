"""Small GPU workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every kernel family and evaluation path once -- dense, top-k (with the many-list fused merge
and its last-block ticket), compact, mode-1/2/3 pipeline paths, the structure table, explain --
each checked against the oracle so a sanitizer-clean run is also a correct one.

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_09075_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from workloads import corpus  # noqa: E402
from workloads import sweeps as W  # noqa: E402

dev = torch.device("cuda:0")
ok = 0


def run(sw, k=16, dense=True):
    global ok
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = O.OracleSweep(sw)
    n = osw.size()
    hits, nf = ctx.topk(spec, k, 0, n)
    oh, onf = osw.topk(0, n, k)
    assert nf == onf and [h[0] for h in hits] == [h[0] for h in oh], sw.name
    if dense:
        c = min(n, 50_000)
        t = torch.empty(c, dtype=torch.float64, device=dev)
        bits = torch.empty((c + 31) // 32, dtype=torch.int32, device=dev)
        ctx.sweep_dense(spec, 0, c, t.data_ptr(), 0, bits.data_ptr(), 0)
        idx = torch.empty(c, dtype=torch.int64, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        ctx.sweep_compact(spec, 0, c, idx.data_ptr(), c, cnt.data_ptr(), t.data_ptr(), 0)
        torch.cuda.synchronize()
        _, _, _, ors = osw.dense(0, c)
        assert int(cnt.item()) == int(np.sum(ors == 0)), sw.name
    ctx.explain(spec, hits[0][0] if hits[0][0] != 2 ** 64 - 1 else 0)
    ok += 1


for seed in (0, 1, 2):
    run(corpus.random_sweep(seed))
run(W.config5(s_max=3), dense=False)                                           # mode 3 (COMB pd)
run(W.config2(n_alpha=3, n_beta=32, b_list=[2, 64], pipe_smax=3), k=64)        # slots, many CTA lists
run(W.config2(n_alpha=8, n_beta=64, b_list=[2, 32], pipe_smax=3), k=64, dense=False)   # structure table
sw = W.config3(n_alpha=2, n_beta=2)
from workloads import models as M  # noqa: E402
vgg = M.vgg16()
sw.models = [M.Model("vgg14", vgg.layers[:14], vgg.D, default_Ls=14)]
sw.subs = [W.SubSweep(W.PIPELINE, part_mode=W.PART_MASK, S=[4], b=[64])]
run(sw, k=64, dense=False)                                                      # mode 2 masks
run(W.next_layerwise(n_alpha=2, n_beta=32), dense=False)
print(f"sanitize driver: {ok} workloads ok")
