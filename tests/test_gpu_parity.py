"""GPU parity: the CUDA path through the C-ABI vs the CPU oracle (-m gpu).

Bar (BASELINE.json north_star): bit-exact feasibility masks, reasons, feasible counts,
partition decodes, argmin / top-k indices (ties -> lowest index); fp64 times and memory
within 1e-9 relative (the design target is bit-identical, so the tests
also report how many differ at all).
"""
from __future__ import annotations

import math
import random

import numpy as np
import pytest

from workloads import corpus
from workloads import sweeps as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2104_09075_b200 as P   # noqa: E402

REL = 1e-9


@pytest.fixture(scope="module")
def dev():
    return torch.device("cuda:0")


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    both_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
    with np.errstate(invalid="ignore"):   # inf - inf: same-sign infinities are zeroed below
        d = np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)
    d[both_inf] = 0.0
    d[(a == b)] = 0.0
    return d


def gpu_dense(ctx, spec, first, count, dev):
    t = torch.empty(count, dtype=torch.float64, device=dev)
    m = torch.empty(count, dtype=torch.float64, device=dev)
    bits = torch.empty((count + 31) // 32, dtype=torch.int32, device=dev)
    rs = torch.empty(count, dtype=torch.uint8, device=dev)
    ctx.sweep_dense(spec, first, count, t.data_ptr(), m.data_ptr(), bits.data_ptr(), rs.data_ptr(),
                    stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    return (t.cpu().numpy(), m.cpu().numpy(), bits.cpu().numpy().view(np.uint32), rs.cpu().numpy())


def check_dense(ctx, spec, osw, first, count, dev):
    t, m, bits, rs = gpu_dense(ctx, spec, first, count, dev)
    ot, om, obits, ors = osw.dense(first, count)
    assert np.array_equal(rs, ors), np.nonzero(rs != ors)[0][:10]
    assert np.array_equal(bits, obits)
    assert rel_err(t, ot).max() <= REL
    assert rel_err(m, om).max() <= REL
    return int(np.sum(t != ot)) + int(np.sum(m != om))


def check_topk(ctx, spec, osw, first, count, k):
    hits, nf = ctx.topk(spec, k, first, count)
    ohits, onf = osw.topk(first, count, k)
    assert nf == onf
    assert [h[0] for h in hits] == [h[0] for h in ohits]
    for (gi, gk), (oi, ok) in zip(hits, ohits):
        if oi == 2 ** 64 - 1:
            assert math.isinf(gk) and gi == oi
        else:
            assert abs(gk - ok) <= REL * abs(ok)
    return hits, nf


# ------------------------------------------------------------------ random corpora (all families)
@pytest.mark.parametrize("seed", range(40))
def test_random_corpus_dense_and_topk(dev, oracle_mod, seed):
    sw = corpus.random_sweep(seed)
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = ctx.sweep_size(spec)
    assert n == osw.size()
    diffs = check_dense(ctx, spec, osw, 0, n, dev)
    assert diffs == 0, f"{diffs} values not bit-identical (within tolerance)"
    for k in (1, 7, 64):
        check_topk(ctx, spec, osw, 0, n, k)
    rng = random.Random(seed)
    for _ in range(3):   # ragged sub-ranges crossing sub-sweep boundaries
        a = rng.randrange(n)
        c = rng.randrange(n - a + 1)
        check_dense(ctx, spec, osw, a, c, dev)
        check_topk(ctx, spec, osw, a, c, rng.choice([1, 5, 33]))


@pytest.mark.parametrize("seed", range(10))
def test_explain_and_decode(dev, oracle_mod, seed):
    sw = corpus.random_sweep(seed)
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    rng = random.Random(seed)
    for idx in [0, n - 1] + [rng.randrange(n) for _ in range(40)]:
        g = ctx.explain(spec, idx)
        o = osw.explain(idx)
        for f in ("t_comp", "t_ge", "t_fb_ag", "t_fb_ar", "t_halo", "t_p2p", "t_iter", "t_epoch", "mem", "I"):
            assert rel_err([getattr(g, f)], [getattr(o, f)])[0] <= REL, (idx, f)
        assert g.reason == o.reason and g.feasible == o.feasible
        gc = ctx.decode(spec, idx)
        oc = osw.decode(idx)
        assert gc.sub == oc.sub and gc.n_stages == oc.n_stages
        assert list(gc.stage_end[:gc.n_stages]) == list(oc.stage_end[:oc.n_stages])
        assert (gc.b, gc.S, gc.Ls, tuple(gc.dims)) == (oc.b, oc.S, oc.Ls, tuple(oc.dims))
        assert gc.B == o.B and gc.p == o.p


def test_empty_and_edge_ranges(dev, oracle_mod):
    sw = corpus.random_sweep(3)
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    hits, nf = ctx.topk(spec, 4, n, 0)
    assert nf == 0 and all(h[0] == 2 ** 64 - 1 for h in hits)
    check_dense(ctx, spec, osw, n - 1, 1, dev)
    check_dense(ctx, spec, osw, 5, 31, dev)
    check_dense(ctx, spec, osw, 3, 33, dev)
    with pytest.raises(P.ParadlError) as e:
        ctx.topk(spec, 4, n, 1)
    assert e.value.status == -5
    with pytest.raises(P.ParadlError):
        ctx.topk(spec, 65, 0, n)


# ------------------------------------------------------------------ BASELINE configs
def test_config1_full(dev, oracle_mod):
    sw = W.config1()
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    assert check_dense(ctx, spec, osw, 0, 33, dev) == 0
    hits, nf = check_topk(ctx, spec, osw, 0, 33, 33)
    assert nf == 22 and hits[0][0] == 31
    (best, key), nf1 = ctx.argmin(spec)
    assert best == 31 and nf1 == 22


def _small(cfg, **kw):
    return W.CONFIGS[cfg](**kw) if kw else W.CONFIGS[cfg]()


@pytest.mark.parametrize("cfg,kw", [(2, dict(n_alpha=3, n_beta=5, b_list=[1, 7, 64, 256], pipe_smax=3)),
                                    (3, dict(n_alpha=3, n_beta=2)),
                                    (4, dict(n_alpha=2, n_beta=3)),
                                    (5, dict(s_max=3))])
def test_reduced_configs(dev, oracle_mod, cfg, kw):
    sw = _small(cfg, **kw)
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    full = n <= 3_000_000
    if full:
        assert check_dense(ctx, spec, osw, 0, n, dev) == 0
        check_topk(ctx, spec, osw, 0, n, 64)
    rng = random.Random(cfg)
    for _ in range(6):
        a = rng.randrange(max(1, n - 100_000))
        c = min(n - a, rng.randrange(1, 100_000))
        check_dense(ctx, spec, osw, a, c, dev)
        check_topk(ctx, spec, osw, a, c, 16)


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_full_size_windows(dev, oracle_mod, cfg):
    """Full BASELINE sizes: dense windows at random offsets (bench's launch configuration)
    against the oracle's one-by-one evaluation."""
    sw = W.CONFIGS[cfg]()
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    rng = random.Random(100 + cfg)
    starts = [0, n - 4000] + [rng.randrange(n - 4000) for _ in range(10)]
    for a in starts:
        c = rng.randrange(1000, 4000)
        check_dense(ctx, spec, osw, a, c, dev)
        check_topk(ctx, spec, osw, a, c, 8)


@pytest.mark.parametrize("cfg", [2, 4])
def test_full_sweep_topk_properties(dev, oracle_mod, cfg):
    """Whole-sweep top-k at full size: every hit re-evaluated by the oracle gives its key;
    hits are feasible, sorted, and no sampled configuration beats the k-th hit; the count
    equals the popcount of the dense feasibility bits over the same range."""
    sw = W.CONFIGS[cfg]()
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    hits, nf = ctx.topk(spec, 64, 0, n)
    keys = [h[1] for h in hits]
    assert keys == sorted(keys)
    idx = np.array([h[0] for h in hits], np.uint64)
    t, m, r, key = osw.eval_many(idx)
    assert np.all(r == 0)
    assert rel_err(key, keys).max() <= REL
    rng = np.random.default_rng(cfg)
    sample = rng.integers(0, n, 200_000, dtype=np.uint64)
    _, _, rs, ks = osw.eval_many(sample)
    kth = (keys[-1], int(idx[-1]))
    better = [(k_, int(i_)) for k_, i_, r_ in zip(ks, sample, rs) if r_ == 0 and (k_, int(i_)) < kth]
    assert all(int(i_) in set(int(x) for x in idx) for _, i_ in better)
    # count vs dense popcount (chunked)
    tot = 0
    chunk = 1 << 27
    dev_bits = torch.empty((chunk + 31) // 32, dtype=torch.int32, device=dev)
    for a in range(0, n, chunk):
        c = min(chunk, n - a)
        ctx.sweep_dense(spec, a, c, 0, 0, dev_bits.data_ptr(), 0, stream=torch.cuda.current_stream())
        nw = (c + 31) // 32
        tot += int(torch.sum(_popcount(dev_bits[:nw])))
    assert tot == nf


def _popcount(x):
    x = x.to(torch.int64) & 0xFFFFFFFF
    x = x - ((x >> 1) & 0x55555555)
    x = (x & 0x33333333) + ((x >> 2) & 0x33333333)
    x = (x + (x >> 4)) & 0x0F0F0F0F
    return ((x * 0x01010101) & 0xFFFFFFFF) >> 24


@pytest.mark.parametrize("kw", [dict(n_alpha=8, n_beta=8, b_list=[2, 32, 256], pipe_smax=3),
                                dict(n_alpha=64, n_beta=64, b_list=[8, 64, 256], pipe_smax=3)])
def test_sharded_topk_merge_equals_single(dev, oracle_mod, kw):
    """Shards (tile t -> shard t % n) merged on the device equal the single call; the second
    sweep is large enough for the pipeline structure table, built per shard for its tiles."""
    sw = W.config2(**kw)
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    n = ctx.sweep_size(spec)
    k = 32
    single, nf = ctx.topk(spec, k)
    for ns in (2, 3, 4, 8):
        lists = torch.empty((ns, k, 2), dtype=torch.int64, device=dev)
        counts = torch.zeros(ns, dtype=torch.int64, device=dev)
        for s in range(ns):
            ctx.topk_async(spec, 0, n, s, ns, k, lists[s].data_ptr(), counts[s:].data_ptr(),
                           stream=torch.cuda.current_stream())
        out = torch.empty((k, 2), dtype=torch.int64, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        ctx.merge_topk(lists.data_ptr(), ns, k, counts.data_ptr(), out.data_ptr(), cnt.data_ptr(),
                       stream=torch.cuda.current_stream())
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        got = [int(v) for v in o[:, 0].astype(np.uint64)]
        assert got == [h[0] for h in single]
        assert int(cnt.item()) == nf


@pytest.mark.parametrize("seed,G,fam", [(11, 10, W.PIPELINE), (12, 12, W.PD), (13, 13, W.LAYERPURE),
                                         (14, 11, W.PD), (15, 14, W.PIPELINE)])
def test_lane_blocked_modes(dev, oracle_mod, seed, G, fam):
    """Lane-blocked evaluation (COMB partitions and 256-mask blocks with the low-bit stage
    table) against the oracle on whole sweeps and ragged sub-ranges."""
    m = corpus.random_model(seed, G=G)
    sysd = corpus.random_system(seed)
    nt = len(sysd.tiers)
    A = [[1e-6 * (i + 1) * (t + 1) for t in range(nt)] for i in range(2)]
    Bt = [[1e-10 * (i + 3) * (t + 1) for t in range(nt)] for i in range(3)]
    common = dict(b=[2, 8], S=[1, 2, 4], alpha=A, beta=Bt, cap=[2.0 ** 20, 2.0 ** 40])
    if fam == W.PD:
        common["dims"] = [(p, 1, 1, 1) for p in (1, 2, 8)]
    subs = [W.SubSweep(fam, part_mode=W.PART_MASK, **common),
            W.SubSweep(fam, part_mode=W.PART_COMB, s_min=1, s_max=min(4, G), **common)]
    sw = W.Sweep([m], sysd, subs, "blocked")
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    for k in (1, 64):
        check_topk(ctx, spec, osw, 0, n, k)
    rng = random.Random(seed)
    for _ in range(4):
        a = rng.randrange(n)
        c = rng.randrange(1, n - a + 1)
        check_topk(ctx, spec, osw, a, c, rng.choice([3, 33]))


@pytest.mark.parametrize("seed,fam,tree", [(21, W.PD, 0.0), (22, W.PD, 1e6), (23, W.PIPELINE, 0.0),
                                           (24, W.PD, 0.0)])
def test_lane_blocked_screened(dev, oracle_mod, seed, fam, tree):
    """Mode-1 screened path (pipeline / pd, ring collectives): several S passes (7 S values,
    one ragged pass), S > b (Segments), power-of-two and other p_d (exact-division shortcut vs
    IEEE division), p_d beyond every tier (Tier), memory-infeasible stages; tree_threshold > 0
    takes the unscreened path.  Whole sweep and ragged windows against the oracle."""
    import dataclasses
    m = corpus.random_model(seed, G=12)
    sysd = dataclasses.replace(corpus.random_system(seed), tree_threshold=tree)
    nt = len(sysd.tiers)
    A = [[1e-6 * (i + 1) * (t + 1) for t in range(nt)] for i in range(2)]
    Bt = [[1e-10 * (i + 3) * (t + 1) for t in range(nt)] for i in range(2)]
    common = dict(b=[3, 16], S=[1, 2, 3, 4, 5, 8, 32], alpha=A, beta=Bt, cap=[2.0 ** 22, 2.0 ** 40])
    if fam == W.PD:
        common["dims"] = [(p, 1, 1, 1) for p in (1, 2, 3, 6, 8, 48, 1024, 4096)]
    subs = [W.SubSweep(fam, part_mode=W.PART_COMB, s_min=1, s_max=5, **common)]
    sw = W.Sweep([m], sysd, subs, "screened")
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    for k in (1, 64):
        check_topk(ctx, spec, osw, 0, n, k)
    rng = random.Random(seed)
    for _ in range(3):
        a = rng.randrange(n)
        c = rng.randrange(1, n - a + 1)
        check_topk(ctx, spec, osw, a, c, rng.choice([5, 64]))


@pytest.mark.parametrize("seed,G,S", [(31, 12, 4), (32, 16, 1), (33, 14, 8), (34, 13, 2)])
def test_mask_blocks_screened(dev, oracle_mod, seed, G, S):
    """Mode-2 screened path (pipeline masks, one configuration per mask as in cfg3-ii):
    memory threshold, tier of the stage count, S > b, two b values, ragged windows."""
    m = corpus.random_model(seed, G=G)
    sysd = corpus.random_system(seed)
    nt = len(sysd.tiers)
    A = [[2e-6 * (t + 1) for t in range(nt)]]
    Bt = [[3e-10 * (t + 1) for t in range(nt)]]
    subs = [W.SubSweep(W.PIPELINE, part_mode=W.PART_MASK, b=[4, 16], S=[S], alpha=A, beta=Bt,
                       cap=[2.0 ** 18, 2.0 ** 24, 2.0 ** 40])]
    sw = W.Sweep([m], sysd, subs, "mask_screened")
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    for k in (1, 64):
        check_topk(ctx, spec, osw, 0, n, k)
    rng = random.Random(seed)
    for _ in range(3):
        a = rng.randrange(n)
        c = rng.randrange(1, n - a + 1)
        check_topk(ctx, spec, osw, a, c, rng.choice([7, 64]))


@pytest.mark.parametrize("seed,G", [(35, 14), (36, 16)])
def test_mask_sorted_tables_two_items(dev, oracle_mod, seed, G):
    """Sorted mask path (one configuration per mask, one flops value, one capacity: the cfg3-ii
    shape) with two b values in each of two work items: the per-CTA low tables of the items
    sit one after the other (64-byte units), so the second item's table and the first
    item's per-(b, e, pop) feasible counts must not overlap.  Whole sweep and windows."""
    m = corpus.random_model(seed, G=G)
    sysd = corpus.random_system(seed)
    nt = len(sysd.tiers)
    A = [[2e-6 * (t + 1) for t in range(nt)]]
    Bt = [[3e-10 * (t + 1) for t in range(nt)]]
    subs = [W.SubSweep(W.PIPELINE, part_mode=W.PART_MASK, b=[4, 16], S=[S], alpha=A, beta=Bt, cap=[2.0 ** 24])
            for S in (2, 1)]
    sw = W.Sweep([m], sysd, subs, "mask_sorted_two")
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    for k in (1, 64):
        check_topk(ctx, spec, osw, 0, n, k)
    rng = random.Random(seed)
    for _ in range(3):
        a = rng.randrange(n)
        c = rng.randrange(1, n - a + 1)
        check_topk(ctx, spec, osw, a, c, rng.choice([7, 64]))


def test_unaligned_windows_all_families(dev, oracle_mod):
    """Ranges starting at every residue mod 32 (lane/slot alignment edge cases), cfg2 shapes."""
    sw = W.config2(n_alpha=3, n_beta=64, b_list=[2, 64], pipe_smax=2)
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    rng = random.Random(7)
    for r in range(32):
        a = rng.randrange(n // 32 - 200) * 32 + r
        c = rng.choice([31, 32, 33, 700, 5000])
        check_topk(ctx, spec, osw, a, c, 5)
        check_dense(ctx, spec, osw, a, c, dev)


def test_merge_records_equals_single(dev):
    """Multi-GPU record layout (k hits + count) merged by paradl_merge_records, shards
    simulated on one GPU, equals the unsharded top-k and count."""
    sw = W.config2(n_alpha=8, n_beta=64, b_list=[2, 32], pipe_smax=3)
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    n = ctx.sweep_size(spec)
    k = 64
    single, nf = ctx.topk(spec, k)
    for ns in (2, 3, 8):
        recs = torch.zeros((ns, k + 1, 2), dtype=torch.int64, device=dev)
        for s in range(ns):
            ctx.topk_async(spec, 0, n, s, ns, k, recs[s].data_ptr(), recs[s, k].data_ptr(),
                           stream=torch.cuda.current_stream())
        out = torch.empty((k, 2), dtype=torch.int64, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        ctx.merge_records(recs.data_ptr(), ns, k, out.data_ptr(), cnt.data_ptr(), stream=torch.cuda.current_stream())
        torch.cuda.synchronize()
        got = [int(v) for v in out.cpu().numpy()[:, 0].astype(np.uint64)]
        assert got == [h[0] for h in single]
        assert int(cnt.item()) == nf


# ------------------------------------------------------------------ SURVEY §8(f) next rows
@pytest.mark.parametrize("name,kw", [("gpipe", dict(n_alpha=3, n_beta=4, b_list=[1, 6, 64], s_max=3)),
                                     ("gpipe", dict(n_alpha=2, n_beta=32, b_list=[8], s_max=2, S_list=(1, 3, 8))),
                                     ("spatial_ag", dict(n_alpha=3, n_beta=2)),
                                     ("data_lw", dict(n_alpha=3, n_beta=5)),
                                     ("data_lw", dict(n_alpha=2, n_beta=64)),
                                     ("layerwise", dict(n_alpha=3, n_beta=2)),
                                     ("layerwise", dict(n_alpha=2, n_beta=32))])
def test_next_rows_reduced(dev, oracle_mod, name, kw):
    """GPipe schedule family and spatial prefix + Allgather family on reduced sweeps: whole
    range dense + top-64 against the oracle, then random windows (ragged tails)."""
    sw = W.NEXT[name](**kw)
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    assert ctx.sweep_size(spec) == n
    if n <= 3_000_000:
        assert check_dense(ctx, spec, osw, 0, n, dev) == 0
        check_topk(ctx, spec, osw, 0, n, 64)
    rng = random.Random(7)
    for _ in range(5):
        a = rng.randrange(max(1, n - 50_000))
        c = min(n - a, rng.randrange(1, 50_000))
        assert check_dense(ctx, spec, osw, a, c, dev) == 0
        check_topk(ctx, spec, osw, a, c, 16)


@pytest.mark.parametrize("name", ["gpipe", "spatial_ag", "data_lw", "layerwise"])
def test_next_rows_full_size(dev, oracle_mod, name):
    """Full-size next-row sweeps (the bench's launch configuration): dense windows and
    window top-k against the oracle; whole-sweep top-k hits re-evaluated one by one."""
    sw = W.NEXT[name]()
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    rng = random.Random(200)
    for a in [0, n - 3000] + [rng.randrange(n - 3000) for _ in range(8)]:
        c = rng.randrange(500, 3000)
        assert check_dense(ctx, spec, osw, a, c, dev) == 0
        check_topk(ctx, spec, osw, a, c, 8)
    hits, nf = ctx.topk(spec, 64, 0, n)
    keys = [h[1] for h in hits]
    assert keys == sorted(keys) and nf > 0
    idx = np.array([h[0] for h in hits], np.uint64)
    _, _, r, key = osw.eval_many(idx)
    assert np.all(r == 0)
    assert rel_err(key, keys).max() == 0.0


def test_gpipe_schedule_matches_table2_for_equal_stages(dev, oracle_mod):
    """On the GPU: a model of equal rows split into equal stages gives the Table 2 Layer
    row's time (PIPELINE family) to rounding, and never more than it otherwise."""
    from workloads import models as M
    rows = [M.Layer("eq", M.CONV, 2, 8, 8, (4, 4, 1), (4, 4, 1), (3, 3, 1), 128, 128, 576, 8,
                    100000, 200000, 1152, M.FLAG_COMM) for _ in range(8)]
    m = M.Model("eq", rows, 1000, default_Ls=8)
    sysm = W.two_tier_system(flops_per_s=1e12)
    A, B = W.ab_grid(np.logspace(-7, -4, 8), 1.0 / np.logspace(9, 12, 8))
    common = dict(part_mode=W.PART_COMB, s_min=1, s_max=8, S=[1, 2, 4, 8], b=[8, 16], alpha=A, beta=B)
    sw = W.Sweep([m], sysm, [W.SubSweep(W.GPIPE, **common), W.SubSweep(W.PIPELINE, **common)], "eq")
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size() // 2
    tg, _, _, _ = gpu_dense(ctx, spec, 0, n, dev)
    tp, _, _, _ = gpu_dense(ctx, spec, n, n, dev)
    assert np.all(tg <= tp * (1 + 1e-14))
    for idx in range(0, n, 97):
        c = osw.decode(idx)
        ends = list(c.stage_end[:c.n_stages])
        sizes = np.diff([0] + ends)
        if np.all(sizes == sizes[0]):
            assert rel_err([tg[idx]], [tp[idx]]).max() <= 1e-14


@pytest.mark.parametrize("kw", [dict(n_alpha=4, n_beta=8, b_list=[1, 3, 16, 256], pipe_smax=3),
                                dict(n_alpha=5, n_beta=7, b_list=[2, 64], pipe_smax=3, S_list=(1, 3, 8)),
                                dict(n_alpha=9, n_beta=64, b_list=[4], pipe_smax=2)])
def test_pipeline_ab_blocks(dev, oracle_mod, kw):
    """cfg2-shaped pipeline sub-sweeps (alpha x beta blocks of 32, 35 and 576 configurations,
    beta-slot reuse when n_beta = 32 M): top-k + count of the whole sub-sweep and of ragged
    windows against the oracle."""
    sw = W.config2(**kw)
    sw.subs = [s for s in sw.subs if s.family == W.PIPELINE]
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    check_topk(ctx, spec, osw, 0, n, 64)
    check_topk(ctx, spec, osw, 0, n, 1)
    rng = random.Random(len(kw))
    for _ in range(4):
        a = rng.randrange(n // 2)
        c = rng.randrange(n // 4, n - a)
        check_topk(ctx, spec, osw, a, c, 32)


# ------------------------------------------------------------------ headline-path parity (round 2)
def test_pipeline_structure_table_vs_oracle(dev, oracle_mod):
    """The pipeline path behind the headline sweeps' dominant sub-sweep: lane-strided work
    items of >= 2^22 configurations read their structure terms from the structure table
    (struct_table_kernel).  Whole sub-sweep top-64 / argmin and count, and ragged windows of
    >= 2^22 configurations, against the oracle (Table 2 Layer row)."""
    sw = W.config2(n_alpha=8, n_beta=64, b_list=[2, 32], pipe_smax=3)
    sw.subs = [s for s in sw.subs if s.family == W.PIPELINE]
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    assert ctx.sweep_size(spec) == n and n >= (1 << 22)
    check_topk(ctx, spec, osw, 0, n, 64)
    check_topk(ctx, spec, osw, 0, n, 1)
    (best, key), nf = ctx.argmin(spec)
    ohits, onf = osw.topk(0, n, 1)
    assert best == ohits[0][0] and nf == onf
    for a, c in [(12345, (1 << 22) + 777), (n - (1 << 22) - 31, (1 << 22) + 31), (3, n - 5)]:
        check_topk(ctx, spec, osw, a, c, 64)


def test_sharded_large_vs_oracle(dev, oracle_mod):
    """The 60M-configuration cfg2 shape (structure table built per shard) sharded 4 ways and
    merged on the device, against the oracle's top-64 and count of the same range."""
    sw = W.config2(n_alpha=64, n_beta=64, b_list=[8, 64, 256], pipe_smax=3)
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    k, ns = 64, 4
    ohits, onf = osw.topk(0, n, k)
    recs = torch.zeros((ns, k + 1, 2), dtype=torch.int64, device=dev)
    for s in range(ns):
        ctx.topk_async(spec, 0, n, s, ns, k, recs[s].data_ptr(), recs[s, k].data_ptr(),
                       stream=torch.cuda.current_stream())
    out = torch.empty((k, 2), dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    ctx.merge_records(recs.data_ptr(), ns, k, out.data_ptr(), cnt.data_ptr(), stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    assert [int(v) for v in o[:, 0].astype(np.uint64)] == [h[0] for h in ohits]
    assert o[:, 1].view(np.float64).tolist() == [h[1] for h in ohits]
    assert int(cnt.item()) == onf


def test_config4_full_sweep_vs_oracle(dev, oracle_mod):
    """cfg4 (CosmoFlow 128^3 / 512^3 spatial + ds, 1.58e8 configurations) in full: the bench's
    launch (whole-sweep top-64 + count) against the oracle's whole-sweep reduction."""
    sw = W.config4()
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    hits, nf = ctx.topk(spec, 64, 0, n)
    ohits, onf = osw.topk(0, n, 64)
    assert nf == onf
    assert [h[0] for h in hits] == [h[0] for h in ohits]
    assert [h[1] for h in hits] == [h[1] for h in ohits]


def _golden_full(cfg):
    import json
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", f"full_cfg{cfg}.json")
    if not os.path.exists(p):
        pytest.skip(f"no whole-sweep oracle golden for cfg{cfg} (tools/golden_full.py {cfg})")
    return json.load(open(p))


@pytest.mark.parametrize("cfg", [2, 3, 5])
def test_full_sweep_vs_oracle_golden(dev, cfg):
    """Whole BASELINE sweep exactly as bench.py launches it (one top-64 + count call over
    [0, N)) against the oracle's whole-sweep top-64 and count, written offline by
    tools/golden_full.py from oracle/ alone."""
    g = _golden_full(cfg)
    sw = W.CONFIGS[cfg]()
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    n = ctx.sweep_size(spec)
    assert n == g["configs"] and sw.name == g["workload"]
    hits, nf = ctx.topk(spec, 64, 0, n)
    assert nf == g["n_feasible"]
    assert [h[0] for h in hits[:len(g["hits"])]] == [i for i, _ in g["hits"]]
    assert [h[1] for h in hits[:len(g["hits"])]] == [float.fromhex(k) for _, k in g["hits"]]


# ------------------------------------------------------------------ a9 compact mode
def gpu_compact(ctx, spec, first, count, dev, capacity=None):
    cap = count if capacity is None else capacity
    idx = torch.empty(max(1, cap), dtype=torch.int64, device=dev)
    t = torch.empty(max(1, cap), dtype=torch.float64, device=dev)
    m = torch.empty(max(1, cap), dtype=torch.float64, device=dev)
    nf = torch.zeros(1, dtype=torch.int64, device=dev)
    ctx.sweep_compact(spec, first, count, idx.data_ptr(), cap, nf.data_ptr(), t.data_ptr(), m.data_ptr(),
                      stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    n = int(nf.item())
    k = min(n, cap)
    return n, idx[:k].cpu().numpy().view(np.uint64), t[:k].cpu().numpy(), m[:k].cpu().numpy()


def check_compact(ctx, spec, osw, first, count, dev):
    """Compact output == the oracle's dense output filtered by its feasibility bits, in index order."""
    n, idx, t, m = gpu_compact(ctx, spec, first, count, dev)
    ot, om, obits, ors = osw.dense(first, count)
    feas = np.nonzero(ors == 0)[0]
    assert n == len(feas)
    assert np.array_equal(idx, (feas + first).astype(np.uint64))
    assert np.array_equal(t, ot[feas]) and np.array_equal(m, om[feas])
    return n


@pytest.mark.parametrize("seed", range(12))
def test_compact_random_corpus(dev, oracle_mod, seed):
    """Row a9 compact mode on random corpora (all families): whole range and ragged windows."""
    sw = corpus.random_sweep(seed)
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    check_compact(ctx, spec, osw, 0, n, dev)
    rng = random.Random(seed)
    for _ in range(3):
        a = rng.randrange(n)
        c = rng.randrange(n - a + 1)
        check_compact(ctx, spec, osw, a, c, dev)


@pytest.mark.parametrize("cfg,kw", [(2, dict(n_alpha=3, n_beta=5, b_list=[1, 7, 64, 256], pipe_smax=3)),
                                    (4, dict(n_alpha=2, n_beta=3))])
def test_compact_reduced_configs_and_capacity(dev, oracle_mod, cfg, kw):
    """Compact mode on reduced BASELINE configs (many tiles, several launches), plus a capacity
    smaller than the feasible count: the first `capacity` entries, and the full count."""
    sw = W.CONFIGS[cfg](**kw)
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    nf = check_compact(ctx, spec, osw, 0, n, dev)
    cap = max(1, nf // 3)
    n2, idx, t, _ = gpu_compact(ctx, spec, 0, n, dev, capacity=cap)
    ot, _, _, ors = osw.dense(0, n)
    feas = np.nonzero(ors == 0)[0][:cap]
    assert n2 == nf and np.array_equal(idx, feas.astype(np.uint64)) and np.array_equal(t, ot[feas])


@pytest.mark.parametrize("cfg", [2, 3, 5])
def test_compact_full_size_windows(dev, oracle_mod, cfg):
    """Compact mode at full BASELINE sizes: windows at random offsets against the oracle."""
    sw = W.CONFIGS[cfg]()
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    rng = random.Random(300 + cfg)
    for a in [0, n - 5000] + [rng.randrange(n - 5000) for _ in range(6)]:
        check_compact(ctx, spec, osw, a, rng.randrange(1000, 5000), dev)


@pytest.mark.parametrize("cfg", [3, 5])
def test_full_sweep_chunks_vs_oracle_golden(dev, cfg):
    """Whole-sweep oracle runs in progress (tools/golden_full.py checkpoints): every finished
    chunk of 2^30 consecutive configurations -- its top-64 and feasible count, oracle only --
    against the GPU's top-64 + count over the same range."""
    import json
    import os
    p = os.path.join(os.path.dirname(__file__), "golden", f"full_cfg{cfg}.chunks.jsonl")
    if not os.path.exists(p):
        pytest.skip(f"no chunk goldens for cfg{cfg}")
    sw = W.CONFIGS[cfg]()
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    n = ctx.sweep_size(spec)
    done = 0
    for ln in open(p):
        r = json.loads(ln)
        assert r["n"] == n
        hits, nf = ctx.topk(spec, 64, r["first"], r["count"])
        assert nf == r["n_feasible"]
        gh = r["hits"]
        assert [h[0] for h in hits[:len(gh)]] == [i for i, _ in gh]
        assert [h[1] for h in hits[:len(gh)]] == [float.fromhex(k) for _, k in gh]
        done += 1
    assert done > 0


# ------------------------------------------------------------------ f1: per-pattern parameters, contention
@pytest.mark.parametrize("cfg,kw", [(5, dict(s_max=3)), (2, dict(n_alpha=3, n_beta=32, b_list=[2, 64], pipe_smax=3)),
                                    (4, dict(n_alpha=2, n_beta=32)), (3, dict(n_alpha=2, n_beta=3))])
def test_p2p_scales_and_contention_all_paths(dev, oracle_mod, cfg, kw):
    """DESIGN.md Q40: point-to-point alpha/beta scales and the pd / ds
    contention coefficients through every evaluation path (mode-3 COMB pd, mode-0 slots,
    structure-free dense, mode-2 masks) against the oracle: whole-sweep top-64 + count,
    dense windows, and ragged windows."""
    import dataclasses
    sw = W.CONFIGS[cfg](**kw)
    sw.system = dataclasses.replace(sw.system, p2p_alpha_scale=2.5, p2p_beta_scale=1.75, phi_pd=2.0, phi_ds=3.0)
    if cfg == 3:   # a small mask sweep (VGG16's first 14 rows) for the mode-2 path
        from workloads import models as M
        vgg = M.vgg16()
        m = M.Model("vgg14", vgg.layers[:14], vgg.D, default_Ls=14)
        sw.models = [m]
        sw.subs = [W.SubSweep(W.PIPELINE, part_mode=W.PART_MASK, S=[4], b=[64]),
                   W.SubSweep(W.PIPELINE, part_mode=W.PART_MASK, S=[2], b=[8, 64], alpha=sw.subs[0].alpha[:1],
                              beta=sw.subs[0].beta[:2])]
    ctx = P.Context(0)
    spec = ctx.prepare(sw)
    osw = oracle_mod.OracleSweep(sw)
    n = osw.size()
    check_topk(ctx, spec, osw, 0, n, 64)
    rng = random.Random(cfg)
    for _ in range(4):
        a = rng.randrange(n)
        c = min(n - a, rng.randrange(1, 200_000))
        check_topk(ctx, spec, osw, a, c, 16)
        c = min(c, 20_000)
        assert check_dense(ctx, spec, osw, a, c, dev) == 0


def test_repeated_and_concurrent_calls_identical(dev):
    """Race surrogate (compute-sanitizer is unavailable on the pool): a sweep whose top-k uses
    the fused two-level merge (many CTA lists, last-block ticket) and the shared admission
    bound gives bit-identical hits and counts over 20 repeated calls, and when two contexts
    run it at once on two streams."""
    sw = W.config2(n_alpha=8, n_beta=64, b_list=[2, 32, 256], pipe_smax=3)
    ctxs = [P.Context(0), P.Context(0)]
    specs = [c.prepare(sw) for c in ctxs]
    n = ctxs[0].sweep_size(specs[0])
    ref, rnf = ctxs[0].topk(specs[0], 64)
    for _ in range(20):
        hits, nf = ctxs[0].topk(specs[0], 64)
        assert hits == ref and nf == rnf
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    outs = [(torch.empty((64, 2), dtype=torch.int64, device=dev), torch.zeros(1, dtype=torch.int64, device=dev))
            for _ in range(2)]
    for rep in range(5):
        for c, sp, st, (h, cnt) in zip(ctxs, specs, streams, outs):
            c.topk_async(sp, 0, n, 0, 1, 64, h.data_ptr(), cnt.data_ptr(), stream=st)
        torch.cuda.synchronize()
        for h, cnt in outs:
            got = [int(v) % (1 << 64) for v in h.cpu().numpy()[:, 0]]
            assert got == [x[0] for x in ref] and int(cnt.item()) == rnf


def test_calibrated_system_sweep_vs_oracle(dev, oracle_mod):
    """f2: a system assembled by workloads.calibrate from fitted parameters --
    ring-form tiers per group size, the tree form and its crossing as tree_threshold_B, the
    point-to-point fit as p2p scales (Q40), measured per-layer times as the layer table -- swept
    on the GPU (cfg2 shape, cfg5 shape) against the oracle.  The timings are synthetic Hockney
    samples with noise (the fits and the gloo measurement path are tested on CPU)."""
    from workloads import calibrate as CAL
    from workloads import models as M
    rng = random.Random(3)
    sizes = [1 << e for e in range(10, 29, 2)]
    tiers = []
    for p, (a, b) in ((2, (15e-6, 1 / 490e9)), (4, (6e-6, 1 / 580e9)), (1024, (4e-5, 1 / 25e9))):
        t = [2 * (p - 1) * (a + m / p * b) * (1 + rng.uniform(-0.03, 0.03)) for m in sizes]
        fa, fb, _ = CAL.fit_allreduce(p, sizes, t)
        tiers.append({"p": p, "alpha_s": fa, "beta_s_per_B": fb})
    lg = 2
    tt = [2 * (lg + 2) * (3e-6 + m / 4 * (1 / 90e9)) for m in sizes]
    tree = CAL.fit_allreduce_tree(4, sizes, tt, 2)
    thr = CAL.tree_threshold(4, (tiers[1]["alpha_s"], tiers[1]["beta_s_per_B"]), tree[:2], 2)
    tp = [30e-6 + m / 12e9 for m in sizes]
    ka, kb = CAL.p2p_scales(tiers[1], CAL.fit_p2p(sizes, tp)[:2])
    sysm = CAL.system_from_tiers(tiers, flops_per_s=1e15, hbm_bytes=180 * W.GiB, tree_threshold=thr,
                                 tree_chunks=2, p2p_alpha_scale=ka, p2p_beta_scale=kb, phi_pd=2.0)
    r50 = M.resnet(50)
    times = [(1e-4 * (i % 7 + 1), 2e-4 * (i % 5 + 1)) if r.kind == M.CONV else None for i, r in enumerate(r50.layers)]
    em = CAL.empirical_model(r50, times, 1e15)
    for sw in (W.config2(n_alpha=1, n_beta=1, b_list=[8, 64], pipe_smax=3), W.config5(s_max=3)):
        sw.system = sysm
        if sw.models[0].name.startswith("resnet50"):
            sw.models = [em]
        for sb in sw.subs:
            sb.alpha, sb.beta = [], []
        ctx = P.Context(0)
        spec = ctx.prepare(sw)
        osw = oracle_mod.OracleSweep(sw)
        n = osw.size()
        check_topk(ctx, spec, osw, 0, n, 64)
        c = min(n, 200_000)
        assert check_dense(ctx, spec, osw, 0, c, dev) == 0
