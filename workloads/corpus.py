"""Seeded random corpora for property and parity tests (input generator only).

Every instance is a function of (seed); no cost-model arithmetic here.  Seeds follow
SURVEY.md §8(d): 0x5EED + i.
"""
from __future__ import annotations

import random

from . import models as M
from . import sweeps as W

SEED0 = 0x5EED


def random_layer(rng: random.Random, ndim: int, C: int, X: tuple) -> M.Layer:
    k = rng.random()
    if k < 0.55:
        K = rng.choice([1, 3, 5, 7])
        F = rng.choice([1, 2, 3, 4, 8, 16, 32])
        stride = rng.choice([1, 1, 2])
        pad = K // 2
        Xs = tuple(max(x, K) for x in X)
        return M.make_conv("c", C, F, Xs, K, stride=stride, pad=pad, bias=rng.random() < 0.5)
    if k < 0.70:
        K = rng.choice([2, 3])
        Xs = tuple(max(x, K) for x in X)
        return M.make_pool("p", C, Xs, K, K, ceil_mode=rng.random() < 0.5)
    if k < 0.85:
        return M.make_elem("e", C, X, kind=rng.choice([M.ELEM, M.NORM]))
    F = rng.choice([1, 2, 5, 10, 64])
    return M.make_fc("f", C, F, X, bias=True)


def random_model(seed: int, G: int | None = None) -> M.Model:
    rng = random.Random(seed)
    ndim = rng.choice([1, 2, 2, 3])
    G = G if G is not None else rng.randint(1, 14)
    C = rng.choice([1, 3, 4, 8])
    X = tuple(rng.choice([4, 7, 8, 16, 33]) for _ in range(ndim))
    rows = []
    for _ in range(G):
        r = random_layer(rng, ndim, C, X)
        rows.append(r)
        C = r.F
        X = tuple(r.Y[:ndim])
    D = rng.choice([1000, 1281167, 1584, 50000])
    return M.Model(f"rand{seed}", rows, D, default_Ls=rng.randint(0, G))


def random_system(seed: int) -> W.System:
    rng = random.Random(seed ^ 0xABCDEF)
    nt = rng.randint(1, 3)
    pes = sorted(rng.sample([2, 4, 8, 16, 64, 256, 1024], nt))
    tiers = [W.Tier(pe, rng.uniform(1e-7, 1e-4), 1.0 / rng.uniform(1e9, 1e12)) for pe in pes]
    sysd = W.System(tiers=tiers,
                    flops_per_s=rng.choice([1e12, 15.7e12, 37e12, 3.3e11]),
                    hbm_bytes=rng.choice([2.0 ** 20, 2.0 ** 26, 16 * W.GiB]),
                    delta=rng.choice([2, 4, 8]),
                    gamma=rng.choice([1.0, 0.5, 0.37]),
                    phi_df=rng.choice([1.0, 2.0, 3.0]),
                    tree_threshold=rng.choice([0.0, 0.0, 4096.0, 1e6]),
                    tree_chunks=rng.choice([1, 2, 4]),
                    filter_rs=rng.choice([0, 1]))
    # f1 parameters (Q40), drawn after the others so earlier draws keep their values
    if rng.random() < 0.5:
        sysd.p2p_alpha_scale = rng.choice([1.0, 3.0, 0.7])
        sysd.p2p_beta_scale = rng.choice([1.0, 2.5, 1.3])
    if rng.random() < 0.5:
        sysd.phi_pd = rng.choice([1.0, 2.0, 3.0])
        sysd.phi_ds = rng.choice([1.0, 2.0, 4.0])
    return sysd


def random_sweep(seed: int, max_list: int = 3) -> W.Sweep:
    """Small sweep touching every family; sizes stay in the thousands."""
    rng = random.Random(seed + 7)
    models = [random_model(seed), random_model(seed + 1000)]
    sys = random_system(seed)
    nt = len(sys.tiers)

    def some(vals, n=None):
        n = n or rng.randint(1, max_list)
        return [rng.choice(vals) for _ in range(n)]

    def ab():
        na, nb = rng.randint(1, max_list), rng.randint(1, max_list)
        A = [[rng.uniform(1e-7, 1e-4) for _ in range(nt)] for _ in range(na)]
        B = [[1.0 / rng.uniform(1e9, 1e12) for _ in range(nt)] for _ in range(nb)]
        return A, B

    subs = []
    fams = list(range(13))
    rng.shuffle(fams)
    for fam in fams:
        mi = rng.randint(0, 1)
        m = models[mi]
        A, B = ab() if rng.random() < 0.8 else ([], [])
        kw = dict(model=mi, alpha=A, beta=B,
                  b=some([1, 2, 3, 4, 8, 16, 32]),
                  cap=some([2.0 ** 18, 2.0 ** 24, 2.0 ** 30]) if rng.random() < 0.5 else [],
                  flops=some([1e12, 2.5e12]) if rng.random() < 0.5 else [])
        if fam in (W.DATA, W.FILTER, W.CHANNEL, W.DATA_LW):
            kw["dims"] = [(p, 1, 1, 1) for p in some([1, 2, 3, 4, 8, 16, 64, 1024])]
        elif fam == W.DF:
            kw["dims"] = [(rng.choice([1, 2, 3, 4]), rng.choice([1, 2, 4, 5]), 1, 1) for _ in range(rng.randint(1, 3))]
        elif fam in W.SPATIAL_FAMILIES:
            kw["dims"] = [(rng.choice([1, 2, 3]) if fam == W.DS else 1,
                           rng.choice([1, 2, 3, 4]), rng.choice([1, 2, 4]), rng.choice([1, 1, 2]))
                          for _ in range(rng.randint(1, 3))]
            kw["Ls"] = some(list(range(1 if fam == W.SPATIAL_AG else 0, m.G + 2)))
        elif fam == W.PD:
            kw["dims"] = [(p, 1, 1, 1) for p in some([1, 2, 3, 4, 8])]
        if fam in W.PIPE_FAMILIES:
            kw["S"] = some([1, 2, 3, 4, 8])
            smax_fam = 8 if fam == W.GPIPE else m.G     # GPipe: at most 8 stages (GPU limit)
            if m.G <= min(10, smax_fam) and rng.random() < 0.5:
                kw["part_mode"] = W.PART_MASK
            else:
                kw["part_mode"] = W.PART_COMB
                smin = rng.randint(1, min(m.G, smax_fam))
                kw["s_min"] = smin
                kw["s_max"] = rng.randint(smin, min(m.G, smin + 3, smax_fam))
        subs.append(W.SubSweep(fam, **kw))
    # per-layer strategy (appended last, so the other sub-sweeps keep their seeds): on the
    # model with fewer COMM rows, when it has at most 7 (<= 128 assignments)
    nc = [sum(1 for r in m.layers if r.flags & M.FLAG_COMM) for m in models]
    mi = 0 if nc[0] <= nc[1] else 1
    if nc[mi] <= 7:
        A, B = ab()
        subs.append(W.SubSweep(W.LAYERWISE, model=mi, part_mode=W.PART_MASK, alpha=A, beta=B,
                               b=some([1, 2, 3, 8, 32]),
                               cap=some([2.0 ** 18, 2.0 ** 24, 2.0 ** 30]) if rng.random() < 0.5 else [],
                               dims=[(p, 1, 1, 1) for p in some([1, 2, 3, 4, 16, 1024])]))
    return W.Sweep(models, sys, subs, f"rand{seed}")
