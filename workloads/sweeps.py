"""Synthetic sweep specifications shaped like BASELINE.json's five configs.

INPUT GENERATOR ONLY: value lists (p, splits, batches, alpha/beta grids, capacities,
stage-count ranges).  No cost-model arithmetic lives here.  The canonical index order
the lists define (slow -> fast: cap, R, b, partition, S, dims, Ls, alpha, beta) is
documented in DESIGN.md §3 and implemented independently by the oracle and the CUDA
decoder.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import models as M

# Strategy families (Table 2 rows P:455-516)
SERIAL, DATA, SPATIAL, FILTER, CHANNEL, DF, DS, PIPELINE, LAYERPURE, PD = range(10)
# SURVEY §8(f) "next" rows: spatial prefix + Allgather, GPipe schedule
SPATIAL_AG, GPIPE = 10, 11
# per-layer gradient messages with per-message ring / tree dispatch
DATA_LW = 12
# per-layer heterogeneous strategy, one data / filter bit per COMM row
LAYERWISE = 13
FAMILY_NAMES = ["serial", "data", "spatial", "filter", "channel", "df", "ds",
                "pipeline", "layerpure", "pd", "spatial_ag", "gpipe", "data_lw", "layerwise"]
PIPE_FAMILIES = (PIPELINE, LAYERPURE, PD, GPIPE)
SPATIAL_FAMILIES = (SPATIAL, DS, SPATIAL_AG)

# Partition enumeration modes
PART_NONE, PART_COMB, PART_MASK = 0, 1, 2

GiB = float(1 << 30)


@dataclass
class Tier:
    max_pes: int
    alpha: float      # seconds
    beta: float       # seconds per byte


@dataclass
class System:
    tiers: list
    flops_per_s: float = 15.7e12
    hbm_bytes: float = 16 * GiB
    delta: int = 4
    gamma: float = 1.0
    phi_df: float = 2.0
    tree_threshold: float = 0.0     # bytes; 0 => ring everywhere (Table 2 literal)
    tree_chunks: int = 1
    filter_rs: int = 0              # 1: filter/channel backward exchange as Reduce-Scatter (P:355 fn)
    # point-to-point patterns (halo, pipeline sends) on their own
    # alpha/beta (the tier's times these scales, e.g. MPI vs NCCL); contention on
    # the pd stage Allreduces and the ds reduce-to-leader.  1.0 = Table 2 literal.
    p2p_alpha_scale: float = 1.0
    p2p_beta_scale: float = 1.0
    phi_pd: float = 1.0
    phi_ds: float = 1.0


@dataclass
class SubSweep:
    family: int
    model: int = 0
    cap: list = field(default_factory=list)        # empty => system.hbm_bytes
    flops: list = field(default_factory=list)      # empty => system.flops_per_s
    b: list = field(default_factory=lambda: [1])
    part_mode: int = PART_NONE
    s_min: int = 1
    s_max: int = 1
    S: list = field(default_factory=list)          # empty => [1]
    dims: list = field(default_factory=list)       # empty => [(1,1,1,1)]
    Ls: list = field(default_factory=list)         # spatial prefix lengths; empty => [0]
    alpha: list = field(default_factory=list)      # rows of n_tiers alphas; empty => system tiers
    beta: list = field(default_factory=list)       # rows of n_tiers betas;  empty => system tiers


@dataclass
class Sweep:
    models: list          # list[M.Model]
    system: System
    subs: list            # list[SubSweep]
    name: str = ""


# ----------------------------------------------------------------- value-list helpers
def pow2(lo_exp: int, hi_exp: int):
    return [1 << e for e in range(lo_exp, hi_exp + 1)]


def pairs_pow2(max_exp: int):
    """(p1, p2) with p1*p2 = 2^k, k <= max_exp, p1 slowest."""
    out = []
    for e1 in range(max_exp + 1):
        for e2 in range(max_exp + 1 - e1):
            out.append((1 << e1, 1 << e2, 1, 1))
    return out


def splits_pow2(max_exp: int, ndim: int, with_p1: bool):
    """Ordered factorizations (p1;pw,ph,pd) of powers of two with total <= 2^max_exp,
    p1 slowest, then pw, ph, pd (lexicographic)."""
    out = []
    r1 = range(max_exp + 1) if with_p1 else [0]
    for e1 in r1:
        for ew in range(max_exp + 1 - e1):
            for eh in range(max_exp + 1 - e1 - ew):
                if ndim == 3:
                    for ed in range(max_exp + 1 - e1 - ew - eh):
                        out.append((1 << e1, 1 << ew, 1 << eh, 1 << ed))
                else:
                    out.append((1 << e1, 1 << ew, 1 << eh, 1))
    return out


def ab_grid(alphas, betas, n_tiers=2):
    """Tier-expanded alpha/beta rows: (alpha_intra, alpha_inter) = (a, 4a);
    (beta_intra, beta_inter) = (b, 2b)  (SURVEY §8(d) base system)."""
    if n_tiers == 1:
        return [[float(a)] for a in alphas], [[float(b)] for b in betas]
    A = [[float(a), float(a) * 4.0] for a in alphas]
    B = [[float(b), float(b) * 2.0] for b in betas]
    return A, B


def two_tier_system(**kw):
    # {8 PEs: NVLink-class; 1024 PEs: network-class}
    return System(tiers=[Tier(8, 2e-6, 1.0 / 150e9), Tier(1024, 8e-6, 1.0 / 75e9)], **kw)


# ----------------------------------------------------------------- BASELINE configs
def config1() -> Sweep:
    """ResNet-50, data parallelism only, p in 2^0..2^10, b in {32,64,128} (33 configs)."""
    m = M.resnet(50)
    sys = System(tiers=[Tier(1024, 5e-6, 8e-11)], flops_per_s=15.7e12, hbm_bytes=16 * GiB)
    sub = SubSweep(DATA, b=[32, 64, 128], dims=[(p, 1, 1, 1) for p in pow2(0, 10)])
    # canonical order is b slow, dims fast; config 1 lists p slow, b fast -> one subsweep per p
    subs = [SubSweep(DATA, b=[32, 64, 128], dims=[(p, 1, 1, 1)]) for p in pow2(0, 10)]
    del sub
    return Sweep([m], sys, subs, "cfg1_resnet50_data")


def config2(n_alpha=64, n_beta=64, b_list=None, pipe_smax=4, S_list=(1, 2, 4, 8)) -> Sweep:
    """ResNet-50, six strategies (+ds) x alpha/beta grid."""
    m = M.resnet(50)
    sys = two_tier_system(flops_per_s=37e12, hbm_bytes=16 * GiB)
    A, B = ab_grid(np.logspace(-7, -4, n_alpha), 1.0 / np.logspace(9, 12, n_beta))
    b = list(b_list) if b_list is not None else pow2(0, 8)
    common = dict(b=b, alpha=A, beta=B)
    ps = [(p, 1, 1, 1) for p in pow2(0, 10)]
    subs = [
        SubSweep(DATA, dims=ps, **common),
        SubSweep(SPATIAL, dims=splits_pow2(10, 2, False), Ls=[m.default_Ls], **common),
        SubSweep(FILTER, dims=ps, **common),
        SubSweep(CHANNEL, dims=ps, **common),
        SubSweep(DF, dims=pairs_pow2(10), **common),
        SubSweep(DS, dims=splits_pow2(10, 2, True), Ls=[m.default_Ls], **common),
        SubSweep(PIPELINE, part_mode=PART_COMB, s_min=1, s_max=pipe_smax, S=list(S_list), **common),
    ]
    return Sweep([m], sys, subs, "cfg2_resnet50_six_strategies_ab")


def config3(n_alpha=64, n_beta=64, mask_model=None) -> Sweep:
    """VGG16: (i) filter/channel/df x alpha/beta; (ii) all 2^37 contiguous pipeline
    partitions (mask mode), S=4, b=64, one system."""
    m = M.vgg16()
    sys = two_tier_system(flops_per_s=37e12, hbm_bytes=16 * GiB)
    A, B = ab_grid(np.logspace(-7, -4, n_alpha), 1.0 / np.logspace(9, 12, n_beta))
    ps = [(p, 1, 1, 1) for p in pow2(0, 10)]
    common = dict(b=[16, 32, 64], alpha=A, beta=B)
    subs = [
        SubSweep(FILTER, dims=ps, **common),
        SubSweep(CHANNEL, dims=ps, **common),
        SubSweep(DF, dims=pairs_pow2(10), **common),
        SubSweep(PIPELINE, part_mode=PART_MASK, S=[4], b=[64]),
    ]
    return Sweep([m], sys, subs, "cfg3_vgg16_fc_df_pipeline_masks")


def config4(n_alpha=32, n_beta=32) -> Sweep:
    """CosmoFlow 128^3 and 512^3: spatial (3D splits) and ds, prefix L_s, b, alpha/beta, cap."""
    ms = [M.cosmoflow(128), M.cosmoflow(512)]
    sys = two_tier_system(flops_per_s=37e12, hbm_bytes=16 * GiB)
    A, B = ab_grid(np.logspace(-7, -4, n_alpha), 1.0 / np.logspace(9, 12, n_beta))
    caps = [16 * GiB, 32 * GiB, 80 * GiB, 180 * GiB]
    subs = []
    for mi in range(2):
        common = dict(model=mi, cap=caps, b=[1, 2, 4], Ls=[3, 6, 9, 12, 15], alpha=A, beta=B)
        subs.append(SubSweep(SPATIAL, dims=splits_pow2(10, 3, False), **common))
        subs.append(SubSweep(DS, dims=splits_pow2(10, 3, True), **common))
    return Sweep(ms, sys, subs, "cfg4_cosmoflow_spatial_ds")


def config5(s_max=6) -> Sweep:
    """ResNet-152 pipeline+data: all contiguous partitions with s <= 6 (combination mode)
    x S in {1,2,4,8} x p_d in 2^0..2^7 x b=32 x 2x2 system grid (~8.1e10 configs)."""
    m = M.resnet(152)
    sys = two_tier_system(flops_per_s=37e12, hbm_bytes=80 * GiB)
    A, B = ab_grid([2e-6, 1e-5], [1.0 / 150e9, 1.0 / 25e9])
    subs = [SubSweep(PD, part_mode=PART_COMB, s_min=1, s_max=s_max, S=[1, 2, 4, 8],
                     dims=[(p, 1, 1, 1) for p in pow2(0, 7)], b=[32], alpha=A, beta=B)]
    return Sweep([m], sys, subs, "cfg5_resnet152_pd")


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


# ----------------------------------------------------------------- SURVEY §8(f) "next" rows
def next_gpipe(n_alpha=64, n_beta=64, b_list=None, s_max=4, S_list=(1, 2, 4, 8)) -> Sweep:
    """ResNet-50 partitions timed by the GPipe schedule (family GPIPE, Q36): the
    shape of config 2's pipeline sub-sweep (s <= 4 exhaustive, S, b, 64x64 alpha/beta)."""
    m = M.resnet(50)
    sys = two_tier_system(flops_per_s=37e12, hbm_bytes=16 * GiB)
    A, B = ab_grid(np.logspace(-7, -4, n_alpha), 1.0 / np.logspace(9, 12, n_beta))
    b = list(b_list) if b_list is not None else pow2(0, 8)
    subs = [SubSweep(GPIPE, part_mode=PART_COMB, s_min=1, s_max=s_max, S=list(S_list), b=b, alpha=A, beta=B)]
    return Sweep([m], sys, subs, "next_gpipe_resnet50")


def next_spatial_ag(n_alpha=64, n_beta=64) -> Sweep:
    """Spatial prefix + Allgather (family SPATIAL_AG, Q35): ResNet-50 2D
    splits with prefixes ending at each stage boundary, CosmoFlow 128^3 / 512^3 3D splits
    with the config 4 prefixes, capacities and batches."""
    r50 = M.resnet(50)
    ms = [r50, M.cosmoflow(128), M.cosmoflow(512)]
    sys = two_tier_system(flops_per_s=37e12, hbm_bytes=16 * GiB)
    A, B = ab_grid(np.logspace(-7, -4, n_alpha), 1.0 / np.logspace(9, 12, n_beta))
    caps = [16 * GiB, 32 * GiB, 80 * GiB, 180 * GiB]
    subs = [SubSweep(SPATIAL_AG, model=0, dims=splits_pow2(10, 2, False), b=pow2(0, 8),
                     Ls=[1, 10, 22, 40, r50.default_Ls], alpha=A, beta=B)]
    for mi in (1, 2):
        subs.append(SubSweep(SPATIAL_AG, model=mi, cap=caps, b=[1, 2, 4], dims=splits_pow2(10, 3, False),
                             Ls=[3, 6, 9, 12, 15], alpha=A, beta=B))
    return Sweep(ms, sys, subs, "next_spatial_ag")


def next_data_lw(n_alpha=256, n_beta=256) -> Sweep:
    """Per-layer gradient messages with per-message ring / tree dispatch (family DATA_LW,
    P:552, Q37): ResNet-50, ResNet-152 and VGG16, p in 2^0..2^10, b in
    2^0..2^8, a 256 x 256 alpha/beta grid; messages below 1 MiB use the 4-chunk tree form."""
    ms = [M.resnet(50), M.resnet(152), M.vgg16()]
    sys = two_tier_system(flops_per_s=37e12, hbm_bytes=80 * GiB, tree_threshold=float(1 << 20), tree_chunks=4)
    A, B = ab_grid(np.logspace(-7, -4, n_alpha), 1.0 / np.logspace(9, 12, n_beta))
    subs = [SubSweep(DATA_LW, model=mi, dims=[(p, 1, 1, 1) for p in pow2(0, 10)], b=pow2(0, 8), alpha=A, beta=B)
            for mi in range(3)]
    return Sweep(ms, sys, subs, "next_data_lw")


def next_layerwise(n_alpha=32, n_beta=32) -> Sweep:
    """Per-layer heterogeneous strategy (family LAYERWISE, Q39): every
    one of VGG16's 16 weighted layers data- or filter-parallel (2^16 assignments, the paper's
    "fully connected layer ... not spatially parallelized" generalised), p in 2^0..2^10, b in
    {8, 32, 128}, a 32 x 32 alpha/beta grid; and the CosmoFlow-like 128^3 net's 8 weighted
    layers (2^8 assignments) with capacities."""
    vgg, cf = M.vgg16(), M.cosmoflow(128)
    sys = two_tier_system(flops_per_s=37e12, hbm_bytes=16 * GiB)
    A, B = ab_grid(np.logspace(-7, -4, n_alpha), 1.0 / np.logspace(9, 12, n_beta))
    ps = [(p, 1, 1, 1) for p in pow2(0, 10)]
    subs = [SubSweep(LAYERWISE, model=0, part_mode=PART_MASK, dims=ps, b=[8, 32, 128], alpha=A, beta=B),
            SubSweep(LAYERWISE, model=1, part_mode=PART_MASK, dims=ps, b=[1, 2, 4],
                     cap=[16 * GiB, 80 * GiB, 180 * GiB], alpha=A, beta=B)]
    return Sweep([vgg, cf], sys, subs, "next_layerwise_vgg16_cosmoflow")


NEXT = {"gpipe": next_gpipe, "spatial_ag": next_spatial_ag, "data_lw": next_data_lw, "layerwise": next_layerwise}
