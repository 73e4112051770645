"""Pin the CPU oracle to things other than itself (CPU only, -m "not gpu").

Sources of truth: worked examples re-derived from the paper's equations
(tests/golden/spec_examples.json), values the paper prints (tests/golden/paper_pins.json),
brute-force simulators and an exact-rational evaluator (tests/brute.py), closed-form
invariants, and degenerate identities (SPEC S:437 / S:611-612).
"""
from __future__ import annotations

import itertools
import json
import math
import os
import random
from fractions import Fraction as Fr

import pytest

import brute
import toys
from workloads import corpus
from workloads import models as M
from workloads import sweeps as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")
EX = json.load(open(os.path.join(GOLD, "spec_examples.json")))
PIN = json.load(open(os.path.join(GOLD, "paper_pins.json")))


def _one(O, model, system, sub, idx=0, fold=False):
    sw = toys.sweep(model, system, [sub])
    o = O.OracleSweep(sw)
    return o.explain(idx, fold=fold)


def _rel(a, b):
    a, b = float(a), float(b)
    if a == b:
        return 0.0
    return abs(a - b) / max(abs(a), abs(b))


# ------------------------------------------------------------ collective primitives
def test_allreduce_ring_example(oracle_mod):
    e = EX["allreduce_ring"]
    # data(p) GE = AR(p, delta*W): a single weighted row with w = m, delta = 1
    m = toys.model([toys.row(w=e["m"])])
    pr = _one(oracle_mod, m, toys.system(alpha=e["alpha"], beta=e["beta"]),
              W.SubSweep(W.DATA, b=[1], dims=[(e["p"], 1, 1, 1)]))
    assert pr.t_ge == e["expect"]


def test_allgather_ring_example(oracle_mod):
    # filter(p) Allgather phase = (p-1)(NC alpha + (B delta YC / p) beta): choose NC = 1,
    # B*YC/p = m_seg  ->  rows: one comm row with y = m_seg * p, then a last comm row.
    e = EX["allgather_ring"]
    p = e["p"]
    m = toys.model([toys.row(y=e["m_seg"] * p, F=64), toys.row(F=64)])
    pr = _one(oracle_mod, m, toys.system(alpha=e["alpha"], beta=e["beta"]),
              W.SubSweep(W.FILTER, b=[1], dims=[(p, 1, 1, 1)]))
    assert pr.t_fb_ag == e["expect"]
    assert pr.t_fb_ar == 2 * e["expect"]


@pytest.mark.parametrize("case", EX["allreduce_tree"]["cases"])
def test_allreduce_tree_examples(oracle_mod, case):
    p, k, a, b, mbytes, expect = case
    m = toys.model([toys.row(w=mbytes)])
    sysd = toys.system(alpha=a, beta=b, tree_threshold=1e9, tree_chunks=k)
    pr = _one(oracle_mod, m, sysd, W.SubSweep(W.DATA, b=[1], dims=[(p, 1, 1, 1)]))
    assert pr.t_ge == expect


def test_reduce_to_leader_and_ds_ge(oracle_mod):
    e = EX["ds_ge_iter"]
    # ds(p1; p2,1,1) GE = RL(p2, dW) + AR(p1, dW); one 1x1 row so the halo is latency-only
    m = toys.model([toys.row(w=e["dW"], X=(64, 1, 1), Y=(64, 1, 1))], Ls=0)
    pr = _one(oracle_mod, m, toys.system(alpha=e["alpha"], beta=e["beta"]),
              W.SubSweep(W.DS, b=[1], dims=[(e["p1"], e["p2"], 1, 1)], Ls=[0]))
    assert pr.t_ge == e["expect"]
    r = EX["reduce_to_leader"]
    pr1 = _one(oracle_mod, toys.model([toys.row(w=r["m"], X=(64, 1, 1))], Ls=0),
               toys.system(alpha=r["alpha"], beta=r["beta"]),
               W.SubSweep(W.DS, b=[1], dims=[(1, r["p"], 1, 1)], Ls=[0]))
    assert pr1.t_ge == r["expect"]


@pytest.mark.parametrize("p", [2, 3, 4, 5, 8, 13])
@pytest.mark.parametrize("mbytes", [1, 8, 1000, 123457])
def test_allreduce_matches_ring_simulation(oracle_mod, p, mbytes):
    a, b = 3e-6, 1.0 / 7e9
    t_sim, acc = brute.ring_allreduce_sim(p, mbytes, Fr(a), Fr(b))
    col = [sum((i + 1) * 1000 + c for i in range(p)) for c in range(p)]
    assert all(row == col for row in acc)          # the simulated ring really reduces
    pr = _one(oracle_mod, toys.model([toys.row(w=mbytes)]), toys.system(alpha=a, beta=b),
              W.SubSweep(W.DATA, b=[1], dims=[(p, 1, 1, 1)]))
    assert _rel(pr.t_ge, t_sim) <= 4e-16


@pytest.mark.parametrize("p", [2, 3, 4, 7, 16])
def test_allgather_matches_ring_simulation(oracle_mod, p):
    a, b = 2e-6, 1.0 / 3e9
    y = 777 * p
    t_sim = brute.ring_allgather_sim(p, Fr(y, p), Fr(a), Fr(b))
    m = toys.model([toys.row(y=y, F=64), toys.row(F=64)])
    pr = _one(oracle_mod, m, toys.system(alpha=a, beta=b), W.SubSweep(W.FILTER, b=[1], dims=[(p, 1, 1, 1)]))
    assert _rel(pr.t_fb_ag, t_sim) <= 4e-16


def test_no_comm_at_p1_and_monotone(oracle_mod):
    # north_star invariants: no communication term at p = 1; costs monotone in message size
    base = toys.system(alpha=1e-5, beta=1e-9)
    for fam in (W.DATA, W.FILTER, W.CHANNEL, W.SPATIAL):
        m = toys.model([toys.row(w=100, y=50, X=(8, 8, 1), Y=(8, 8, 1), K=(3, 3, 1), C=4, F=4)])
        pr = _one(oracle_mod, m, base, W.SubSweep(fam, b=[2], dims=[(1, 1, 1, 1)], Ls=[1]))
        assert pr.t_ge == pr.t_fb_ag == pr.t_fb_ar == pr.t_halo == pr.t_p2p == 0.0
    prev = -1.0
    for w in [1, 10, 1000, 10 ** 6, 10 ** 9]:
        pr = _one(oracle_mod, toys.model([toys.row(w=w)]), base, W.SubSweep(W.DATA, b=[1], dims=[(8, 1, 1, 1)]))
        assert pr.t_ge > prev
        prev = pr.t_ge


def test_allreduce_bandwidth_asymptote(oracle_mod):
    # S:203 / north_star: AR(p,m)/m -> 2(p-1)/p beta; at m = 1 GB within 1%
    beta = 1e-10
    for p in (2, 8, 64, 1024):
        pr = _one(oracle_mod, toys.model([toys.row(w=10 ** 9)]), toys.system(alpha=1e-7, beta=beta),
                  W.SubSweep(W.DATA, b=[1], dims=[(p, 1, 1, 1)]))
        ratio = pr.t_ge / 1e9
        assert abs(ratio / (2 * (p - 1) / p * beta) - 1) < 0.01


def test_contention_phi_doubles_beta_part(oracle_mod):
    # doubling phi doubles only the beta contribution (df inter-group GE)
    m = toys.model([toys.row(w=4096, y=8, F=64), toys.row(F=64)])
    ge = {}
    for phi in (1.0, 2.0):
        for a in (0.0, 1e-5):
            pr = _one(oracle_mod, m, toys.system(alpha=a, beta=1e-9, phi=phi),
                      W.SubSweep(W.DF, b=[1], dims=[(4, 2, 1, 1)]))
            ge[(phi, a)] = pr.t_ge
    beta1 = ge[(1.0, 0.0)]
    assert ge[(2.0, 0.0)] == 2 * beta1
    assert _rel(ge[(2.0, 1e-5)] - ge[(1.0, 1e-5)], beta1) < 1e-12


def test_weak_scaling_ge_ratio(oracle_mod):
    e = EX["weak_scaling_ratio"]
    m = toys.model([toys.row(w=10 ** 8, fw=10, bw=20, wu=7)], D=10 ** 6)
    out = {}
    for p in (e["p_lo"], e["p_hi"]):
        out[p] = _one(oracle_mod, m, toys.system(alpha=0.0, beta=1e-9),
                      W.SubSweep(W.DATA, b=[4], dims=[(p, 1, 1, 1)]))
    assert abs(out[e["p_hi"]].t_ge / out[e["p_lo"]].t_ge / e["expect"] - 1) <= 1e-12
    # weak scaling: per-PE compute independent of p when B = b p
    assert out[e["p_hi"]].t_comp == out[e["p_lo"]].t_comp


# ------------------------------------------------------------ Table 2 rows: worked examples
def test_serial_examples(oracle_mod):
    e = EX["serial_comp_epoch"]
    m = toys.model([toys.row(fw=e["FW"], bw=e["BW"], wu=e["WU"])], D=e["D"])
    pr = _one(oracle_mod, m, toys.system(R=1.0), W.SubSweep(W.SERIAL, b=[e["B"]]))
    assert pr.t_comp * pr.I == e["expect"]
    e = EX["serial_mem"]
    m = toys.model([toys.row(x=e["x"], y=e["y"], w=e["w"], bi=e["bi"])])
    pr = _one(oracle_mod, m, toys.system(delta=e["delta"], gamma=e["gamma"]), W.SubSweep(W.SERIAL, b=[e["B"]]))
    assert pr.mem == e["expect"]


def test_data_comp_example(oracle_mod):
    e = EX["data_comp_epoch"]
    m = toys.model([toys.row(fw=e["FW"], bw=e["BW"], wu=e["WU"])], D=e["D"])
    pr = _one(oracle_mod, m, toys.system(R=1.0), W.SubSweep(W.DATA, b=[e["B"] // e["p"]], dims=[(e["p"], 1, 1, 1)]))
    assert pr.B == e["B"]
    assert pr.t_comp * pr.I == e["expect"]


def test_halo_elements_examples(oracle_mod):
    e = EX["halo_elements"]
    r = M.make_conv("c", e["C"], e["C"], tuple(e["X"]), e["K"], stride=1, pad=1)
    for pw, expect in e["cases"]:
        assert oracle_mod.halo_elements(r, (pw, 1, 1), 0) == expect
        assert oracle_mod.halo_elements(r, (pw, 1, 1), 1) == expect
    r1 = M.make_conv("c1", 3, 3, (226, 226), 1)
    assert oracle_mod.halo_elements(r1, (4, 4, 1), 0) == 0          # K = 1: no halo


@pytest.mark.parametrize("seed", range(40))
def test_halo_matches_remote_index_enumeration(oracle_mod, seed):
    """Brute force: count remote input cells a PE needs (faces only, Q15) on small grids."""
    rng = random.Random(seed)
    nd = rng.choice([1, 2, 3])
    X = tuple(rng.randint(4, 12) for _ in range(nd))
    K = rng.choice([3, 5])
    C = rng.randint(1, 3)
    r = M.make_conv("c", C, C, X, K, stride=1, pad=K // 2)
    split = [1, 1, 1]
    ax = rng.randrange(nd)
    split[ax] = rng.choice([2, 3, 4])
    # interior PE along `ax` (or PE 0 if 2 parts): enumerate cells within K//2 outside its slab
    h = K // 2
    n = X[ax]
    loc = -(-n // split[ax])
    part = 1 if split[ax] > 2 else 0
    lo, hi = part * loc, min(n, (part + 1) * loc)
    cells = 0
    for cidx in itertools.product(*[range(v) for v in X]):
        c = cidx[ax]
        if (lo - h <= c < lo) or (hi <= c < hi + h):
            cells += 1
    expect = C * cells
    if split[ax] > 2 and hi + h > n:
        pytest.skip("interior slab touches the boundary (ragged split)")
    if loc < h:
        pytest.skip("SplitTooFine: the halo would span several PEs (infeasible)")
    got =oracle_mod.halo_elements(r, tuple(split), 0)
    assert got == expect


def test_spatial_halo_iteration_example(oracle_mod):
    e = EX["spatial_halo_iter"]
    r = M.make_conv("c", 3, 3, (226, 226), 3, stride=1, pad=1)
    r.flags |= M.FLAG_FOLDED
    m = toys.model([r], Ls=1)
    pr = _one(oracle_mod, m, toys.system(alpha=e["alpha"], beta=e["beta"], delta=e["delta"]),
              W.SubSweep(W.SPATIAL, b=[e["B"]], dims=[(1, 2, 1, 1)], Ls=[1]))
    assert abs(pr.t_halo - e["expect"]) <= 1e-18


def test_layer_pure_example(oracle_mod):
    e = EX["layer_pure_p2p_iter"]
    m = toys.model([toys.row(y=e["y"]), toys.row(y=1)])
    pr = _one(oracle_mod, m, toys.system(alpha=e["alpha"], beta=e["beta"], delta=e["delta"]),
              W.SubSweep(W.LAYERPURE, b=[e["B"]], part_mode=W.PART_COMB, s_min=2, s_max=2))
    assert pr.t_p2p == e["expect"]


def test_pipeline_examples(oracle_mod):
    e = EX["pipeline_comp_epoch"]
    m = toys.model([toys.row(fw=1, bw=1), toys.row(fw=1, bw=1)], D=e["D"])
    pr = _one(oracle_mod, m, toys.system(R=1.0),
              W.SubSweep(W.PIPELINE, b=[e["B"]], S=[e["S"]], part_mode=W.PART_COMB, s_min=2, s_max=2))
    assert pr.t_comp * pr.I == e["expect"]
    e = EX["pipeline_comm_iter"]
    m = toys.model([toys.row(y=e["y"]), toys.row(y=3)])
    pr = _one(oracle_mod, m, toys.system(alpha=e["alpha"], beta=e["beta"], delta=e["delta"]),
              W.SubSweep(W.PIPELINE, b=[e["B"]], S=[e["S"]], part_mode=W.PART_COMB, s_min=2, s_max=2))
    assert pr.t_p2p == e["expect"]


@pytest.mark.parametrize("pd", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("ws", [(1000, 7, 123457), (64, 64), (5, 999999, 3, 17)])
def test_pd_ge_equals_concurrent_rings(oracle_mod, pd, ws):
    """pd gradient exchange for p_d > 1 (Q17): the s stages' Allreduces run at once,
    each among the p_d replicas of its stage on disjoint PEs, so the phase is the slowest
    group's ring -- an explicit concurrent ring simulation (tests/brute.py), not the
    AR(p_d, delta max W_i) formula, fixes the value.  One row per stage (s = G)."""
    a, b = 3e-6, 1.0 / 7e9
    rows = [toys.row(w=w, fw=1, bw=1, y=1) for w in ws]
    m = toys.model(rows)
    G = len(rows)
    pr = _one(oracle_mod, m, toys.system(alpha=a, beta=b, delta=4),
              W.SubSweep(W.PD, b=[8], S=[1], dims=[(pd, 1, 1, 1)], part_mode=W.PART_COMB, s_min=G, s_max=G))
    want = brute.concurrent_rings_sim([4 * w for w in ws], pd, Fr(a), Fr(b))
    assert _rel(pr.t_ge, want) <= 4e-16
    assert pr.p == G * pd and pr.B == 8 * pd
    pr1 = _one(oracle_mod, m, toys.system(alpha=a, beta=b, delta=4),
               W.SubSweep(W.PD, b=[8], S=[1], dims=[(1, 1, 1, 1)], part_mode=W.PART_COMB, s_min=G, s_max=G))
    assert pr1.t_ge == 0.0


@pytest.mark.parametrize("seed", range(20))
def test_layerwise_reduces_to_data_and_filter(oracle_mod, seed):
    """Per-layer strategy (Q39): every COMM row data-parallel is the Data row of
    Table 2 and every COMM row filter-parallel is the Filter row at
    mini-batch b p, bit for bit (tolerance 0), for every p including p = 1."""
    m = corpus.random_model(seed)
    sysd = corpus.random_system(seed)
    nt = len(sysd.tiers)
    A = [[1e-5 * (t + 1) for t in range(nt)], [3e-6 * (t + 2) for t in range(nt)]]
    Bt = [[1e-9 * (t + 1) for t in range(nt)], [7e-10 * (t + 1) for t in range(nt)]]
    b = 4
    P = [1, 2, 3, 4, 8]
    nc = sum(1 for r in m.layers if r.flags & M.FLAG_COMM)
    if nc > 10:
        pytest.skip("too many COMM rows for a full mask enumeration")
    dims = [(p, 1, 1, 1) for p in P]
    subs = [W.SubSweep(W.LAYERWISE, b=[b], dims=dims, part_mode=W.PART_MASK, alpha=A, beta=Bt),
            W.SubSweep(W.DATA, b=[b], dims=dims, alpha=A, beta=Bt)]
    subs += [W.SubSweep(W.FILTER, b=[b * p], dims=[(p, 1, 1, 1)], alpha=A, beta=Bt) for p in P]
    sw = W.Sweep([m], sysd, subs, "lw")
    o = oracle_mod.OracleSweep(sw)
    fields = ("t_comp", "t_ge", "t_fb_ag", "t_fb_ar", "t_halo", "t_p2p", "t_iter", "t_epoch", "mem", "reason", "B", "p")
    confs = list(brute.enumerate_configs(sw))
    full = (1 << nc) - 1
    for idx, cfg in confs:
        if cfg["sub"] != 0 or cfg["ends"][1] not in (0, full):
            continue
        x = o.explain(idx)
        p = cfg["dims"][0]
        if cfg["ends"][1] == 0 or nc == 0:
            want = next(i for i, c in confs if c["sub"] == 1 and c["dims"] == cfg["dims"]
                        and c["alpha"] == cfg["alpha"] and c["beta"] == cfg["beta"])
        else:
            want = next(i for i, c in confs if c["sub"] == 2 + P.index(p)
                        and c["alpha"] == cfg["alpha"] and c["beta"] == cfg["beta"])
        y = o.explain(want)
        for f in fields:
            assert getattr(x, f) == getattr(y, f), (f, cfg["ends"], p)


@pytest.mark.parametrize("seed", range(10))
def test_layerwise_matches_exact_rationals(oracle_mod, seed):
    """Every configuration of the random corpora's per-layer-strategy sub-sweep (Q39) against
    the exact per-row rational evaluator and the buffer enumeration."""
    sw = corpus.random_sweep(seed)
    if sw.subs[-1].family != W.LAYERWISE:
        pytest.skip("no layerwise sub-sweep in this corpus")
    o = oracle_mod.OracleSweep(sw)
    si = len(sw.subs) - 1
    confs = [(i, c) for i, c in brute.enumerate_configs(sw) if c["sub"] == si]
    rng = random.Random(seed)
    for idx, cfg in rng.sample(confs, min(400, len(confs))):
        pr = o.explain(idx)
        ex = brute.exact(sw, cfg)
        assert pr.reason == ex["reason"], (idx, cfg)
        for f in ("t_comp", "t_ge", "t_fb_ag", "t_fb_ar", "t_iter", "mem", "I"):
            v = ex[f]
            got = getattr(pr, f)
            if v is None:
                assert math.isinf(got), (f, idx)
            else:
                assert _rel(got, v) <= 1e-14, (f, idx, got, float(v))
        assert _rel(pr.mem, brute.buffer_bytes(sw, cfg)) <= 1e-15


def test_layerwise_transitions_are_ring_collectives(oracle_mod):
    """Strategy changes (Q39): conv rows data-parallel, the FC rows filter-parallel (the
    'one weird trick' split P:413 cites), so one D -> F change at the first FC row: its
    input y (b samples per PE) is all-gathered forward and reduce-scattered backward,
    each the explicit ring simulation; the F rows' own Allgathers follow the
    Filter row.  Checked against the simulators, not the formula."""
    a, be = 2e-6, 1.0 / 9e9
    rows = [toys.row(y=1000, w=50, F=64), toys.row(y=600, w=70, F=64),
            toys.row(kind=M.FC, y=40, w=900, F=40), toys.row(kind=M.FC, y=10, w=400, F=10)]
    m = toys.model(rows)
    p, b = 4, 3
    sub = W.SubSweep(W.LAYERWISE, b=[b], dims=[(p, 1, 1, 1)], part_mode=W.PART_MASK)
    sw = toys.sweep(m, toys.system(alpha=a, beta=be, delta=4), [sub])
    o = oracle_mod.OracleSweep(sw)
    mask = 0b1100                      # rows 2, 3 filter-parallel
    pr = o.explain(mask)
    seg = Fr(b * 600 * 4)              # y_1 of b samples, delta = 4
    ag_in = brute.ring_allgather_sim(p, seg, Fr(a), Fr(be))
    full, _ = brute.ring_allreduce_sim(p, seg * p, Fr(a), Fr(be))
    rs_back = full - ag_in             # the ring's reduce-scatter half
    ag_fc = brute.ring_allgather_sim(p, Fr(b * p * 40 * 4, p), Fr(a), Fr(be))   # row 2 (not the last COMM row)
    assert _rel(pr.t_fb_ag, ag_fc + ag_in + rs_back) <= 2e-16
    assert _rel(pr.t_fb_ar, 2 * ag_fc) <= 2e-16
    back = o.explain(0b0011)           # F -> D at row 2: dL/dy_1 all-gathered backward only
    ag_fc2 = brute.ring_allgather_sim(p, Fr(b * p * 1000 * 4, p), Fr(a), Fr(be)) + \
        brute.ring_allgather_sim(p, Fr(b * p * 600 * 4, p), Fr(a), Fr(be))
    assert _rel(back.t_fb_ag, ag_fc2 + ag_in) <= 4e-16


@pytest.mark.parametrize("s,pd,node", [(2, 4, 4), (3, 2, 6), (4, 8, 8), (2, 2, 2), (1, 8, 4)])
def test_pd_ge_contention_equals_flow_count(oracle_mod, s, pd, node):
    """f1 contention (P:561 'divides the bandwidth of a link by the number of communication
    flows'; Q40): the s stage Allreduces of pd share the inter-node links; a link-level
    simulation of the concurrent rings counts the flows on the busiest link, and the oracle
    with phi_pd = that count gives the simulated makespan (s = 1: a single ring, no phi)."""
    a, be = 4e-6, 1.0 / 11e9
    ws = [4096 * (i + 1) for i in range(s)]
    rows = [toys.row(w=w, fw=1, bw=1, y=1) for w in ws]
    m = toys.model(rows)
    want, flows = brute.contended_stage_rings_sim(s, pd, node, 4 * max(ws), Fr(a), Fr(be))
    sysd = toys.system(alpha=a, beta=be, delta=4)
    sysd.phi_pd = float(max(flows, 1)) if s > 1 else 7.0   # s = 1 must ignore phi_pd
    pr = _one(oracle_mod, m, sysd, W.SubSweep(W.PD, b=[8], S=[1], dims=[(pd, 1, 1, 1)], part_mode=W.PART_COMB,
                                              s_min=s, s_max=s))
    assert _rel(pr.t_ge, want) <= 4e-16
    if s > 1:   # replica-major layout: every stage ring crosses the same inter-node links
        assert flows == (s if s * pd > node else 1)


def test_p2p_scales_touch_point_to_point_patterns_only(oracle_mod):
    """f1 per-pattern parameters (P:768-769 'different network parameters ... for MPI and
    NCCL'; Q40): with p2p scales (ka, kb) the halo exchange and the pipeline boundary sends
    equal those of a system whose tiers are (alpha ka, beta kb), while every collective
    (GE Allreduce, filter Allgather) equals the unscaled system's; and a 2-stage pipeline's
    boundary term is 2 (S) Hockney sends T_p2p(m) = alpha' + m beta'."""
    import dataclasses
    ka, kb = 3.0, 2.5
    a, be = 2e-6, 1.0 / 8e9
    spat = toys.model([toys.row(kind=M.CONV, C=4, F=4, X=(16, 16, 1), Y=(16, 16, 1), K=(3, 3, 1), x=1024,
                                y=1024, w=144, fw=10, bw=20)], Ls=1)
    base = toys.system(alpha=a, beta=be, delta=4)
    scaled = dataclasses.replace(base, p2p_alpha_scale=ka, p2p_beta_scale=kb)
    shifted = toys.system(alpha=a * ka, beta=be * kb, delta=4)
    sub = W.SubSweep(W.SPATIAL, b=[2], dims=[(1, 2, 2, 1)], Ls=[1])
    x, y, z = (_one(oracle_mod, spat, sd, sub) for sd in (scaled, shifted, base))
    assert x.t_halo == y.t_halo and x.t_halo != z.t_halo
    assert x.t_ge == z.t_ge and x.t_ge != y.t_ge
    pipe = toys.model([toys.row(y=5000, fw=10, bw=20), toys.row(y=3, fw=10, bw=20)])
    S, b = 2, 4
    pr = _one(oracle_mod, pipe, scaled, W.SubSweep(W.PIPELINE, b=[b], S=[S], part_mode=W.PART_COMB, s_min=2, s_max=2))
    send = Fr(a * ka) + Fr(b, S) * 5000 * 4 * Fr(be * kb)        # T_p2p(m) = alpha + m beta
    assert _rel(pr.t_p2p, 2 * (2 + S - 2) * send) <= 4e-16
    filt = toys.model([toys.row(y=64, F=64), toys.row(F=64)])
    fs = W.SubSweep(W.FILTER, b=[2], dims=[(4, 1, 1, 1)])
    assert _one(oracle_mod, filt, scaled, fs).t_fb_ag == _one(oracle_mod, filt, base, fs).t_fb_ag


def test_ds_reduce_to_leader_contention(oracle_mod):
    """phi_ds (Q40) multiplies the beta part of the ds reduce-to-leader only, and only when
    p1 > 1 groups reduce at once; the leaders' Allreduce and ds(1; split) are unchanged."""
    import dataclasses
    m = toys.model([toys.row(w=8192, X=(64, 1, 1), Y=(64, 1, 1))], Ls=0)
    base = toys.system(alpha=0.0, beta=1e-9)
    sub = W.SubSweep(W.DS, b=[1], dims=[(4, 2, 1, 1), (1, 2, 1, 1)], Ls=[0])
    o0 = oracle_mod.OracleSweep(toys.sweep(m, base, [sub]))
    o2 = oracle_mod.OracleSweep(toys.sweep(m, dataclasses.replace(base, phi_ds=2.0), [sub]))
    g0, g2 = o0.explain(0), o2.explain(0)
    al = 2 * (4 - 1) * (8192 / 4) * 1e-9          # leaders' Allreduce, alpha = 0
    rl = 2 * (2 - 1) * (8192 / 2) * 1e-9           # reduce-to-leader
    assert _rel(g0.t_ge, rl + al) <= 1e-15 and _rel(g2.t_ge, 2 * rl + al) <= 1e-15
    assert o0.explain(1).t_ge == o2.explain(1).t_ge


def test_partition_balanced_example(oracle_mod):
    e = EX["partition_balanced"]
    m = toys.model([toys.row(fw=c, bw=0) for c in e["costs"]], D=1)
    sw = toys.sweep(m, toys.system(R=1.0), [W.SubSweep(W.PIPELINE, b=[1], S=[1], part_mode=W.PART_COMB,
                                                        s_min=e["p"], s_max=e["p"])])
    o = oracle_mod.OracleSweep(sw)
    (best, key), = o.topk(0, o.size(), 1)[0][:1]
    # comp = (s+S-1)(B/S) maxFW = 2 * bottleneck  ->  bottleneck 4 with the cut after row 2
    assert key == 2 * e["bottleneck"]
    assert list(o.decode(best).stage_end[:2]) == [2, 4]


def test_filter_and_df_examples(oracle_mod):
    e = EX["filter_comm_epoch"]
    m = toys.model([toys.row(y=e["y1"], F=64), toys.row(F=64)], D=e["B"])
    pr = _one(oracle_mod, m, toys.system(alpha=e["alpha"], beta=e["beta"], delta=e["delta"]),
              W.SubSweep(W.FILTER, b=[e["B"]], dims=[(e["p"], 1, 1, 1)]))
    assert (pr.t_fb_ag + pr.t_fb_ar) * pr.I == e["expect"]
    e = EX["df_comm_epoch"]
    m = toys.model([toys.row(y=e["y1"], F=64, w=e["W"]), toys.row(F=64)], D=e["B"])
    pr = _one(oracle_mod, m, toys.system(alpha=e["alpha"], beta=e["beta"], delta=e["delta"], phi=1.0),
              W.SubSweep(W.DF, b=[e["B"] // e["p1"]], dims=[(e["p1"], e["p2"], 1, 1)]))
    assert (pr.t_fb_ag + pr.t_fb_ar + pr.t_ge) * pr.I == e["expect"]


def test_gpipe_schedule_vs_closed_form(oracle_mod):
    """Equal groups: the discrete-event makespan equals (p+S-1)(B/S)(FW+BW).
    Unequal groups: the closed form uses the slowest stage, so it upper-bounds the
    schedule, which is itself at least S segments of the slowest stage (Q34)."""
    rng = random.Random(3)
    for trial in range(200):
        s = rng.choice([2, 3, 4])
        S = rng.choice([1, 2, 4, 8])
        B = S * rng.choice([1, 2, 3])
        equal = trial < 40
        f = [rng.randint(1, 9) for _ in range(s)]
        g = [rng.randint(1, 9) for _ in range(s)]
        if equal:
            f = [f[0]] * s
            g = [g[0]] * s
        rows = [toys.row(fw=f[i], bw=g[i]) for i in range(s)]
        m = toys.model(rows, D=B)
        pr = _one(oracle_mod, m, toys.system(R=1.0),
                  W.SubSweep(W.PIPELINE, b=[B], S=[S], part_mode=W.PART_COMB, s_min=s, s_max=s))
        des = brute.gpipe_makespan([Fr(v) for v in f], [Fr(v) for v in g], S, Fr(B, S))
        if equal:
            assert Fr(pr.t_comp) == des
        else:
            assert des <= Fr(pr.t_comp)
            assert des >= S * Fr(B, S) * (max(f) + max(g)) / 2


# ------------------------------------------------------------ GPipe schedule family (Q36)
def test_gpipe_family_equals_event_simulation(oracle_mod):
    """No communication (alpha = beta = 0) and no WU: the family's time is the makespan of
    brute.gpipe_makespan, an independent discrete-event schedule.  Small
    integer stage times and R = 1 keep every fp64 value exact, so equality is exact."""
    rng = random.Random(11)
    for trial in range(150):
        s = rng.choice([1, 2, 3, 4, 5])
        S = rng.choice([1, 2, 3, 4, 8])
        B = S * rng.choice([1, 2, 3])
        f = [rng.randint(1, 9) for _ in range(s)]
        g = [rng.randint(1, 9) for _ in range(s)]
        rows = [toys.row(fw=f[i], bw=g[i]) for i in range(s)]
        m = toys.model(rows, D=B)
        pr = _one(oracle_mod, m, toys.system(R=1.0),
                  W.SubSweep(W.GPIPE, b=[B], S=[S], part_mode=W.PART_COMB, s_min=s, s_max=s,
                             alpha=[[0.0]], beta=[[0.0]]))
        des = brute.gpipe_makespan([Fr(v) for v in f], [Fr(v) for v in g], S, Fr(B, S))
        assert Fr(pr.t_comp) == des and pr.t_iter == pr.t_comp
        assert pr.t_p2p == 0.0 and pr.t_ge == 0.0


def test_gpipe_equal_stages_reduce_to_table2_row(oracle_mod):
    """Equal stages (compute, WU and boundary message): the schedule time equals Table 2's
    Layer row exactly in rationals, (s+S-1)(b/S)(FW+BW) + WU + 2(s+S-2)(alpha +
    (b/S) delta y beta); unequal stages: the row is an upper bound (P:1008 'approximated by
    the maximum', Q34) and S segments of the slowest stage a lower bound."""
    rng = random.Random(12)
    for trial in range(120):
        s = rng.choice([1, 2, 3, 4, 6, 8])
        S = rng.choice([1, 2, 4, 8])
        b = S * rng.choice([1, 2, 4])
        equal = trial < 50
        f = [rng.randint(1, 50) * 1000 for _ in range(s)]
        g = [rng.randint(1, 50) * 1000 for _ in range(s)]
        u = [rng.randint(0, 30) * 1000 for _ in range(s)]
        y = [rng.randint(1, 40) for _ in range(s)]
        if equal:
            f, g, u, y = [f[0]] * s, [g[0]] * s, [u[0]] * s, [y[0]] * s
        rows = [toys.row(fw=f[i], bw=g[i], wu=u[i], y=y[i]) for i in range(s)]
        m = toys.model(rows, D=b)
        A, Bt = [[rng.choice([0.0, 1e-6, 3e-5])]], [[rng.choice([0.0, 1e-9, 2e-10])]]
        sub = dict(b=[b], S=[S], part_mode=W.PART_COMB, s_min=s, s_max=s, alpha=A, beta=Bt)
        sysm = toys.system(R=1e9)
        gp = _one(oracle_mod, m, sysm, W.SubSweep(W.GPIPE, **sub))
        pl = _one(oracle_mod, m, sysm, W.SubSweep(W.PIPELINE, **sub))
        assert gp.mem == pl.mem and gp.reason == pl.reason
        if equal:
            assert _rel(gp.t_iter, pl.t_iter) <= 1e-14
        else:
            assert gp.t_iter <= pl.t_iter * (1 + 1e-14)
            assert gp.t_iter >= S * (b / S) * (max(f) + max(g)) / 1e9 * (1 - 1e-14)


def test_gpipe_single_segment_is_a_chain(oracle_mod):
    """S = 1: nothing overlaps, so the time is the chain sum f_1+c_1+...+f_s then
    g_s+c_{s-1}+...+g_1, plus the WU of the stage that finishes last (stage 1), unless
    a later stage's WU ends later."""
    rng = random.Random(13)
    for trial in range(60):
        s = rng.choice([1, 2, 3, 4])
        f = [rng.randint(1, 9) for _ in range(s)]
        g = [rng.randint(1, 9) for _ in range(s)]
        u = [rng.randint(0, 20) for _ in range(s)]
        y = [rng.randint(1, 5) for _ in range(s)]
        b = rng.choice([1, 2, 3])
        rows = [toys.row(fw=f[i], bw=g[i], wu=u[i], y=y[i]) for i in range(s)]
        m = toys.model(rows, D=b)
        a, be = 0.5, 0.25
        pr = _one(oracle_mod, m, toys.system(R=1.0),
                  W.SubSweep(W.GPIPE, b=[b], S=[1], part_mode=W.PART_COMB, s_min=s, s_max=s,
                             alpha=[[a]], beta=[[be]]))
        dl = 1   # toys.system delta
        c = [Fr(a) + b * dl * y[i] * Fr(be) for i in range(s - 1)]
        t_f = sum(b * Fr(v) for v in f) + sum(c)
        # stage i ends its backward after g_s..g_i and the sends of stages s..i (stage k
        # sends dL/dx to stage k-1 as part of its task, so stage i's own send is included)
        ends = [t_f + sum(b * Fr(g[k]) for k in range(i, s)) + sum(c[k - 1] for k in range(max(i, 1), s))
                for i in range(s)]
        want = max(ends[i] + u[i] for i in range(s))
        assert Fr(pr.t_iter) == want


# ------------------------------------------------------------ spatial prefix + Allgather (Q35)
def test_spatial_ag_allgather_is_a_ring_allgather(oracle_mod):
    """The boundary Allgather of y_Ls over p PEs with the per-PE segment B delta |y|/p
    (Q19) equals the explicit ring allgather simulation; it vanishes at Ls >= G."""
    rows = [toys.row(kind=M.CONV, X=(8, 8, 1), Y=(8, 8, 1), C=2, F=2, K=(3, 3, 1), x=128, y=128 + 8 * l)
            for l in range(3)]
    m = toys.model(rows, D=64)
    for p in (2, 4, 8):
        for Ls in (1, 2, 3):
            sub = W.SubSweep(W.SPATIAL_AG, b=[4], dims=[(1, p, 1, 1)], Ls=[Ls], alpha=[[1e-6]], beta=[[1e-9]])
            pr = _one(oracle_mod, m, toys.system(), sub)
            if Ls >= 3:
                assert pr.t_fb_ag == 0.0
                continue
            seg = Fr(4 * 1 * rows[Ls - 1].y, p)   # B = b = 4, delta = 1 (toys.system)
            want = brute.ring_allgather_sim(p, seg, Fr(1e-6), Fr(1e-9))
            assert _rel(pr.t_fb_ag, want) <= 1e-15


def test_spatial_ag_limits(oracle_mod):
    """Ls = G is the Spatial row bit for bit (no boundary, nothing replicated); p = 1 has
    no communication and the serial compute and memory (up to rounding order); a longer
    prefix never increases compute or memory (more rows divided by p)."""
    for seed in range(8):
        m = corpus.random_model(seed)
        sysd = corpus.random_system(seed)
        nt = len(sysd.tiers)
        A, Bt = [[1e-5] * nt], [[1e-9] * nt]
        dims = [(1, 1, 1, 1), (1, 2, 1, 1), (1, 2, 2, 1)]
        sp = W.SubSweep(W.SPATIAL, b=[4], dims=dims, Ls=[m.G], alpha=A, beta=Bt)
        ag = W.SubSweep(W.SPATIAL_AG, b=[4], dims=dims, Ls=list(range(1, m.G + 1)), alpha=A, beta=Bt)
        se = W.SubSweep(W.SERIAL, b=[4], alpha=A, beta=Bt)
        sw = W.Sweep([m], sysd, [sp, ag, se], "ag")
        o = oracle_mod.OracleSweep(sw)
        serial = _pred(o, 2, sw)
        for d in dims:
            x, y = _pred(o, 0, sw, dims=d), _pred(o, 1, sw, dims=d, Ls=m.G)
            for f in ("t_comp", "t_ge", "t_fb_ag", "t_halo", "t_iter", "t_epoch", "mem", "reason"):
                assert getattr(x, f) == getattr(y, f), (seed, d, f)
            prev = None
            for Ls in range(1, m.G + 1):
                z = _pred(o, 1, sw, dims=d, Ls=Ls)
                if d == (1, 1, 1, 1):
                    assert z.t_ge == z.t_fb_ag == z.t_halo == 0.0
                    assert _rel(z.t_comp, serial.t_comp) <= 1e-14 and _rel(z.mem, serial.mem) <= 1e-14
                if prev is not None:
                    assert z.t_comp <= prev.t_comp * (1 + 1e-15) and z.mem <= prev.mem * (1 + 1e-15)
                prev = z


# ------------------------------------------------------------ per-layer gradient messages (Q37)
def test_data_lw_reduces_to_table2(oracle_mod):
    """Ring only: one Allreduce per weighted layer costs Table 2's data GE plus one extra
    startup 2(p-1) alpha per additional message, exactly (rationals); a model with one
    weighted layer is the Data row bit for bit; compute and memory are the Data row's."""
    rng = random.Random(21)
    for trial in range(60):
        n = rng.randint(1, 6)
        ws = [rng.choice([0, rng.randint(1, 5000)]) for _ in range(n)]
        if not any(ws):
            ws[0] = 7
        rows = [toys.row(w=w, fw=rng.randint(1, 99), bw=rng.randint(1, 99), x=3, y=5) for w in ws]
        m = toys.model(rows, D=1000)
        p = rng.choice([1, 2, 3, 4, 8, 64])
        a, be = rng.choice([1e-6, 3e-5]), rng.choice([1e-9, 5e-10])
        sysm = toys.system(delta=4)
        sub = dict(b=[4], dims=[(p, 1, 1, 1)], alpha=[[a]], beta=[[be]])
        lw = _one(oracle_mod, m, sysm, W.SubSweep(W.DATA_LW, **sub))
        dp = _one(oracle_mod, m, sysm, W.SubSweep(W.DATA, **sub))
        nw = sum(1 for w in ws if w > 0)
        want = Fr(dp.t_ge) + (nw - 1) * 2 * (p - 1) * Fr(a) if p > 1 else Fr(0)
        assert _rel(lw.t_ge, want) <= 1e-14
        assert lw.t_comp == dp.t_comp and lw.mem == dp.mem and lw.reason == dp.reason
        if nw == 1:
            assert lw.t_ge == dp.t_ge and lw.t_iter == dp.t_iter


def test_data_lw_per_message_dispatch(oracle_mod):
    """Each message is timed by the tree form when smaller than the threshold and by the
    ring otherwise: a small and a large layer straddling the threshold give
    tree(small) + ring(large), checked against the explicit ring simulation."""
    rows = [toys.row(w=100), toys.row(w=1_000_000)]
    m = toys.model(rows, D=10)
    a, be, p, k = 2e-6, 1e-9, 8, 4
    sysm = toys.system(delta=4, tree_threshold=1e5, tree_chunks=k)
    lw = _one(oracle_mod, m, sysm, W.SubSweep(W.DATA_LW, b=[2], dims=[(p, 1, 1, 1)], alpha=[[a]], beta=[[be]]))
    tree_small = 2 * (3 + k) * (Fr(a) + Fr(400, 2 * k) * Fr(be))
    ring_large, _ = brute.ring_allreduce_sim(p, Fr(4_000_000), Fr(a), Fr(be))
    assert _rel(lw.t_ge, tree_small + ring_large) <= 1e-15


# ------------------------------------------------------------ filter Reduce-Scatter variant (Q38)
def test_filter_reduce_scatter_variant(oracle_mod):
    """P:355 footnote: layer l-1 needs only its partition of dL/dx, so the backward exchange
    can be a Reduce-Scatter: (p-1) steps of the per-PE segment (the ring's first half,
    P:553-556), i.e. one Allgather's cost instead of the Allreduce's two.  With filter_rs
    the FB-AR phase equals FB-AG bit for bit; filter / channel / df all switch."""
    m = corpus.random_model(3)
    for fam, dims in ((W.FILTER, (4, 1, 1, 1)), (W.CHANNEL, (2, 1, 1, 1)), (W.DF, (2, 2, 1, 1))):
        for rs in (0, 1):
            sysm = toys.system(delta=4, alpha=1e-6, beta=1e-9)
            sysm.filter_rs = rs
            pr = _one(oracle_mod, m, sysm, W.SubSweep(fam, b=[2], dims=[dims]))
            if pr.t_fb_ag == 0.0:
                continue
            if rs:
                assert pr.t_fb_ar == pr.t_fb_ag
            else:
                assert pr.t_fb_ar == 2.0 * pr.t_fb_ag
    # the Reduce-Scatter cost is the ring simulation's reduce-scatter half
    p, seg = 4, Fr(1000)
    full, _ = brute.ring_allreduce_sim(p, seg * p, Fr(1e-6), Fr(1e-9))
    assert full / 2 == brute.ring_allgather_sim(p, seg, Fr(1e-6), Fr(1e-9))


# ------------------------------------------------------------ memory
@pytest.mark.parametrize("seed", range(25))
def test_memory_rows_equal_buffer_enumeration(oracle_mod, seed):
    sw = corpus.random_sweep(seed)
    o = oracle_mod.OracleSweep(sw)
    n = o.size()
    rng = random.Random(seed)
    confs = list(brute.enumerate_configs(sw))
    for idx, cfg in rng.sample(confs, min(60, len(confs))):
        pr = o.explain(idx)
        want = brute.buffer_bytes(sw, cfg)
        assert _rel(pr.mem, want) <= 1e-15, (idx, cfg["family"])
    assert n == len(confs)


# ------------------------------------------------------------ exact rational evaluator
@pytest.mark.parametrize("seed", range(30))
def test_oracle_matches_exact_rationals(oracle_mod, seed):
    sw = corpus.random_sweep(seed)
    o = oracle_mod.OracleSweep(sw)
    confs = list(brute.enumerate_configs(sw))
    rng = random.Random(1000 + seed)
    for idx, cfg in rng.sample(confs, min(80, len(confs))):
        pr = o.explain(idx)
        ex = brute.exact(sw, cfg)
        assert pr.reason == ex["reason"], (idx, cfg, pr.reason, ex["reason"])
        assert pr.B == ex["B"] and pr.p == ex["p"]
        for f in ("t_comp", "t_ge", "t_fb_ag", "t_fb_ar", "t_halo", "t_p2p", "t_iter", "mem", "I"):
            v = ex[f]
            got = getattr(pr, f)
            if v is None:
                assert math.isinf(got), (f, idx)
            else:
                assert _rel(got, v) <= 1e-14, (f, idx, cfg["family"], got, float(v))


@pytest.mark.parametrize("seed", range(12))
def test_decoder_matches_itertools_enumeration(oracle_mod, seed):
    sw = corpus.random_sweep(seed, max_list=2)
    o = oracle_mod.OracleSweep(sw)
    confs = list(brute.enumerate_configs(sw))
    assert o.size() == len(confs)
    rng = random.Random(seed)
    for idx, cfg in rng.sample(confs, min(300, len(confs))):
        c = o.decode(idx)
        assert c.sub == cfg["sub"] and c.b == cfg["b"] and c.S == cfg["S"]
        assert tuple(c.dims) == tuple(cfg["dims"]) and c.Ls == cfg["Ls"]
        if cfg["family"] == W.LAYERWISE:
            assert c.i_part == cfg["ends"][1] and c.n_stages == 1
        else:
            assert tuple(c.stage_end[:c.n_stages]) == cfg["ends"]
        nt = len(sw.system.tiers)
        assert list(c.alpha[:nt]) == list(cfg["alpha"]) and list(c.beta[:nt]) == list(cfg["beta"])
        assert c.cap == cfg["cap"] and c.flops == cfg["R"]


def test_partition_counts():
    from math import comb
    for G in range(1, 20):
        assert sum(comb(G - 1, s - 1) for s in range(1, G + 1)) == 2 ** (G - 1)
    assert sum(comb(151, k) for k in range(6)) == 633_245_832
    assert sum(comb(49, k) for k in range(4)) == 19650


# ------------------------------------------------------------ literal fold vs canonical trees
@pytest.mark.parametrize("seed", range(30))
def test_canonical_tree_matches_literal_fold(oracle_mod, seed):
    sw = corpus.random_sweep(seed)
    o = oracle_mod.OracleSweep(sw)
    n = o.size()
    rng = random.Random(seed)
    for idx in rng.sample(range(n), min(200, n)):
        a = o.explain(idx)
        b = o.explain(idx, fold=True)
        for f in ("t_comp", "t_ge", "t_fb_ag", "t_fb_ar", "t_halo", "t_p2p", "t_iter", "mem"):
            x, y = getattr(a, f), getattr(b, f)
            if math.isinf(x) or math.isinf(y):
                assert x == y
            else:
                assert _rel(x, y) <= 1e-12, (f, idx, x, y)


# ------------------------------------------------------------ degenerate identities (tolerance 0)
def _pred(o, sub_i, sw, **fix):
    confs = [c for c in brute.enumerate_configs(sw) if c[1]["sub"] == sub_i]
    for idx, cfg in confs:
        if all(cfg[k] == v for k, v in fix.items()):
            return o.explain(idx)
    raise KeyError(fix)


@pytest.mark.parametrize("seed", range(20))
def test_degenerate_identities(oracle_mod, seed):
    m = corpus.random_model(seed)
    sysd = corpus.random_system(seed)
    nt = len(sysd.tiers)
    A = [[1e-5 * (t + 1) for t in range(nt)]]
    Bt = [[1e-9 * (t + 1) for t in range(nt)]]
    b = 4
    P = [2, 3, 4]
    subs = [
        W.SubSweep(W.SERIAL, b=[b], alpha=A, beta=Bt),                                           # 0
        W.SubSweep(W.DATA, b=[b], dims=[(1, 1, 1, 1)] + [(p, 1, 1, 1) for p in P], alpha=A, beta=Bt),
        W.SubSweep(W.SPATIAL, b=[b], dims=[(1, 1, 1, 1), (1, 2, 1, 1), (1, 2, 2, 1)], Ls=[m.G], alpha=A, beta=Bt),
        W.SubSweep(W.FILTER, b=[b], dims=[(1, 1, 1, 1)] + [(p, 1, 1, 1) for p in P], alpha=A, beta=Bt),
        W.SubSweep(W.CHANNEL, b=[b], dims=[(1, 1, 1, 1)] + [(p, 1, 1, 1) for p in P], alpha=A, beta=Bt),
        W.SubSweep(W.DF, b=[b], dims=[(1, p, 1, 1) for p in P] + [(p, 1, 1, 1) for p in P], alpha=A, beta=Bt),
        W.SubSweep(W.DS, b=[b], dims=[(p, 1, 1, 1) for p in P] + [(1, 2, 1, 1), (1, 2, 2, 1)], Ls=[m.G],
                   alpha=A, beta=Bt),
        W.SubSweep(W.PIPELINE, b=[b], S=[1, 2], part_mode=W.PART_COMB, s_min=1, s_max=min(3, m.G), alpha=A, beta=Bt),
        W.SubSweep(W.PD, b=[b], S=[1, 2], dims=[(1, 1, 1, 1)], part_mode=W.PART_COMB, s_min=1,
                   s_max=min(3, m.G), alpha=A, beta=Bt),
    ]
    sw = W.Sweep([m], sysd, subs, "deg")
    o = oracle_mod.OracleSweep(sw)
    fields = ("t_comp", "t_ge", "t_fb_ag", "t_fb_ar", "t_halo", "t_p2p", "t_iter", "t_epoch", "mem", "reason")

    def same(x, y, fs=fields):
        for f in fs:
            assert getattr(x, f) == getattr(y, f), f

    serial = _pred(o, 0, sw)
    for si, d in ((1, (1, 1, 1, 1)), (2, (1, 1, 1, 1)), (3, (1, 1, 1, 1)), (4, (1, 1, 1, 1))):
        x = _pred(o, si, sw, dims=d)
        same(x, serial, ("t_comp", "t_iter", "t_epoch", "mem"))
    for p in P:
        f = _pred(o, 3, sw, dims=(p, 1, 1, 1))
        c = _pred(o, 4, sw, dims=(p, 1, 1, 1))
        same(f, c, ("t_comp", "t_iter", "t_epoch", "mem"))                  # filter == channel
        same(_pred(o, 5, sw, dims=(1, p, 1, 1)), f, fields[:-1])            # df(1,p) == filter(p)
        same(_pred(o, 5, sw, dims=(p, 1, 1, 1)), _pred(o, 1, sw, dims=(p, 1, 1, 1)))   # df(p,1) == data(p)
        same(_pred(o, 6, sw, dims=(p, 1, 1, 1)), _pred(o, 1, sw, dims=(p, 1, 1, 1)))   # ds(p;1) == data(p)
    for d in ((1, 2, 1, 1), (1, 2, 2, 1)):
        same(_pred(o, 6, sw, dims=d), _pred(o, 2, sw, dims=d))                     # ds(1;split) == spatial
    pipe1 = _pred(o, 7, sw, ends=(m.G,), S=1)
    assert pipe1.t_comp == serial.t_comp                                           # pipeline(1,1) == serial comp
    for c in brute.enumerate_configs(sw):
        if c[1]["sub"] == 8:
            q = _pred(o, 7, sw, ends=c[1]["ends"], S=c[1]["S"])
            same(o.explain(c[0]), q)                                               # pd(1) == pipeline


# ------------------------------------------------------------ paper pins: layer tables, limits
def test_table4_layer_tables():
    pin = PIN["table4_layers"]
    assert M.resnet(50).G == pin["resnet50"]
    assert M.resnet(152).G == pin["resnet152"]
    assert M.vgg16().G == pin["vgg16"]
    assert M.cosmoflow(256).G == pin["cosmoflow"]
    pp = PIN["table4_params_approx"]
    for name, mdl in (("resnet50", M.resnet(50)), ("resnet152", M.resnet(152)),
                      ("vgg16", M.vgg16()), ("cosmoflow", M.cosmoflow(256))):
        tol = pp["vgg16_rel_tol"] if name == "vgg16" else pp["rel_tol"]
        assert abs(M.param_count(mdl) / pp[name] - 1) <= tol, name
    assert M.resnet(50).D == 1_281_167 and abs(M.resnet(50).D / PIN["imagenet_samples"]["D_approx"] - 1) < 0.01
    assert M.cosmoflow(512).D == PIN["cosmoflow_samples"]["D"]
    assert M.vgg16().layers[0].C == PIN["channel_first_layer"]["first_C"]
    c1 = M.cosmoflow(512).layers[0]
    assert (c1.x + c1.y) * PIN["cosmoflow512_conv1_activation"]["delta"] > PIN["cosmoflow512_conv1_activation"]["min_bytes"]


def test_filter_limit_64(oracle_mod):
    pin = PIN["filter_limit"]
    for name in ("vgg16", "resnet50"):
        m = M.by_name(name)
        sw = W.Sweep([m], W.two_tier_system(hbm_bytes=1e30),
                     [W.SubSweep(W.FILTER, b=[1], dims=[(pin[name], 1, 1, 1), (2 * pin[name], 1, 1, 1)])])
        o = oracle_mod.OracleSweep(sw)
        assert o.explain(0).reason & brute.R_SCALING == 0
        assert o.explain(1).reason & brute.R_SCALING


def test_cosmoflow_data_parallel_memory_infeasible(oracle_mod):
    """CosmoFlow 512^3 cannot run data-parallel in 16 GB; ds with a spatial split can
    (SPEC acceptance 10).  The rejection reason is Memory, not ScalingLimit."""
    m = M.cosmoflow(512)
    cap = PIN["cosmoflow_data_infeasible"]["cap_bytes"]
    sysd = W.two_tier_system(hbm_bytes=cap)
    sw = W.Sweep([m], sysd, [
        W.SubSweep(W.DATA, b=[1], dims=[(p, 1, 1, 1) for p in (1, 16, 256)]),
        W.SubSweep(W.FILTER, b=[1], dims=[(4, 1, 1, 1)]),
        W.SubSweep(W.PIPELINE, b=[1], part_mode=W.PART_COMB, s_min=1, s_max=4),
        W.SubSweep(W.DS, b=[1], dims=[(4, 4, 4, 2)], Ls=[6]),
    ])
    o = oracle_mod.OracleSweep(sw)
    for i in range(3):
        r = o.explain(i).reason
        assert r & brute.R_MEMORY and not r & brute.R_SCALING
    assert o.explain(3).reason & brute.R_MEMORY
    npipe = 1 + 19 + 171 + 969
    assert all(o.explain(4 + i).reason & brute.R_MEMORY for i in range(npipe))
    assert o.explain(4 + npipe).feasible


def test_config1_expectations(oracle_mod):
    """22 of 33 feasible; argmin p=1024, b=64 (idx 31); b=128 needs > 16 GiB."""
    sw = W.config1()
    o = oracle_mod.OracleSweep(sw)
    hits, nf = o.topk(0, o.size(), 3)
    assert o.size() == 33 and nf == 22
    assert hits[0][0] == 31
    c = o.decode(31)
    assert c.b == 64 and c.dims[0] == 1024
    for idx in range(33):
        pr = o.explain(idx)
        assert (pr.reason == 0) == (o.decode(idx).b != 128)
