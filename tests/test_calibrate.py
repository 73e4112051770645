"""Empirical parametrization on CPU: the alpha/beta fit inverts
the ring Allreduce form exactly, the gloo world-2 measurement path runs end to end, and
measured per-layer times become a layer table the oracle accepts (FW_l = measured)."""
from __future__ import annotations

import os
import random
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import toys
from workloads import calibrate as CAL
from workloads import models as M
from workloads import sweeps as W


def test_fit_recovers_ring_parameters():
    rng = random.Random(5)
    for _ in range(20):
        p = rng.choice([2, 4, 8, 64])
        a, b = rng.uniform(1e-6, 5e-5), 1.0 / rng.uniform(1e9, 9e11)
        sizes = [1 << e for e in range(10, 29, 2)]
        t = [2 * (p - 1) * (a + m / p * b) for m in sizes]
        fa, fb, rms = CAL.fit_allreduce(p, sizes, t)
        assert abs(fa - a) <= 1e-9 * a and abs(fb - b) <= 1e-9 * b and rms < 1e-12
        noisy = [v * (1 + rng.uniform(-0.02, 0.02)) for v in t]
        fa, fb, rms = CAL.fit_allreduce(p, sizes, noisy)
        assert abs(fa - a) <= 0.1 * a and abs(fb - b) <= 0.1 * b and rms < 0.05


def test_fit_rejects_single_pe():
    with pytest.raises(ValueError):
        CAL.fit_allreduce(1, [1, 2], [1.0, 2.0])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        tier = CAL.calibrate_tier([1 << 12, 1 << 16, 1 << 20], reps=3, device=torch.device("cpu"))
        if rank == 0:
            q.put(tier)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_calibration():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    tier = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert tier["p"] == 2 and len(tier["times_s"]) == 3
    assert all(t > 0 for t in tier["times_s"])
    assert tier["alpha_s"] >= 0 and tier["beta_s_per_B"] > 0
    s = CAL.system_from_tiers([tier], flops_per_s=1e12, hbm_bytes=16e9)
    assert s.tiers[0].max_pes == 2


def test_measured_layer_table(oracle_mod):
    """Per-layer times on CPU for a small conv / FC model; the empirical table gives the
    oracle's serial compute = sum of the measured per-sample times x b (+ WU)."""
    rows = [M.make_conv("c1", 3, 8, (16, 16), 3, pad=1), M.make_conv("c2", 8, 8, (16, 16), 3, stride=2, pad=1),
            M.make_fc("fc", 8 * 8 * 8, 10, (1, 1))]
    m = M.Model("tiny", rows, 100, default_Ls=2)
    times = CAL.time_layers(m, b=4, reps=2, warmup=1, device=torch.device("cpu"))
    assert times[0] is not None and times[2] is not None
    R = 1e12
    em = CAL.empirical_model(m, times, R)
    for r, t in zip(em.layers, times):
        if t is not None:
            assert abs(r.fw / R - t[0]) <= 1e-12 + 1e-9 * t[0]
    sysm = W.two_tier_system(flops_per_s=R)
    sw = W.Sweep([em], sysm, [W.SubSweep(W.SERIAL, b=[4])], "emp")
    o = oracle_mod.OracleSweep(sw)
    pr = o.explain(0)
    want = 4 * sum((r.fw + r.bw) for r in em.layers) / R + sum(r.wu for r in em.layers) / R
    assert abs(pr.t_comp - want) <= 1e-12 * want


def test_tree_p2p_allgather_fits_recover_parameters():
    """f2 per-pattern fits: each least-squares fit inverts its own form
    on exact samples, and stays within 10 % under 2 % noise."""
    rng = random.Random(11)
    sizes = [1 << e for e in range(8, 29, 2)]
    for _ in range(10):
        p, k = rng.choice([2, 4, 8, 64]), rng.choice([1, 2, 4])
        a, b = rng.uniform(1e-6, 5e-5), 1.0 / rng.uniform(1e9, 9e11)
        lg = (p - 1).bit_length()
        cases = [(lambda m: 2 * (lg + k) * (a + m / (2 * k) * b), lambda t: CAL.fit_allreduce_tree(p, sizes, t, k)),
                 (lambda m: a + m * b, lambda t: CAL.fit_p2p(sizes, t)),
                 (lambda m: (p - 1) * (a + m * b), lambda t: CAL.fit_allgather(p, sizes, t))]
        for form, fit in cases:
            t = [form(m) for m in sizes]
            fa, fb, rms = fit(t)
            assert abs(fa - a) <= 1e-9 * a and abs(fb - b) <= 1e-9 * b and rms < 1e-12
            fa, fb, rms = fit([v * (1 + rng.uniform(-0.02, 0.02)) for v in t])
            assert abs(fa - a) <= 0.1 * a and abs(fb - b) <= 0.1 * b


def test_tree_threshold_is_the_crossing():
    """tree_threshold_B = the message size where the fitted tree and ring forms
    cross: the tree is faster below it and slower above it."""
    p, k = 16, 2
    ring, tree = (2e-5, 1.0 / 3e11), (4e-6, 1.0 / 5e10)
    thr = CAL.tree_threshold(p, ring, tree, k)
    lg = 4

    def rt(m):
        return 2 * (p - 1) * (ring[0] + m / p * ring[1])

    def tt(m):
        return 2 * (lg + k) * (tree[0] + m / (2 * k) * tree[1])
    assert 1 < thr < 1 << 34
    assert tt(thr * 0.99) < rt(thr * 0.99) and tt(thr * 1.01) > rt(thr * 1.01)
    assert CAL.tree_threshold(p, (1e-6, 1e-12), (1e-3, 1e-9), k) == 0.0   # tree never wins


def _worker_patterns(rank, ws, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        sizes = [1 << 12, 1 << 16, 1 << 20]
        tp = CAL.time_p2p(sizes, reps=3, warmup=1, device=torch.device("cpu"))
        tg = CAL.time_allgather(sizes, reps=3, warmup=1, device=torch.device("cpu"))
        tier = CAL.calibrate_tier(sizes, reps=3, device=torch.device("cpu"))
        if rank == 0:
            q.put((sizes, tp, tg, tier))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_point_to_point_and_allgather():
    """The per-pattern measurements run end to end on a gloo world of 2 and give the system's
    p2p scales (Q40)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_patterns, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    sizes, tp, tg, tier = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
    assert all(t > 0 for t in tp) and all(t > 0 for t in tg)
    fa, fb, _ = CAL.fit_p2p(sizes, tp)
    ka, kb = CAL.p2p_scales(tier, (fa, fb))
    assert ka >= 0 and kb > 0
    ga, gb, _ = CAL.fit_allgather(2, sizes, tg)
    assert ga >= 0 and gb > 0
