"""Empirical parametrization (PAPER.md "Empirical Parametrization").

INPUT GENERATOR, like the rest of workloads/: it produces the two kinds of inputs the paper
measures instead of deriving -- the Hockney alpha/beta of the collectives on the target
system and per-layer compute times -- and turns them into the layer tables / system
descriptions the sweep takes.  None of the cost model's arithmetic lives here (no Table 2
terms); the fits only invert the ring Allreduce form the paper uses to define alpha and
beta (T_ar(p, m) = 2(p-1)(alpha + (m/p) beta)).

* time_allreduce / calibrate_tier: "we empirically measure the communication time of
  collective communication patterns, such as Allreduce, with different message size ...
  We then use those benchmark results to interpolate alpha and beta" -- here
  with torch.distributed (NCCL over NVLink on a B200 box, gloo on CPU for the tests) and
  a least-squares fit of the ring form over the message sizes.
* time_layers / empirical_model: "We empirically profile the average computation time per
  sample of each layer" -- conv / FC rows timed forward and forward+backward with
  torch (cuDNN on the GPU), per sample; the model's fw/bw become "effective FLOPs"
  fw' = t * R_ref so that FW_l = fw'/R_ref is the measured time (Q28's FLOP convention is
  the fallback for rows that are not timed).
"""
from __future__ import annotations

import copy
import statistics
import time

import numpy as np

from . import models as M
from . import sweeps as W


# ------------------------------------------------------------------ collectives
def fit_allreduce(p: int, sizes_bytes, times_s):
    """Least-squares alpha, beta of the ring Allreduce form T = 2(p-1) alpha + 2(p-1)(m/p) beta
     over (message size, time) samples.  Returns (alpha, beta, rms relative residual);
    alpha is clipped at 0 and beta at a tiny positive value (the library needs beta > 0)."""
    if p < 2:
        raise ValueError("an Allreduce fit needs p >= 2")
    m = np.asarray(sizes_bytes, np.float64)
    t = np.asarray(times_s, np.float64)
    c = 2.0 * (p - 1)
    A = np.stack([np.full_like(m, c), c * m / p], axis=1)
    # relative least squares: every size weighs the same
    w = 1.0 / t
    sol, *_ = np.linalg.lstsq(A * w[:, None], t * w, rcond=None)
    alpha, beta = float(max(sol[0], 0.0)), float(max(sol[1], 1e-18))
    pred = A @ np.array([alpha, beta])
    rms = float(np.sqrt(np.mean(((pred - t) / t) ** 2)))
    return alpha, beta, rms


def _lstsq_rel(A, t):
    """Relative least squares (every sample weighs the same), non-negative alpha, positive beta."""
    w = 1.0 / t
    sol, *_ = np.linalg.lstsq(A * w[:, None], t * w, rcond=None)
    alpha, beta = float(max(sol[0], 0.0)), float(max(sol[1], 1e-18))
    pred = A @ np.array([alpha, beta])
    return alpha, beta, float(np.sqrt(np.mean(((pred - t) / t) ** 2)))


def fit_allreduce_tree(p: int, sizes_bytes, times_s, k: int = 1):
    """Least-squares alpha, beta of the footnote's tree Allreduce form (Q18):
    T = 2(ceil(log2 p) + k)(alpha + (m / (2k)) beta) -- NCCL's choice for small messages."""
    if p < 2:
        raise ValueError("an Allreduce fit needs p >= 2")
    m = np.asarray(sizes_bytes, np.float64)
    t = np.asarray(times_s, np.float64)
    lg = 0
    while (1 << lg) < p:
        lg += 1
    c = 2.0 * (lg + k)
    return _lstsq_rel(np.stack([np.full_like(m, c), c * m / (2.0 * k)], axis=1), t)


def tree_threshold(p: int, ring, tree, k: int = 1, lo: float = 1.0, hi: float = float(1 << 34)) -> float:
    """Message size below which the fitted tree form predicts less time than the fitted ring
    form (both forms of P:556 / P:559): the system's tree_threshold_B.  0 when the ring is never
    slower in [lo, hi]; ring / tree = (alpha, beta) pairs."""
    lg = 0
    while (1 << lg) < p:
        lg += 1

    def t_ring(m):
        return 2 * (p - 1) * (ring[0] + m / p * ring[1])

    def t_tree(m):
        return 2 * (lg + k) * (tree[0] + m / (2 * k) * tree[1])

    if not t_tree(lo) < t_ring(lo):
        return 0.0
    if t_tree(hi) < t_ring(hi):
        return hi
    a, b = lo, hi
    for _ in range(200):   # bisection on the crossing (both forms are affine in m)
        mid = 0.5 * (a + b)
        if t_tree(mid) < t_ring(mid):
            a = mid
        else:
            b = mid
    return b


def fit_p2p(sizes_bytes, times_s):
    """Hockney point-to-point alpha, beta (T_p2p(m) = alpha + m beta) from one-way times."""
    m = np.asarray(sizes_bytes, np.float64)
    t = np.asarray(times_s, np.float64)
    return _lstsq_rel(np.stack([np.ones_like(m), m], axis=1), t)


def fit_allgather(p: int, seg_bytes, times_s):
    """Ring Allgather alpha, beta (T_ag = (p-1)(alpha + m_seg beta), per-PE segment, Q19)."""
    if p < 2:
        raise ValueError("an Allgather fit needs p >= 2")
    m = np.asarray(seg_bytes, np.float64)
    t = np.asarray(times_s, np.float64)
    c = float(p - 1)
    return _lstsq_rel(np.stack([np.full_like(m, c), c * m], axis=1), t)


def p2p_scales(collective_tier: dict, p2p_fit) -> tuple:
    """The system's p2p_alpha_scale / p2p_beta_scale (Q40): measured point-to-point
    alpha, beta over the collective tier's (the paper plugs 'different network parameters ...
    for MPI and NCCL')."""
    a, b = p2p_fit[0], p2p_fit[1]
    ca, cb = collective_tier["alpha_s"], collective_tier["beta_s_per_B"]
    return (a / ca if ca > 0 else 1.0), (b / cb if cb > 0 else 1.0)


def time_p2p(sizes_bytes, reps: int = 20, warmup: int = 3, device=None, group=None, peer=(0, 1)):
    """One-way send time between two ranks of the group (half the median ping-pong round trip,
    max over the pair); other ranks only join the final reduction."""
    import torch
    import torch.distributed as dist
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if torch.cuda.is_available() else torch.device("cpu"))
    rank = dist.get_rank(group)
    a_, b_ = peer
    out = []
    for m in sizes_bytes:
        n = max(1, int(m) // 4)
        buf = torch.ones(n, dtype=torch.float32, device=dev)
        ts = []
        for it in range(warmup + reps):
            dist.barrier(group=group)
            t0 = time.perf_counter()
            if rank == a_:
                dist.send(buf, dst=b_ if group is None else dist.get_global_rank(group, b_), group=group)
                dist.recv(buf, src=b_ if group is None else dist.get_global_rank(group, b_), group=group)
            elif rank == b_:
                dist.recv(buf, src=a_ if group is None else dist.get_global_rank(group, a_), group=group)
                dist.send(buf, dst=a_ if group is None else dist.get_global_rank(group, a_), group=group)
            if dev.type == "cuda":
                torch.cuda.synchronize()
            if it >= warmup:
                ts.append((time.perf_counter() - t0) / 2)
        med = torch.tensor([statistics.median(ts) if rank in peer else 0.0], dtype=torch.float64, device=dev)
        dist.all_reduce(med, op=dist.ReduceOp.MAX, group=group)
        out.append(float(med.item()))
    return out


def time_allgather(seg_bytes, reps: int = 20, warmup: int = 3, device=None, group=None):
    """Median all_gather time per per-PE segment size, max over the ranks."""
    import torch
    import torch.distributed as dist
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if torch.cuda.is_available() else torch.device("cpu"))
    ws = dist.get_world_size(group)
    out = []
    for m in seg_bytes:
        n = max(1, int(m) // 4)
        buf = torch.ones(n, dtype=torch.float32, device=dev)
        parts = [torch.empty_like(buf) for _ in range(ws)]
        ts = []
        for it in range(warmup + reps):
            dist.barrier(group=group)
            t0 = time.perf_counter()
            dist.all_gather(parts, buf, group=group)
            if dev.type == "cuda":
                torch.cuda.synchronize()
            if it >= warmup:
                ts.append(time.perf_counter() - t0)
        med = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev)
        dist.all_reduce(med, op=dist.ReduceOp.MAX, group=group)
        out.append(float(med.item()))
    return out


def time_allreduce(sizes_bytes, reps: int = 20, warmup: int = 5, device=None, group=None):
    """Median wall time of dist.all_reduce per message size (float32 buffers), max over the
    ranks of the group.  CUDA tensors are timed with CUDA events on the current stream."""
    import torch
    import torch.distributed as dist
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if torch.cuda.is_available() else torch.device("cpu"))
    out = []
    for m in sizes_bytes:
        n = max(1, int(m) // 4)
        buf = torch.ones(n, dtype=torch.float32, device=dev)
        for _ in range(warmup):
            dist.all_reduce(buf, group=group)
        ts = []
        for _ in range(reps):
            if dev.type == "cuda":
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                dist.barrier(group=group)
                a.record()
                dist.all_reduce(buf, group=group)
                b.record()
                b.synchronize()
                ts.append(a.elapsed_time(b) * 1e-3)
            else:
                dist.barrier(group=group)
                t0 = time.perf_counter()
                dist.all_reduce(buf, group=group)
                ts.append(time.perf_counter() - t0)
        med = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev)
        dist.all_reduce(med, op=dist.ReduceOp.MAX, group=group)
        out.append(float(med.item()))
    return out


def calibrate_tier(sizes_bytes=None, reps: int = 20, device=None, group=None):
    """One tier of the system (alpha, beta per PE-count level): the group's
    size p, measured Allreduce times and the fitted alpha / beta."""
    import torch.distributed as dist
    p = dist.get_world_size(group)
    sizes = list(sizes_bytes) if sizes_bytes is not None else [1 << e for e in range(16, 29, 2)]
    ts = time_allreduce(sizes, reps=reps, device=device, group=group)
    alpha, beta, rms = fit_allreduce(p, sizes, ts)
    return {"p": p, "alpha_s": alpha, "beta_s_per_B": beta, "fit_rms_rel": rms,
            "sizes_B": sizes, "times_s": ts}


def system_from_tiers(tiers, flops_per_s: float, hbm_bytes: float, **kw) -> W.System:
    """A sweep System whose tiers are calibrated ones (increasing p); max_pes = p."""
    ts = sorted(tiers, key=lambda d: d["p"])
    return W.System(tiers=[W.Tier(int(d["p"]), float(d["alpha_s"]), float(d["beta_s_per_B"])) for d in ts],
                    flops_per_s=flops_per_s, hbm_bytes=hbm_bytes, **kw)


# ------------------------------------------------------------------ per-layer compute
def _conv_args(r):
    stride = max(1, round(r.X[0] / r.Y[0])) if r.Y[0] else 1
    return stride, r.K[0] // 2


def time_layers(model: M.Model, b: int = 32, reps: int = 10, warmup: int = 3, device=None, dtype=None):
    """Per-sample forward and backward seconds of every CONV (2D) / FC row, timed with torch
    at batch b (None for rows that are not timed: pooling / element-wise rows, 3D convs,
    folded rows whose shortcut is not a plain conv).  Backward = forward+backward - forward."""
    import torch
    import torch.nn.functional as F
    dev = device if device is not None else torch.device("cuda" if torch.cuda.is_available() else "cpu")
    dt = dtype or torch.float32

    def clock(fn):
        for _ in range(warmup):
            fn()
        if dev.type == "cuda":
            torch.cuda.synchronize()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                fn()
            e.record()
            e.synchronize()
            return a.elapsed_time(e) * 1e-3 / reps
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        return (time.perf_counter() - t0) / reps

    out = []
    for r in model.layers:
        if r.kind == M.CONV and r.ndim == 2 and not (r.flags & M.FLAG_FOLDED):
            stride, pad = _conv_args(r)
            x = torch.randn(b, r.C, r.X[0], r.X[1], device=dev, dtype=dt, requires_grad=True)
            w = torch.randn(r.F, r.C, r.K[0], r.K[1], device=dev, dtype=dt, requires_grad=True)
            y = F.conv2d(x, w, stride=stride, padding=pad)
            if tuple(y.shape[2:]) != (r.Y[0], r.Y[1]):
                out.append(None)
                continue
            g = torch.ones_like(y)
            tf = clock(lambda: F.conv2d(x, w, stride=stride, padding=pad))
            tfb = clock(lambda: torch.autograd.grad(F.conv2d(x, w, stride=stride, padding=pad), (x, w), g))
        elif r.kind == M.FC:   # FC over the whole per-sample input: x -> y features
            x = torch.randn(b, r.x, device=dev, dtype=dt, requires_grad=True)
            w = torch.randn(r.y, r.x, device=dev, dtype=dt, requires_grad=True)
            g = torch.ones(b, r.y, device=dev, dtype=dt)
            tf = clock(lambda: F.linear(x, w))
            tfb = clock(lambda: torch.autograd.grad(F.linear(x, w), (x, w), g))
        else:
            out.append(None)
            continue
        out.append((tf / b, max(tfb - tf, 0.0) / b))
    return out


def empirical_model(model: M.Model, times, R_ref: float) -> M.Model:
    """Copy of the layer table whose fw / bw are effective FLOPs t * R_ref (so that the
    library's FW_l = fw / R with R = R_ref is the measured per-sample time).  Rows without a
    timing keep their FLOP counts rescaled by the measured effective rate of the timed rows
    (sum of their FLOPs / sum of their times)."""
    flops = sum(r.fw + r.bw for r, t in zip(model.layers, times) if t is not None)
    secs = sum(t[0] + t[1] for t in times if t is not None)
    r_eff = flops / secs if secs > 0 else R_ref
    m = copy.deepcopy(model)
    for r, t in zip(m.layers, times):
        if t is not None:
            r.fw, r.bw = max(1, round(t[0] * R_ref)), max(1, round(t[1] * R_ref))
        else:
            r.fw = max(1 if r.fw else 0, round(r.fw * R_ref / r_eff))
            r.bw = max(1 if r.bw else 0, round(r.bw * R_ref / r_eff))
    m.name = model.name + "-measured"
    m.meta = dict(model.meta, effective_flops_per_s=r_eff, R_ref=R_ref)
    return m
