"""Tiny hand-built layer tables and sweeps for the worked examples (test inputs only)."""
from __future__ import annotations

from workloads import models as M
from workloads import sweeps as W


def row(kind=M.CONV, C=1, F=1, X=(1, 1, 1), Y=(1, 1, 1), K=(1, 1, 1), x=0, y=0, w=0, bi=0,
        fw=0, bw=0, wu=0, flags=M.FLAG_COMM | M.FLAG_FOLDED, ndim=2):
    return M.Layer("toy", kind, ndim, C, F, tuple(X), tuple(Y), tuple(K), x, y, w, bi, fw, bw, wu, flags)


def model(rows, D=100, Ls=None):
    return M.Model("toy", list(rows), D, default_Ls=len(rows) if Ls is None else Ls)


def system(alpha=0.0, beta=1.0, R=1.0, cap=1e30, delta=1, gamma=1.0, phi=1.0, tiers=None,
           tree_threshold=0.0, tree_chunks=1):
    tiers = tiers or [W.Tier(1 << 20, alpha, beta)]
    return W.System(tiers=tiers, flops_per_s=R, hbm_bytes=cap, delta=delta, gamma=gamma,
                    phi_df=phi, tree_threshold=tree_threshold, tree_chunks=tree_chunks)


def sweep(models, system, subs):
    if not isinstance(models, list):
        models = [models]
    return W.Sweep(models, system, subs, "toy")
