"""Brute-force / exact-rational re-derivations used to PIN the oracle (test code only).

Written directly from PAPER.md, independently of oracle/oracle.c:
  * enumerate(): the canonical index order by itertools (no unranking arithmetic);
  * exact(): Table 2 per-iteration terms with per-layer sums in fractions.Fraction;
  * ring_allreduce_sim / ring_allgather_sim: explicit ring data movement;
  * gpipe_makespan: discrete-event GPipe schedule;
  * buffer_bytes: enumeration of every per-layer buffer.
"""
from __future__ import annotations

import itertools
from fractions import Fraction as Fr
from math import prod

from workloads import models as M
from workloads import sweeps as W

R_SCALING, R_MEMORY, R_SPLIT, R_TIER, R_SEGMENTS = 1, 2, 4, 8, 16


# ------------------------------------------------------------------ enumeration
def partitions(G, sub, model=None):
    if sub.family == W.LAYERWISE:
        # one strategy bit per COMM row (Q39): every assignment, mask value ascending
        nc = sum(1 for r in model.layers if r.flags & M.FLAG_COMM)
        return [("lw", mask) for mask in range(1 << nc)]
    if sub.family not in W.PIPE_FAMILIES:
        return [(G,)]
    if sub.part_mode == W.PART_MASK:
        out = []
        for mask in range(1 << (G - 1)):
            ends = [j + 1 for j in range(G - 1) if (mask >> j) & 1] + [G]
            out.append(tuple(ends))
        return out
    out = []
    for s in range(sub.s_min, sub.s_max + 1):
        for cuts in itertools.combinations(range(1, G), s - 1):
            out.append(tuple(cuts) + (G,))
    return out


def enumerate_configs(sweep):
    """Yield (idx, cfg dict) in canonical order: cap, flops, b, partition, S, dims, Ls, alpha, beta."""
    sys = sweep.system
    idx = 0
    for si, sub in enumerate(sweep.subs):
        m = sweep.models[sub.model]
        caps = sub.cap or [sys.hbm_bytes]
        flops = sub.flops or [sys.flops_per_s]
        Ss = sub.S or [1]
        dimss = sub.dims or [(1, 1, 1, 1)]
        Lss = sub.Ls or [0]
        alphas = sub.alpha or [[t.alpha for t in sys.tiers]]
        betas = sub.beta or [[t.beta for t in sys.tiers]]
        parts = partitions(m.G, sub, m)
        for cap, R, b, part, S, dims, Ls, a, bb in itertools.product(
                caps, flops, sub.b, parts, Ss, dimss, Lss, alphas, betas):
            yield idx, dict(sub=si, family=sub.family, model=sub.model, cap=cap, R=R, b=b,
                            ends=part, S=S, dims=dims, Ls=Ls, alpha=a, beta=bb)
            idx += 1


# ------------------------------------------------------------------ exact evaluation
def tier_of(sys, span):
    for t, tr in enumerate(sys.tiers):
        if tr.max_pes >= span:
            return t
    return None


def _ceil(a, b):
    return -(-a // b)


def halo_rows(layer, split, which):
    """halo(x) (which=0) / halo(dL/dy) (which=1) of one row, elements per sample (Q15)."""
    tot = 0
    for a in range(3):
        if split[a] <= 1:
            continue
        h = layer.K[a] // 2
        if h == 0:
            continue
        ext = layer.X if which == 0 else layer.Y
        ch = layer.C if which == 0 else layer.F
        cross = prod(_ceil(ext[o], split[o]) for o in range(3) if o != a)
        tot += ch * h * cross * (2 if split[a] > 2 else 1)
    return tot


def ar_exact(sys, n, m, seg, alpha, beta):
    if n == 1:
        return Fr(0)
    if sys.tree_threshold > 0 and m < Fr(sys.tree_threshold):
        lg = 0
        while (1 << lg) < n:
            lg += 1
        return 2 * (lg + sys.tree_chunks) * (alpha + m / (2 * sys.tree_chunks) * beta)
    return 2 * (n - 1) * (alpha + seg * beta)


def exact(sweep, cfg):
    """Per-iteration Table 2 terms in exact rationals with literal per-layer sums."""
    sys = sweep.system
    m = sweep.models[cfg["model"]]
    L = m.layers
    fam = cfg["family"]
    b = cfg["b"]
    tau = Fr(1) / Fr(cfg["R"])
    dl = sys.delta
    A = [Fr(v) for v in cfg["alpha"]]
    Bt = [Fr(v) for v in cfg["beta"]]
    # point-to-point patterns (Q40): the tier's parameters times the p2p scales, each product
    # rounded to double as the system would hold it
    Ap = [Fr(float(v) * sys.p2p_alpha_scale) for v in cfg["alpha"]]
    Bp = [Fr(float(v) * sys.p2p_beta_scale) for v in cfg["beta"]]
    gamma = Fr(sys.gamma)
    p1, d1, d2, d3 = cfg["dims"]
    reason = 0
    comp = ge = ag = ar = halo = p2p = Fr(0)
    inf = None

    comm_rows = [l for l, r in enumerate(L) if r.flags & M.FLAG_COMM]
    Cm = comm_rows[:-1]
    FW = sum(r.fw for r in L)
    BW = sum(r.bw for r in L)

    def comp_row(Bc, pc, pu):
        return Fr(Bc, pc) * (FW + BW) * tau + Fr(sum(r.wu for r in L), pu) * tau

    def mem_row(Bm, pa, pw):
        return gamma * dl * sum(Fr(2 * Bm * (r.x + r.y), pa) + Fr(2 * r.w, pw) + r.bi for r in L)

    def tier(span):
        nonlocal reason
        t = tier_of(sys, span)
        if t is None:
            reason |= R_TIER
        return t

    W_ = sum(r.w for r in L)
    if fam == W.SERIAL:
        B, p = b, 1
        comp = comp_row(B, 1, 1)
        mem = mem_row(B, 1, 1)
    elif fam == W.DATA:
        p = p1
        B = b * p
        comp = comp_row(B, p, 1)
        t = tier(p)
        ge = inf if t is None else ar_exact(sys, p, Fr(dl * W_), Fr(dl * W_, p), A[t], Bt[t])
        mem = mem_row(B, p, 1)
        if p > B:
            reason |= R_SCALING
    elif fam in (W.SPATIAL, W.DS):
        split = (d1, d2, d3)
        p2 = d1 * d2 * d3
        p = p1 * p2
        B = b * p1
        comp = comp_row(B, p, 1)
        Sp = [r for l, r in enumerate(L) if l < cfg["Ls"] and r.kind in (M.CONV, M.POOL)]
        for r in Sp:
            for a in range(3):
                if split[a] <= 1:
                    continue
                if split[a] > r.X[a]:
                    reason |= R_SCALING
                h = r.K[a] // 2
                if _ceil(r.X[a], split[a]) < h or _ceil(r.Y[a], split[a]) < h:
                    reason |= R_SPLIT
        ti, to = tier(p2), tier(p)
        if p2 > 1:
            halo = inf if ti is None else 2 * sum(
                2 * Ap[ti] + b * dl * Bp[ti] * (halo_rows(r, split, 0) + halo_rows(r, split, 1)) for r in Sp)
        if fam == W.SPATIAL:
            ge = inf if to is None else ar_exact(sys, p, Fr(dl * W_), Fr(dl * W_, p), A[to], Bt[to])
        else:
            phi = Fr(float(cfg["beta"][ti]) * sys.phi_ds) if (ti is not None and p1 > 1) else None
            rl = inf if ti is None else ar_exact(sys, p2, Fr(dl * W_), Fr(dl * W_, p2), A[ti],
                                                 phi if phi is not None else Bt[ti])
            al = inf if to is None else ar_exact(sys, p1, Fr(dl * W_), Fr(dl * W_, p1), A[to], Bt[to])
            ge = inf if (rl is None or al is None) else rl + al
        mem = mem_row(B, p, 1)
    elif fam == W.DATA_LW:
        # data parallelism, one Allreduce per weighted layer, ring or tree per message (Q37)
        p = p1
        B = b * p
        comp = comp_row(B, p, 1)
        t = tier(p)
        ge = inf if t is None else sum(ar_exact(sys, p, Fr(dl * r.w), Fr(dl * r.w, p), A[t], Bt[t])
                                       for r in L if r.w > 0)
        mem = mem_row(B, p, 1)
        if p > B:
            reason |= R_SCALING
    elif fam == W.LAYERWISE:
        # per-layer data / filter strategy over the same p PEs (Q39): every
        # row is evaluated with its own Table 2 row (Data P:469-473 with b samples, Filter
        # P:493-498 with all B samples) and the activations cross a strategy change by one
        # Allgather (D -> F forward, F -> D backward) and one Reduce-Scatter (D -> F
        # backward) of the b-sample boundary tensor
        p = p1
        B = b * p
        mask = cfg["ends"][1]
        strat = []
        cur = None
        j = 0
        for r in L:
            if r.flags & M.FLAG_COMM:
                cur = (mask >> j) & 1
                j += 1
            strat.append(cur)
        first = next((s_ for s_ in strat if s_ is not None), 0)
        strat = [first if s_ is None else s_ for s_ in strat]
        comp = sum(Fr(B, p) * (r.fw + r.bw) * tau for r in L) + sum(Fr(r.wu, p if f else 1) * tau
                                                                    for r, f in zip(L, strat))
        t = tier(p)
        has_d = not comm_rows or any(strat[l] == 0 for l in comm_rows)
        if has_d:
            WD = sum(r.w for r, f in zip(L, strat) if not f)
            ge = inf if t is None else ar_exact(sys, p, Fr(dl * WD), Fr(dl * WD, p), A[t], Bt[t])
        n_f = sum(1 for l in comm_rows if strat[l])
        changes = sum(1 for i in range(1, len(comm_rows)) if strat[comm_rows[i]] != strat[comm_rows[i - 1]])
        if p > 1 and (n_f or changes):
            if t is None:
                ag = ar = inf
            else:
                msg = [A[t] + Fr(B * L[l].y, p) * dl * Bt[t] for l in Cm if strat[l]]
                agf = (p - 1) * sum(msg)
                tr = Fr(0)
                for i in range(1, len(comm_rows)):
                    l = comm_rows[i]
                    if strat[l] != strat[comm_rows[i - 1]]:
                        one = (p - 1) * (A[t] + b * L[l - 1].y * dl * Bt[t])
                        tr += 2 * one if strat[l] else one
                ag = agf + tr
                ar = (1 if sys.filter_rs else 2) * agf
        mem = gamma * dl * sum(Fr(2 * B * (r.x + r.y), 1 if f else p) + Fr(2 * r.w, p if f else 1) + r.bi
                               for r, f in zip(L, strat))
        lim = min((L[l].F for l in comm_rows if strat[l]), default=None)
        if lim is not None and p > lim:
            reason |= R_SCALING
    elif fam == W.SPATIAL_AG:
        # spatial on rows [0, Ls), Allgather of y_Ls, rows [Ls, G) replicated (Q35)
        split = (d1, d2, d3)
        p = d1 * d2 * d3
        B = b
        Lp = min(cfg["Ls"], len(L))
        comp = (sum(Fr(B, p) * (r.fw + r.bw) * tau for r in L[:Lp])
                + sum(B * (r.fw + r.bw) * tau for r in L[Lp:]) + sum(r.wu for r in L) * tau)
        Sp = [r for r in L[:Lp] if r.kind in (M.CONV, M.POOL)]
        for r in Sp:
            for a in range(3):
                if split[a] <= 1:
                    continue
                if split[a] > r.X[a]:
                    reason |= R_SCALING
                h = r.K[a] // 2
                if _ceil(r.X[a], split[a]) < h or _ceil(r.Y[a], split[a]) < h:
                    reason |= R_SPLIT
        t = tier(p)
        if p > 1:
            halo = inf if t is None else 2 * sum(
                2 * Ap[t] + b * dl * Bp[t] * (halo_rows(r, split, 0) + halo_rows(r, split, 1)) for r in Sp)
            if Lp < len(L):
                ag = inf if t is None else (p - 1) * (A[t] + Fr(B * L[Lp - 1].y, p) * dl * Bt[t])
        ge = inf if t is None else ar_exact(sys, p, Fr(dl * W_), Fr(dl * W_, p), A[t], Bt[t])
        mem = gamma * dl * sum(Fr(2 * B * (r.x + r.y), p if l < Lp else 1) + 2 * r.w + r.bi
                               for l, r in enumerate(L))
    elif fam in (W.FILTER, W.CHANNEL):
        p = p1
        B = b
        comp = comp_row(B, p, p)
        t = tier(p)
        if p > 1:
            ag = inf if t is None else (p - 1) * sum(A[t] + Fr(B * L[l].y, p) * dl * Bt[t] for l in Cm)
            ar = inf if t is None else (1 if sys.filter_rs else 2) * (p - 1) * sum(A[t] + Fr(B * L[l].y, p) * dl * Bt[t] for l in Cm)
        mem = mem_row(B, 1, p)
        if fam == W.FILTER:
            lim = min((L[l].F for l in comm_rows), default=None)
        else:
            lim = min((L[l].C for l in comm_rows[1:]), default=None)
        if lim is not None and p > lim:
            reason |= R_SCALING
    elif fam == W.DF:
        p2 = d1
        p = p1 * p2
        B = b * p1
        comp = comp_row(B, p, p2)
        ti, to = tier(p2), tier(p)
        if p2 > 1:
            ag = inf if ti is None else (p2 - 1) * sum(A[ti] + Fr(B * L[l].y, p) * dl * Bt[ti] for l in Cm)
            ar = inf if ti is None else (1 if sys.filter_rs else 2) * (p2 - 1) * sum(A[ti] + Fr(B * L[l].y, p) * dl * Bt[ti] for l in Cm)
        phi = Fr(sys.phi_df) if p2 > 1 else Fr(1)
        if to is None:
            ge = inf if p1 > 1 else Fr(0)
        else:
            ge = ar_exact(sys, p1, Fr(dl * W_, p2), Fr(dl * W_, p), A[to], Bt[to] * phi)
        mem = mem_row(B, p1, p2)
        lim = min((L[l].F for l in comm_rows), default=None)
        if lim is not None and p2 > lim:
            reason |= R_SCALING
    else:
        ends = cfg["ends"]
        s = len(ends)
        S = cfg["S"]
        pd = p1 if fam == W.PD else 1
        p = s * pd
        B = b * pd
        groups = []
        beg = 0
        for e in ends:
            groups.append(L[beg:e])
            beg = e
        FWg = [sum(r.fw for r in g) * tau for g in groups]
        BWg = [sum(r.bw for r in g) * tau for g in groups]
        WUg = [sum(r.wu for r in g) * tau for g in groups]
        Wg = [sum(r.w for r in g) for g in groups]
        ycut = [g[-1].y for g in groups[:-1]]
        ts = tier(s)
        if fam == W.GPIPE:
            # GPipe schedule time by the identical-job flow-shop closed form (Q36): a flow
            # shop of S identical jobs over stage times t_1..t_m finishes its last job at
            # stage m at sum(t) + (S-1) max(t); forward stage i is busy f_i + c_i (blocking
            # send), backward stage i is busy g_i + c_{i-1}, all backward jobs are released
            # at the forward makespan, and stage i applies WU after its last backward job.
            mb = Fr(b, S)
            if ts is None:
                comp = inf
            else:
                c = [Ap[ts] + mb * dl * y * Bp[ts] for y in ycut] + [Fr(0)]
                d = [mb * FWg[i] + c[i] for i in range(s)]
                e = [mb * BWg[i] + (c[i - 1] if i > 0 else 0) for i in range(s)]
                t_f = sum(d) + (S - 1) * max(d)
                comp = max(t_f + sum(e[i:]) + (S - 1) * max(e[i:]) + WUg[i] for i in range(s))
        elif fam == W.LAYERPURE:
            comp = comp_row(b, 1, 1)
            if s > 1:
                p2p = inf if ts is None else 2 * sum(Ap[ts] + dl * b * y * Bp[ts] for y in ycut)
        else:
            comp = Fr(s + S - 1, S) * b * (max(FWg) + max(BWg)) + max(WUg)
            if s > 1:
                p2p = inf if ts is None else 2 * (s + S - 2) * max(Ap[ts] + Fr(b, S) * y * dl * Bp[ts] for y in ycut)
            if fam == W.PD:
                tp = tier(p)
                if tp is None:
                    ge = inf if pd > 1 else Fr(0)
                else:
                    mW = dl * max(Wg)
                    bh = Fr(float(cfg["beta"][tp]) * sys.phi_pd) if s > 1 else Bt[tp]
                    ge = ar_exact(sys, pd, Fr(mW), Fr(mW, pd), A[tp], bh)
        mem = gamma * dl * max(sum(2 * b * (r.x + r.y) + 2 * r.w + r.bi for r in g) for g in groups)
        if S < 1 or S > b:
            reason |= R_SEGMENTS
    terms = [comp, ge, ag, ar, halo, p2p]
    t_iter = None if any(v is None for v in terms) else sum(terms)
    if not (mem <= Fr(cfg["cap"])):
        reason |= R_MEMORY
    I = Fr(m.D, B)
    return dict(t_comp=comp, t_ge=ge, t_fb_ag=ag, t_fb_ar=ar, t_halo=halo, t_p2p=p2p,
                t_iter=t_iter, I=I, t_epoch=None if t_iter is None else t_iter * I,
                mem=mem, reason=reason, B=B, p=p)


# ------------------------------------------------------------------ simulators
def ring_allreduce_sim(p, m, alpha, beta):
    """Explicit ring reduce-scatter + allgather over p PEs of an m-byte buffer in p chunks
    (P:553-555).  Returns (time, final buffers) with exact rationals."""
    if p == 1:
        return Fr(0), None
    seg = Fr(m, p)
    # data[i][c] = contribution of PE i to chunk c (use distinct primes to check the sum)
    vals = [[(i + 1) * 1000 + c for c in range(p)] for i in range(p)]
    acc = [list(v) for v in vals]
    t = Fr(0)
    for step in range(p - 1):            # reduce-scatter
        sends = [(i, (i - step) % p, acc[i][(i - step) % p]) for i in range(p)]
        for i, c, v in sends:
            acc[(i + 1) % p][c] += v
        t += alpha + seg * beta
    owner = {}
    for i in range(p):
        owner[(i + 1) % p] = (i + 1) % p
    for step in range(p - 1):            # allgather
        sends = [(i, (i + 1 - step) % p, acc[i][(i + 1 - step) % p]) for i in range(p)]
        for i, c, v in sends:
            acc[(i + 1) % p][c] = v
        t += alpha + seg * beta
    return t, acc


def concurrent_rings_sim(group_bytes, p, alpha, beta):
    """pd gradient exchange (Q17): one ring Allreduce per pipeline stage, each among
    the p replicas of that stage, all stages at once over disjoint PE groups.  A discrete-
    event run: every group owns its PEs and links, so a step of group g starts when that
    group's previous step ends; a step sends one chunk per PE (reduce-scatter, then
    allgather) and the reduced buffers are checked.  Returns the makespan (exact rationals)."""
    if p == 1:
        return Fr(0)
    clock = [Fr(0)] * len(group_bytes)
    accs = []
    for g, m in enumerate(group_bytes):
        seg = Fr(m, p)
        acc = [[(i + 1) * 1000 + c + 7 * g for c in range(p)] for i in range(p)]
        events = []
        for step in range(p - 1):
            events.append(("rs", step))
        for step in range(p - 1):
            events.append(("ag", step))
        for kind, step in events:            # interleaving across groups cannot matter:
            if kind == "rs":                 # links and PEs are disjoint
                sends = [(i, (i - step) % p, acc[i][(i - step) % p]) for i in range(p)]
                for i, c, v in sends:
                    acc[(i + 1) % p][c] += v
            else:
                sends = [(i, (i + 1 - step) % p, acc[i][(i + 1 - step) % p]) for i in range(p)]
                for i, c, v in sends:
                    acc[(i + 1) % p][c] = v
            clock[g] += alpha + seg * beta
        accs.append(acc)
    for g, acc in enumerate(accs):
        col = [sum((i + 1) * 1000 + c + 7 * g for i in range(p)) for c in range(p)]
        assert all(row == col for row in acc)
    return max(clock)


def contended_stage_rings_sim(s, pd, node, m_bytes, alpha, beta):
    """pd gradient exchange with contention (Q40): PEs numbered replica-major (PE =
    r s + i for stage i of replica r), `node` PEs per node; stage i's ring Allreduce runs
    over PEs i, s + i, ..., (pd - 1) s + i, all s rings at once and in lockstep.  Every ring
    step sends one m/pd segment from each member to the next; a directed inter-node link
    carrying f flows gives each flow 1/f of its bandwidth (beta x f), so a step lasts
    alpha + seg beta (the busiest link's flow count).  Returns (makespan, flows on the busiest
    link) in exact rationals -- the contention coefficient phi is counted, not assumed."""
    if pd == 1:
        return Fr(0), 0
    seg = Fr(m_bytes, pd)
    t = Fr(0)
    worst = 0
    for step in range(2 * (pd - 1)):
        flows = {}
        msgs = []
        for i in range(s):
            for r in range(pd):
                a, b = r * s + i, ((r + 1) % pd) * s + i
                na, nb = a // node, b // node
                msgs.append((i, na, nb))
                if na != nb:
                    flows[(na, nb)] = flows.get((na, nb), 0) + 1
        f = max(flows.values(), default=1)
        worst = max(worst, f)
        t += alpha + seg * beta * f
    return t, worst


def ring_allgather_sim(p, m_seg, alpha, beta):
    if p == 1:
        return Fr(0)
    have = [{i} for i in range(p)]
    t = Fr(0)
    for step in range(p - 1):
        sends = [(i, (i - step) % p) for i in range(p)]
        for i, c in sends:
            assert c in have[i]
            have[(i + 1) % p].add(c)
        t += alpha + Fr(m_seg) * beta
    assert all(len(h) == p for h in have)
    return t


def gpipe_makespan(fw_stage, bw_stage, S, seg_samples):
    """Discrete-event GPipe schedule: forward wave of S segments through the stages, then
    the backward wave in reverse stage order.  Times per segment = samples x
    per-sample stage time."""
    s = len(fw_stage)
    done = [[Fr(0)] * S for _ in range(s)]
    free = [Fr(0)] * s
    for j in range(S):
        for i in range(s):
            start = max(free[i], done[i - 1][j] if i > 0 else Fr(0))
            done[i][j] = start + seg_samples * fw_stage[i]
            free[i] = done[i][j]
    t_fwd = max(free)
    bdone = [[Fr(0)] * S for _ in range(s)]
    bfree = [t_fwd] * s
    for j in range(S):
        for i in reversed(range(s)):
            start = max(bfree[i], bdone[i + 1][j] if i < s - 1 else t_fwd)
            bdone[i][j] = start + seg_samples * bw_stage[i]
            bfree[i] = bdone[i][j]
    return max(bfree)


def buffer_bytes(sweep, cfg):
    """Enumerate every buffer one PE holds (input, activation, their gradients, weights,
    weight gradients, bias -- P:538 / P:942) with its sharded size; sum x delta x gamma."""
    sys = sweep.system
    L = sweep.models[cfg["model"]].layers
    fam = cfg["family"]
    b = cfg["b"]
    p1, d1, d2, d3 = cfg["dims"]
    dl = sys.delta

    def layer_bufs(r, act_samples, act_div, w_div):
        bufs = [Fr(act_samples * r.x, act_div), Fr(act_samples * r.y, act_div),      # x, y
                Fr(act_samples * r.x, act_div), Fr(act_samples * r.y, act_div),      # dL/dx, dL/dy
                Fr(r.w, w_div), Fr(r.w, w_div), Fr(r.bi)]                            # w, dL/dw, bi
        return sum(bufs)

    if fam == W.SERIAL:
        tot = sum(layer_bufs(r, b, 1, 1) for r in L)
    elif fam in (W.DATA, W.DATA_LW):
        tot = sum(layer_bufs(r, b * p1, p1, 1) for r in L)          # B' = B/p samples
    elif fam in (W.SPATIAL, W.DS):
        p2 = d1 * d2 * d3
        tot = sum(layer_bufs(r, b * p1, p1 * p2, 1) for r in L)     # spatial shard of the group batch
    elif fam == W.LAYERWISE:
        # data rows hold b = B/p samples and whole weights, filter rows all B samples and
        # 1/p of the weights (Q39)
        B = b * p1
        mask = cfg["ends"][1]
        strat, cur, j = [], None, 0
        for r in L:
            if r.flags & M.FLAG_COMM:
                cur = (mask >> j) & 1
                j += 1
            strat.append(cur)
        first = next((s_ for s_ in strat if s_ is not None), 0)
        strat = [first if s_ is None else s_ for s_ in strat]
        tot = sum(layer_bufs(r, B, 1, p1) if f else layer_bufs(r, B, p1, 1) for r, f in zip(L, strat))
    elif fam == W.SPATIAL_AG:
        p2 = d1 * d2 * d3
        Lp = min(cfg["Ls"], len(L))
        tot = sum(layer_bufs(r, b, p2 if l < Lp else 1, 1) for l, r in enumerate(L))   # prefix sharded
    elif fam in (W.FILTER, W.CHANNEL):
        tot = sum(layer_bufs(r, b, 1, p1) for r in L)               # full activations, w/p
    elif fam == W.DF:
        tot = sum(layer_bufs(r, b * p1, p1, d1) for r in L)
    else:
        groups = []
        beg = 0
        for e in cfg["ends"]:
            groups.append(L[beg:e])
            beg = e
        tot = max(sum(layer_bufs(r, b, 1, 1) for r in g) for g in groups)
    return Fr(sys.gamma) * dl * tot
