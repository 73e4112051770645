/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain scalar C, fp64, compiled with -O2 -ffp-contract=off (no FMA contraction,
 * no fast-math).  Every configuration is evaluated from scratch with literal
 * loops over the layer rows and pipeline stages: no hoisting, no prefix sums,
 * no tiling.  Sums of integer counts (elements, bytes, FLOPs) are exact int64;
 * each real-valued term is one fixed fp64 expression tree written next to the
 * paper passage it follows.  The trees are listed in DESIGN.md §2.3.
 *
 * Pins (tests/test_oracle_pins.py): SPEC.md worked examples re-derived from the
 * paper formulas, ring / pipeline / buffer brute-force simulators, an exact
 * rational (fractions.Fraction) evaluator, the per-layer literal fold
 * (or_eval_fold), Table 4 parameter counts and limits, degenerate identities.
 * Parity unpinned by the paper itself: the FLOP-based compute parametrisation
 * (Q28), gamma (Q22), the ds / pd compositions (Q16, Q17), the per-layer strategy
 * composition (LAYERWISE, Q39) and the p2p scales / pd, ds contention (Q40) -- pinned
 * by the self-consistency checks above and by simulators the paper's primitives define
 * (concurrent ring Allreduces for the pd exchange, with a link-level flow count for its
 * contention; ring Allgather / Reduce-Scatter for the LAYERWISE strategy changes; all-D /
 * all-F LAYERWISE == the Data / Filter rows bit for bit).  See DESIGN.md §2.4.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static __thread char g_err[256];
const char *or_last_error(void) { return g_err; }
#define FAIL(code, ...) do { snprintf(g_err, sizeof g_err, __VA_ARGS__); return (code); } while (0)

enum { E_INVAL = -1, E_OVERFLOW = -4, E_RANGE = -5 };

/* ------------------------------------------------------------------ integer helpers */
static int mul_ok(int64_t a, int64_t b, int64_t *r) { return !__builtin_mul_overflow(a, b, r); }

/* C(n, k) by the multiplicative formula in 128-bit (own implementation). */
static uint64_t binom(int64_t n, int64_t k)
{
    if (k < 0 || n < 0 || k > n) return 0;
    if (k > n - k) k = n - k;
    unsigned __int128 r = 1;
    for (int64_t i = 1; i <= k; i++) {
        r = r * (unsigned __int128)(n - k + i) / (unsigned __int128)i;
    }
    return (uint64_t)r;
}

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

static int64_t ceil_log2(int64_t n)
{
    int64_t l = 0;
    while (((int64_t)1 << l) < n) l++;
    return l;
}

/* ------------------------------------------------------------------ spec helpers */
static int64_t nz(int32_t n) { return n > 0 ? n : 1; }

static int64_t comm_rows(const or_model *m)
{
    int64_t n = 0;
    for (int64_t l = 0; l < m->G; l++) n += (m->rows[l].flags & OR_FLAG_COMM) != 0;
    return n;
}

static int part_count(const or_model *m, const or_sub *s, uint64_t *out)
{
    int fam = s->family;
    if (fam == OR_LAYERWISE) {
        /* one bit per COMM row: 1 = filter-parallel, 0 = data-parallel (Q39) */
        if (s->part_mode != OR_PART_MASK) FAIL(E_INVAL, "layerwise needs the mask partition mode");
        int64_t nc = comm_rows(m);
        if (nc > 62) FAIL(E_INVAL, "layerwise needs at most 62 COMM rows");
        *out = (uint64_t)1 << nc;
        return 0;
    }
    int is_pipe = (fam == OR_PIPELINE || fam == OR_LAYERPURE || fam == OR_PD || fam == OR_GPIPE);
    if (!is_pipe) {
        if (s->part_mode != OR_PART_NONE) FAIL(E_INVAL, "partition mode on a non-pipeline family");
        *out = 1;
        return 0;
    }
    int64_t G = m->G;
    if (s->part_mode == OR_PART_MASK) {
        if (G > 64) FAIL(E_INVAL, "mask mode needs G <= 64");
        *out = (G - 1 == 64) ? 0 : ((uint64_t)1 << (G - 1));
        return 0;
    }
    if (s->part_mode != OR_PART_COMB) FAIL(E_INVAL, "pipeline family needs a partition mode");
    if (s->s_min < 1 || s->s_max < s->s_min || s->s_max > G || s->s_max > OR_MAX_STAGES)
        FAIL(E_INVAL, "bad stage-count range");
    uint64_t t = 0;
    for (int64_t st = s->s_min; st <= s->s_max; st++) t += binom(G - 1, st - 1);
    *out = t;
    return 0;
}

static int sub_count(const or_model *models, int n_models, const or_system *sys,
                     const or_sub *s, uint64_t *out)
{
    if (s->model < 0 || s->model >= n_models) FAIL(E_INVAL, "bad model index");
    if (s->family < 0 || s->family >= OR_N_FAMILIES) FAIL(E_INVAL, "bad family");
    if (s->n_b <= 0) FAIL(E_INVAL, "empty batch list");
    if ((s->family == OR_SPATIAL || s->family == OR_DS || s->family == OR_SPATIAL_AG) && s->n_Ls <= 0)
        FAIL(E_INVAL, "spatial family needs an Ls list");
    if (s->family == OR_SPATIAL_AG)
        for (int i = 0; i < s->n_Ls; i++)
            if (s->Ls[i] < 1) FAIL(E_INVAL, "spatial_ag needs Ls >= 1");
    if (s->family == OR_GPIPE)
        for (int i = 0; i < s->n_S; i++)
            if (s->S[i] < 1) FAIL(E_INVAL, "gpipe needs S >= 1");
    if (s->n_alpha > 0 && sys->n_tiers <= 0) FAIL(E_INVAL, "no tiers");
    uint64_t np;
    int rc = part_count(&models[s->model], s, &np);
    if (rc) return rc;
    unsigned __int128 t = np;
    t *= (uint64_t)nz(s->n_cap);
    t *= (uint64_t)nz(s->n_flops);
    t *= (uint64_t)s->n_b;
    t *= (uint64_t)nz(s->n_S);
    t *= (uint64_t)nz(s->n_dims);
    t *= (uint64_t)nz(s->n_Ls);
    t *= (uint64_t)nz(s->n_alpha);
    t *= (uint64_t)nz(s->n_beta);
    if (t >> 63) FAIL(E_OVERFLOW, "sweep larger than 2^63");
    *out = (uint64_t)t;
    return 0;
}

int or_sweep_size(const or_model *models, int n_models, const or_system *sys,
                  const or_spec *spec, uint64_t *n_out)
{
    unsigned __int128 tot = 0;
    for (int i = 0; i < spec->n_sub; i++) {
        uint64_t c;
        int rc = sub_count(models, n_models, sys, &spec->subs[i], &c);
        if (rc) return rc;
        tot += c;
    }
    if (tot >> 63) FAIL(E_OVERFLOW, "sweep larger than 2^63");
    *n_out = (uint64_t)tot;
    return 0;
}

/* Lexicographic unranking of a k-subset {c_1<...<c_k} of {1..n}. */
static void unrank_lex(int64_t n, int64_t k, uint64_t r, int32_t *c)
{
    int64_t v = 0;
    for (int64_t j = 1; j <= k; j++) {
        for (v = v + 1;; v++) {
            uint64_t cnt = binom(n - v, k - j);
            if (r < cnt) break;
            r -= cnt;
        }
        c[j - 1] = (int32_t)v;
    }
}

/*
 * Canonical index order: sub-sweeps in spec order; inside one,
 * digits slow -> fast: cap, flops, b, partition, S, dims, Ls, alpha, beta.
 */
int or_decode(const or_model *models, int n_models, const or_system *sys,
              const or_spec *spec, uint64_t idx, or_config *c)
{
    memset(c, 0, sizeof *c);
    uint64_t u = idx;
    int si = -1;
    for (int i = 0; i < spec->n_sub; i++) {
        uint64_t n;
        int rc = sub_count(models, n_models, sys, &spec->subs[i], &n);
        if (rc) return rc;
        if (u < n) { si = i; break; }
        u -= n;
    }
    if (si < 0) FAIL(E_RANGE, "index outside the sweep");
    const or_sub *s = &spec->subs[si];
    const or_model *m = &models[s->model];
    c->sub = si;
    c->family = s->family;
    c->model = s->model;
    uint64_t np;
    part_count(m, s, &np);
    uint64_t r;
    r = nz(s->n_beta);  c->i_beta = (int64_t)(u % r);  u /= r;
    r = nz(s->n_alpha); c->i_alpha = (int64_t)(u % r); u /= r;
    r = nz(s->n_Ls);    c->i_Ls = (int64_t)(u % r);    u /= r;
    r = nz(s->n_dims);  c->i_dims = (int64_t)(u % r);  u /= r;
    r = nz(s->n_S);     c->i_S = (int64_t)(u % r);     u /= r;
    c->i_part = u % np; u /= np;
    r = s->n_b;         c->i_b = (int64_t)(u % r);     u /= r;
    r = nz(s->n_flops); c->i_flops = (int64_t)(u % r); u /= r;
    r = nz(s->n_cap);   c->i_cap = (int64_t)(u % r);   u /= r;

    c->cap = s->n_cap > 0 ? s->cap[c->i_cap] : sys->hbm_bytes;
    c->flops = s->n_flops > 0 ? s->flops[c->i_flops] : sys->flops_per_s;
    c->b = s->b[c->i_b];
    c->S = s->n_S > 0 ? s->S[c->i_S] : 1;
    for (int a = 0; a < 4; a++) c->dims[a] = s->n_dims > 0 ? s->dims[4 * c->i_dims + a] : 1;
    c->Ls = s->n_Ls > 0 ? s->Ls[c->i_Ls] : 0;
    for (int t = 0; t < sys->n_tiers; t++) {
        c->alpha[t] = s->n_alpha > 0 ? s->alpha[c->i_alpha * sys->n_tiers + t] : sys->tiers[t].alpha;
        c->beta[t] = s->n_beta > 0 ? s->beta[c->i_beta * sys->n_tiers + t] : sys->tiers[t].beta;
    }
    /* stage partition (groups g_i, P:519 footnote) */
    int64_t G = m->G;
    if (s->part_mode == OR_PART_NONE || s->family == OR_LAYERWISE) {
        c->n_stages = 1;
        c->stage_end[0] = (int32_t)G;
    } else if (s->part_mode == OR_PART_MASK) {
        /* bit j set <=> cut after row j+1 */
        int ns = 0;
        for (int64_t j = 0; j < G - 1; j++)
            if ((c->i_part >> j) & 1) c->stage_end[ns++] = (int32_t)(j + 1);
        c->stage_end[ns++] = (int32_t)G;
        c->n_stages = ns;
    } else {
        uint64_t rr = c->i_part;
        int64_t st = s->s_min;
        for (;; st++) {
            uint64_t blk = binom(G - 1, st - 1);
            if (rr < blk) break;
            rr -= blk;
        }
        int32_t cuts[OR_MAX_STAGES];
        unrank_lex(G - 1, st - 1, rr, cuts);
        for (int64_t j = 0; j < st - 1; j++) c->stage_end[j] = cuts[j];
        c->stage_end[st - 1] = (int32_t)G;
        c->n_stages = (int32_t)st;
    }
    return 0;
}

/* ------------------------------------------------------------------ cost model */

/* Tier lookup ("alpha and beta become different when changing the number of
 * processing elements"; Q29): smallest tier whose max_pes covers the communicator. */
static int tier_of(const or_system *sys, int64_t span)
{
    for (int t = 0; t < sys->n_tiers; t++)
        if (sys->tiers[t].max_pes >= span) return t;
    return -1;
}

/* Point-to-point parameters of tier t (Q40): the collective tier's alpha and beta times the
 * system's p2p scales ("we plugged different network parameters in ParaDL ... for MPI and
 * NCCL"). */
static double p2p_alpha(const or_system *sys, const or_config *c, int t) { return c->alpha[t] * sys->p2p_alpha_scale; }
static double p2p_beta(const or_system *sys, const or_config *c, int t) { return c->beta[t] * sys->p2p_beta_scale; }

/* Allreduce over n PEs of an m-byte buffer (P:556 ring: 2(p-1)(alpha + (m/p) beta);
 * P:559 footnote tree: 2(log p + k)(alpha + m/(2k) beta), Q18).  `seg` is the ring
 * step segment the caller's Table 2 row prints (m/p for data, sum|w|/p for df). */
static double t_allreduce(const or_system *sys, int64_t n, double m, double seg,
                          double alpha, double beta_hat)
{
    if (n == 1) return 0.0;
    if (sys->tree_threshold > 0.0 && m < sys->tree_threshold) {
        double c = (double)(2 * (ceil_log2(n) + sys->tree_chunks));
        return c * (alpha + (m / (double)(2 * sys->tree_chunks)) * beta_hat);
    }
    double c = (double)(2 * (n - 1));
    return c * (alpha + seg * beta_hat);
}

/* Literal per-model integer sums (Table 2's Sigma_l over the G rows). */
typedef struct {
    int64_t FB, WU, W, BI, XY;
    int64_t YC, NC;        /* filter/channel communication rows: COMM rows except the last (Q10) */
    int64_t Fmin, Cmin2;   /* min F over COMM rows (Q11); min C over COMM rows but the first (Q12) */
} sums_t;

static int model_sums(const or_model *m, sums_t *s)
{
    memset(s, 0, sizeof *s);
    s->Fmin = INT64_MAX;
    s->Cmin2 = INT64_MAX;
    int64_t last_comm = -1, first_comm = -1;
    for (int64_t l = 0; l < m->G; l++) {
        const or_layer *r = &m->rows[l];
        s->FB += r->fw + r->bw;
        s->WU += r->wu;
        s->W += r->w;
        s->BI += r->bi;
        s->XY += r->x + r->y;
        if (r->flags & OR_FLAG_COMM) {
            if (first_comm < 0) first_comm = l;
            last_comm = l;
            if (r->F < s->Fmin) s->Fmin = r->F;
        }
    }
    for (int64_t l = 0; l < m->G; l++) {
        const or_layer *r = &m->rows[l];
        if (!(r->flags & OR_FLAG_COMM)) continue;
        if (l != last_comm) { s->YC += r->y; s->NC += 1; }
        if (l != first_comm && r->C < s->Cmin2) s->Cmin2 = r->C;
    }
    return 0;
}

/* Halo volume ("a small number (e.g. K/2) of rows and/or columns";
 * P:985 "depends on how each spatial dimension is split"; Q15): per split axis a,
 * floor(K_a/2) planes of the PE's local cross-section, from 2 neighbours (1 if the
 * axis has 2 parts).  which = 0: halo(x) (C channels over the input grid X);
 * which = 1: halo(dL/dy) (F channels over the output grid Y). */
int64_t or_halo_elements(const or_layer *row, const int32_t split[3], int which)
{
    int64_t tot = 0;
    for (int a = 0; a < 3; a++) {
        if (split[a] <= 1) continue;
        int64_t h = row->K[a] / 2;
        if (h == 0) continue;
        const int64_t *ext = which == 0 ? row->X : row->Y;
        int64_t ch = which == 0 ? row->C : row->F;
        int64_t cross = 1;
        for (int b = 0; b < 3; b++)
            if (b != a) cross *= ceil_div(ext[b], split[b]);
        int64_t nnb = split[a] > 2 ? 2 : 1;
        tot += ch * h * cross * nnb;
    }
    return tot;
}

/* Spatial set Sp = Conv/Pool rows among the first Ls rows (Table 3, Q14). */
static uint32_t spatial_terms(const or_model *m, int32_t Ls, const int32_t split[3],
                              int64_t *NS, int64_t *HV)
{
    uint32_t reason = 0;
    *NS = 0;
    *HV = 0;
    for (int64_t l = 0; l < m->G && l < Ls; l++) {
        const or_layer *r = &m->rows[l];
        if (r->kind != OR_CONV && r->kind != OR_POOL) continue;
        *NS += 1;
        *HV += or_halo_elements(r, split, 0) + or_halo_elements(r, split, 1);
        for (int a = 0; a < 3; a++) {
            if (split[a] <= 1) continue;
            /* P:325 "pw, ph, pd <= W, H, D" (per axis, Q13) */
            if (split[a] > r->X[a]) reason |= OR_R_SCALING;
            /* local extent must hold the halo (SplitTooFine) */
            int64_t h = r->K[a] / 2;
            if (ceil_div(r->X[a], split[a]) < h || ceil_div(r->Y[a], split[a]) < h)
                reason |= OR_R_SPLIT;
        }
    }
    return reason;
}

/* Per-stage sums for a contiguous partition (FW_{G_i} = sum_{l in g_i} FW_l). */
typedef struct {
    int64_t maxF, maxB, maxU, maxW, maxY, sumY, memI;
} stage_t;

static int stage_terms(const or_model *m, const or_config *c, int64_t Bs, stage_t *st)
{
    memset(st, 0, sizeof *st);
    int64_t beg = 0;
    for (int i = 0; i < c->n_stages; i++) {
        int64_t end = c->stage_end[i];
        int64_t F = 0, Bw = 0, U = 0, W = 0, XY = 0, BI = 0;
        for (int64_t l = beg; l < end; l++) {
            const or_layer *r = &m->rows[l];
            F += r->fw;
            Bw += r->bw;
            U += r->wu;
            W += r->w;
            XY += r->x + r->y;
            BI += r->bi;
        }
        if (F > st->maxF) st->maxF = F;
        if (Bw > st->maxB) st->maxB = Bw;
        if (U > st->maxU) st->maxU = U;
        if (W > st->maxW) st->maxW = W;
        /* Table 2 pipeline memory: max_i sum_{l in g_i} (2B(|x|+|y|) + 2|w| + |bi|) (Q6) */
        int64_t a, mem;
        if (!mul_ok(2 * Bs, XY, &a)) FAIL(E_OVERFLOW, "2B*XY_i overflows int64");
        mem = a + 2 * W + BI;
        if (mem > st->memI) st->memI = mem;
        if (i < c->n_stages - 1) {
            /* boundary message: |y| of the last row of stage i (Q8) */
            int64_t y = m->rows[end - 1].y;
            if (y > st->maxY) st->maxY = y;
            st->sumY += y;
        }
        beg = end;
    }
    return 0;
}

static int tier_or_flag(const or_system *sys, int64_t span, uint32_t *reason)
{
    int t = tier_of(sys, span);
    if (t < 0) *reason |= OR_R_TIER;
    return t;
}

/* comp for a row of Table 2: ((B*FB)/p_c) tau + (WU/p_u) tau   (per iteration, Q1) */
static double comp_term(int64_t BFB, int64_t WU, int64_t pc, int64_t pu, double tau)
{
    return ((double)BFB / (double)pc) * tau + ((double)WU / (double)pu) * tau;
}

/* mem for a row of Table 2: gamma (delta ((2B XY)/p_a + (2W)/p_w + BI)) */
static double mem_term(const or_system *sys, int64_t twoBXY, int64_t W, int64_t BI,
                       int64_t pa, int64_t pw)
{
    return sys->gamma * ((double)sys->delta *
                         (((double)twoBXY / (double)pa + (double)(2 * W) / (double)pw) + (double)BI));
}

int or_eval(const or_model *models, const or_system *sys, const or_config *c, or_pred *o)
{
    memset(o, 0, sizeof *o);
    const or_model *m = &models[c->model];
    sums_t s;
    model_sums(m, &s);
    const double tau = 1.0 / c->flops;
    const int64_t delta = sys->delta;
    const int64_t b = c->b;
    uint32_t reason = 0;
    double comp = 0, ge = 0, ag = 0, ar = 0, halo = 0, p2p = 0, mem = 0;
    int64_t B = b, p = 1, tmp, BFB, twoBXY, dW;
    if (!mul_ok(delta, s.W, &dW)) FAIL(E_OVERFLOW, "delta*W");
    const int32_t *d = c->dims;

    switch (c->family) {
    case OR_SERIAL: {   /* Table 2 Serial row P:463-467; Appendix Eq. orig_time */
        B = b; p = 1;
        if (!mul_ok(B, s.FB, &BFB) || !mul_ok(2 * B, s.XY, &twoBXY)) FAIL(E_OVERFLOW, "B*FB");
        comp = comp_term(BFB, s.WU, 1, 1, tau);
        mem = mem_term(sys, twoBXY, s.W, s.BI, 1, 1);
        break;
    }
    case OR_DATA: {     /* Table 2 Data row P:469-473; Eqs. data_comp/comm/mem P:916-953 */
        p = d[0];
        if (!mul_ok(b, p, &B)) FAIL(E_OVERFLOW, "b*p");
        if (!mul_ok(B, s.FB, &BFB) || !mul_ok(2 * B, s.XY, &twoBXY)) FAIL(E_OVERFLOW, "B*FB");
        comp = comp_term(BFB, s.WU, p, 1, tau);
        int t = tier_or_flag(sys, p, &reason);
        ge = t < 0 ? INFINITY
                   : t_allreduce(sys, p, (double)dW, (double)dW / (double)p, c->alpha[t], c->beta[t]);
        mem = mem_term(sys, twoBXY, s.W, s.BI, p, 1);
        if (p > B) reason |= OR_R_SCALING;           /* p <= B */
        break;
    }
    case OR_SPATIAL:    /* Table 2 Spatial row P:475-481; Eqs. spatial_* P:954-985 */
    case OR_DS: {       /* data+spatial: prose only P:413, P:613, P:760-761 (Q16) */
        int64_t p1 = d[0];
        int32_t split[3] = {d[1], d[2], d[3]};
        int64_t p2 = (int64_t)d[1] * d[2] * d[3];
        if (c->family == OR_SPATIAL && p1 != 1) FAIL(E_INVAL, "spatial needs p1 == 1");
        p = p1 * p2;
        if (!mul_ok(b, p1, &B)) FAIL(E_OVERFLOW, "b*p1");
        if (!mul_ok(B, s.FB, &BFB) || !mul_ok(2 * B, s.XY, &twoBXY)) FAIL(E_OVERFLOW, "B*FB");
        comp = comp_term(BFB, s.WU, p, 1, tau);
        int64_t NS, HV, bdHV;
        reason |= spatial_terms(m, c->Ls, split, &NS, &HV);
        if (!mul_ok(b * delta, HV, &bdHV)) FAIL(E_OVERFLOW, "b*delta*HV");
        int ti = tier_or_flag(sys, p2, &reason);
        int to = tier_or_flag(sys, p, &reason);
        /* FB-Halo per iteration: 2 sum_{l in Sp}(2 alpha + b delta beta (halo(x_l)+halo(dy_l))) */
        if (p2 > 1)
            halo = ti < 0 ? INFINITY
                          : 2.0 * ((double)(2 * NS) * p2p_alpha(sys, c, ti) + (double)bdHV * p2p_beta(sys, c, ti));
        if (c->family == OR_SPATIAL) {
            ge = to < 0 ? INFINITY
                        : t_allreduce(sys, p, (double)dW, (double)dW / (double)p, c->alpha[to], c->beta[to]);
        } else {
            /* reduce to a leader inside the group, then Allreduce between leaders;
             * the p1 groups reduce at once: contention phi_ds when p1 > 1 (Q40) */
            const double phi = p1 > 1 ? sys->phi_ds : 1.0;
            double rl = ti < 0 ? INFINITY
                               : t_allreduce(sys, p2, (double)dW, (double)dW / (double)p2, c->alpha[ti],
                                             c->beta[ti] * phi);
            double al = to < 0 ? INFINITY
                               : t_allreduce(sys, p1, (double)dW, (double)dW / (double)p1, c->alpha[to], c->beta[to]);
            ge = rl + al;
        }
        mem = mem_term(sys, twoBXY, s.W, s.BI, p, 1);
        break;
    }
    case OR_FILTER:     /* Table 2 Filter row P:493-498; Eqs. filter_comm1/mem P:1038-1062 */
    case OR_CHANNEL: {  /* Table 2 Channel row P:500-505; Eqs. */
        p = d[0];
        B = b;
        if (!mul_ok(B, s.FB, &BFB) || !mul_ok(2 * B, s.XY, &twoBXY)) FAIL(E_OVERFLOW, "B*FB");
        comp = comp_term(BFB, s.WU, p, p, tau);
        int64_t BdYC;
        if (!mul_ok(B * delta, s.YC, &BdYC)) FAIL(E_OVERFLOW, "B*delta*YC");
        int t = tier_or_flag(sys, p, &reason);
        /* 3(p-1) sum_{l<G}(alpha + (B|y_l|/p) delta beta) = Allgather (1x) + Allreduce (2x) */
        if (p > 1) {
            ag = t < 0 ? INFINITY
                       : (double)(p - 1) * ((double)s.NC * c->alpha[t] + ((double)BdYC / (double)p) * c->beta[t]);
            ar = (sys->filter_rs ? 1.0 : 2.0) * ag;   /* Reduce-Scatter = one Allgather's cost (P:355 fn) */
        }
        mem = mem_term(sys, twoBXY, s.W, s.BI, 1, p);
        if (c->family == OR_FILTER ? (p > s.Fmin) : (p > s.Cmin2)) reason |= OR_R_SCALING;
        break;
    }
    case OR_DF: {       /* Table 2 Data+Filter row P:507-511; Eqs. hybrid_* P:1091-1122 (Q20) */
        int64_t p1 = d[0], p2 = d[1];
        if (d[2] != 1 || d[3] != 1) FAIL(E_INVAL, "df dims are (p1,p2,1,1)");
        p = p1 * p2;
        if (!mul_ok(b, p1, &B)) FAIL(E_OVERFLOW, "b*p1");
        if (!mul_ok(B, s.FB, &BFB) || !mul_ok(2 * B, s.XY, &twoBXY)) FAIL(E_OVERFLOW, "B*FB");
        comp = comp_term(BFB, s.WU, p, p2, tau);
        int64_t BdYC;
        if (!mul_ok(B * delta, s.YC, &BdYC)) FAIL(E_OVERFLOW, "B*delta*YC");
        int ti = tier_or_flag(sys, p2, &reason);
        int to = tier_or_flag(sys, p, &reason);
        if (p2 > 1) {
            ag = ti < 0 ? INFINITY
                        : (double)(p2 - 1) * ((double)s.NC * c->alpha[ti] + ((double)BdYC / (double)p) * c->beta[ti]);
            ar = (sys->filter_rs ? 1.0 : 2.0) * ag;   /* Reduce-Scatter = one Allgather's cost (P:355 fn) */
        }
        /* 2(p1-1)(alpha + (sum|w|/p) delta beta), contention phi on the shared link (Q30) */
        double phi = p2 > 1 ? sys->phi_df : 1.0;
        if (to < 0) ge = p1 > 1 ? INFINITY : 0.0;
        else ge = t_allreduce(sys, p1, (double)dW / (double)p2, (double)dW / (double)p,
                              c->alpha[to], c->beta[to] * phi);
        mem = mem_term(sys, twoBXY, s.W, s.BI, p1, p2);
        if (p2 > s.Fmin) reason |= OR_R_SCALING;
        break;
    }
    case OR_PIPELINE:   /* Table 2 Layer(Pipeline) row P:483-491; Eqs. pipe_* P:1005-1036 */
    case OR_LAYERPURE:  /* Eq. layer_comp */
    case OR_PD: {       /* pipeline + data, P:797 (composed, Q17) */
        int64_t ns = c->n_stages;
        int64_t S = c->S;
        int64_t pd = c->family == OR_PD ? d[0] : 1;
        if (c->family != OR_PD && d[0] != 1) FAIL(E_INVAL, "pipeline dims must be 1");
        p = ns * pd;
        if (!mul_ok(b, pd, &B)) FAIL(E_OVERFLOW, "b*pd");
        stage_t st;
        int rc = stage_terms(m, c, b, &st);
        if (rc) return rc;
        int ts = tier_or_flag(sys, ns, &reason);
        if (c->family == OR_LAYERPURE) {
            if (!mul_ok(b, s.FB, &BFB)) FAIL(E_OVERFLOW, "B*FB");
            comp = comp_term(BFB, s.WU, 1, 1, tau);
            int64_t dBY;
            if (!mul_ok(delta * b, st.sumY, &dBY)) FAIL(E_OVERFLOW, "delta*B*y");
            /* 2 sum_{i<p} T_p2p(delta B |y_{G_i}|) */
            if (ns > 1)
                p2p = ts < 0 ? INFINITY
                             : 2.0 * ((double)(ns - 1) * p2p_alpha(sys, c, ts) + (double)dBY * p2p_beta(sys, c, ts));
        } else {
            /* (p+S-1)(B/S)(max FW + max BW) + max WU  (per iteration, Q4/Q7) */
            double cseg = (double)(ns + S - 1) * ((double)b / (double)S);
            comp = (cseg * (double)(st.maxF + st.maxB)) * tau + (double)st.maxU * tau;
            /* 2(p+S-2) max_{i<p}(alpha + (B/S)|y_{G_i}| delta beta)  (Q5) */
            if (ns > 1)
                p2p = ts < 0 ? INFINITY
                             : (double)(2 * (ns + S - 2)) *
                                   (p2p_alpha(sys, c, ts) +
                                    (((double)b / (double)S) * (double)(delta * st.maxY)) * p2p_beta(sys, c, ts));
            if (c->family == OR_PD) {
                int tp = tier_or_flag(sys, p, &reason);
                double mW = (double)(delta * st.maxW);
                /* the s stage Allreduces run at once: contention phi_pd when s > 1 (Q40) */
                const double phi = ns > 1 ? sys->phi_pd : 1.0;
                if (tp < 0) ge = pd > 1 ? INFINITY : 0.0;
                else ge = t_allreduce(sys, pd, mW, mW / (double)pd, c->alpha[tp], c->beta[tp] * phi);
            }
        }
        mem = sys->gamma * ((double)delta * (double)st.memI);
        if (S < 1 || S > b) reason |= OR_R_SEGMENTS;   /* S <= B (Q9) */
        break;
    }
    case OR_DATA_LW: {
        /* Data row of Table 2 with the gradient exchanged as one Allreduce per
         * weighted layer (message delta |w_l|, row order), each message sent with the ring
         * algorithm when large and the tree algorithm when small: "ring-based algorithm for
         * ... large message sizes and a tree-based algorithm for small message sizes"
         * (P:552), tree time of the footnote (Q37).  GE = left fold over the layers. */
        p = d[0];
        if (d[1] != 1 || d[2] != 1 || d[3] != 1) FAIL(E_INVAL, "data_lw dims are (p,1,1,1)");
        if (!mul_ok(b, p, &B)) FAIL(E_OVERFLOW, "b*p");
        if (!mul_ok(B, s.FB, &BFB) || !mul_ok(2 * B, s.XY, &twoBXY)) FAIL(E_OVERFLOW, "B*FB");
        comp = comp_term(BFB, s.WU, p, 1, tau);
        int t = tier_or_flag(sys, p, &reason);
        if (t < 0) {
            ge = INFINITY;
        } else {
            for (int64_t l = 0; l < m->G; l++) {
                const int64_t w = m->rows[l].w;
                if (w <= 0) continue;
                const double ml = (double)(delta * w);
                ge = ge + t_allreduce(sys, p, ml, ml / (double)p, c->alpha[t], c->beta[t]);
            }
        }
        mem = mem_term(sys, twoBXY, s.W, s.BI, p, 1);
        if (p > B) reason |= OR_R_SCALING;
        break;
    }
    case OR_LAYERWISE: {
        /* "the hybrid strategy could be more complex when applying different parallel
         * strategies for different layers"; "there can be cases at which a
         * different type of parallelism is used ... the fully connected layer in spatial
         * parallelism is not spatially parallelized".  Q39: every COMM row (in row
         * order, bit j of the mask for the j-th) is data-parallel (0) or filter-parallel (1)
         * over the same p PEs; other rows follow the COMM row before them (the first COMM
         * row's strategy before it).  Mini-batch B = b p: a data row holds b samples and
         * the whole weights (Data row of Table 2), a filter row all B samples
         * and 1/p of the weights (Filter row).
         *   comp = ((B FB)/p) tau + (WU_D + WU_F/p) tau
         *   GE   = AR(p, delta W_D) over the data rows' weights (absent if every COMM row is F)
         *   AG   = (p-1)(NC_F alpha + (B delta YC_F / p) beta)  (filter rows' Allgathers, Q10)
         *        + (p-1)(n_T alpha + (b delta Y_T) beta)      (strategy changes, below)
         *   AR   = 2 x the filter rows' Allgather term (1 x with filter_rs, P:355 fn)
         *   mem  = gamma (delta (((2B XY_D)/p + 2B XY_F) + (2W_D + (2W_F)/p)) + BI))
         * A change D -> F at COMM row l gathers the b-sample activations y_{l-1} of every
         * PE (Allgather, forward) and reduce-scatters dL/dx back (backward); F -> D
         * gathers the b-sample gradients dL/dy_{l-1} (Allgather, backward): per-PE segment
         * b |y_{l-1}| each (P:553-556 ring steps), so n_T = 2 n_DF + n_FD and Y_T =
         * 2 sum_DF y_{l-1} + sum_FD y_{l-1}.  Limit: p <= min F over the filter COMM rows. */
        p = d[0];
        if (d[1] != 1 || d[2] != 1 || d[3] != 1) FAIL(E_INVAL, "layerwise dims are (p,1,1,1)");
        if (!mul_ok(b, p, &B)) FAIL(E_OVERFLOW, "b*p");
        const uint64_t mask = c->i_part;
        int64_t FB = 0, WUD = 0, WUF = 0, WD = 0, WF = 0, XYD = 0, XYF = 0, BI = 0;
        int64_t NCF = 0, YCF = 0, nT = 0, YT = 0, FminF = INT64_MAX, ncomm = 0, nF = 0;
        int64_t last_comm = -1, first_comm = -1;
        for (int64_t l = 0; l < m->G; l++)
            if (m->rows[l].flags & OR_FLAG_COMM) { if (first_comm < 0) first_comm = l; last_comm = l; }
        int cur = first_comm >= 0 ? (int)(mask & 1) : 0;   /* strategy of the rows: 0 D, 1 F */
        for (int64_t l = 0; l < m->G; l++) {
            const or_layer *r = &m->rows[l];
            if (r->flags & OR_FLAG_COMM) {
                int sf = (int)((mask >> ncomm) & 1);
                if (ncomm > 0 && sf != cur) {
                    const int64_t yb = m->rows[l - 1].y;
                    nT += sf ? 2 : 1;
                    YT += sf ? 2 * yb : yb;
                }
                cur = sf;
                ncomm++;
                if (cur) {
                    nF++;
                    if (r->F < FminF) FminF = r->F;
                    if (l != last_comm) { NCF += 1; YCF += r->y; }
                }
            }
            FB += r->fw + r->bw;
            BI += r->bi;
            if (cur) { WUF += r->wu; WF += r->w; XYF += r->x + r->y; }
            else     { WUD += r->wu; WD += r->w; XYD += r->x + r->y; }
        }
        int64_t BFB, tBXYD, tBXYF, BdYCF, bdYT, dWD;
        if (!mul_ok(B, FB, &BFB) || !mul_ok(2 * B, XYD, &tBXYD) || !mul_ok(2 * B, XYF, &tBXYF) ||
            !mul_ok(B * delta, YCF, &BdYCF) || !mul_ok(b * delta, YT, &bdYT) || !mul_ok(delta, WD, &dWD))
            FAIL(E_OVERFLOW, "layerwise sums");
        comp = ((double)BFB / (double)p) * tau + ((double)WUD + (double)WUF / (double)p) * tau;
        int t = tier_or_flag(sys, p, &reason);
        const int all_f = ncomm > 0 && nF == ncomm;
        if (!all_f)
            ge = t < 0 ? INFINITY
                       : t_allreduce(sys, p, (double)dWD, (double)dWD / (double)p, c->alpha[t], c->beta[t]);
        if (p > 1 && (nF > 0 || nT > 0)) {   /* no filter row and no change: no exchange at all */
            double agf = t < 0 ? INFINITY
                               : (double)(p - 1) * ((double)NCF * c->alpha[t] + ((double)BdYCF / (double)p) * c->beta[t]);
            double tr = t < 0 ? INFINITY
                              : (double)(p - 1) * ((double)nT * c->alpha[t] + (double)bdYT * c->beta[t]);
            ag = agf + tr;
            ar = (sys->filter_rs ? 1.0 : 2.0) * agf;
        }
        mem = sys->gamma * ((double)delta * ((((double)tBXYD / (double)p + (double)tBXYF) +
                                              ((double)(2 * WD) + (double)(2 * WF) / (double)p)) +
                                             (double)BI));
        if (nF > 0 && p > FminF) reason |= OR_R_SCALING;
        break;
    }
    case OR_SPATIAL_AG: {
        /* "we implement the spatial strategy for some first layers ... We then
         * implement an Allgather to collect the full set of activations before passing
         * it to the following layers which perform similar to the sequential
         * implementation."  Rows [0, Ls) as the Spatial row of Table 2;
         * rows [Ls, G) replicated on every PE (compute and activations not divided by
         * p); one Allgather of the boundary activation y_Ls (per-PE segment B|y_Ls|/p,
         * P:556 with Q19); GE over all weights as Spatial (Q35). */
        int32_t split[3] = {d[1], d[2], d[3]};
        if (d[0] != 1) FAIL(E_INVAL, "spatial_ag needs p1 == 1");
        if (c->Ls < 1) FAIL(E_INVAL, "spatial_ag needs Ls >= 1");
        p = (int64_t)d[1] * d[2] * d[3];
        B = b;
        int64_t Lp = c->Ls < m->G ? c->Ls : m->G;
        int64_t FBp = 0, FBs = 0, XYp = 0, XYs = 0;
        for (int64_t l = 0; l < m->G; l++) {
            const or_layer *r = &m->rows[l];
            if (l < Lp) { FBp += r->fw + r->bw; XYp += r->x + r->y; }
            else        { FBs += r->fw + r->bw; XYs += r->x + r->y; }
        }
        int64_t BFBp, BFBs, tBXYp, tBXYs, BdY;
        if (!mul_ok(B, FBp, &BFBp) || !mul_ok(B, FBs, &BFBs) || !mul_ok(2 * B, XYp, &tBXYp) ||
            !mul_ok(2 * B, XYs, &tBXYs) || !mul_ok(B * delta, m->rows[Lp - 1].y, &BdY))
            FAIL(E_OVERFLOW, "B*FB");
        /* comp: prefix rows / p, suffix rows in full, WU in full (replicated weights) */
        comp = ((((double)BFBp / (double)p) * tau) + (double)BFBs * tau) + (double)s.WU * tau;
        int64_t NS, HV, bdHV;
        reason |= spatial_terms(m, c->Ls, split, &NS, &HV);
        if (!mul_ok(b * delta, HV, &bdHV)) FAIL(E_OVERFLOW, "b*delta*HV");
        int t = tier_or_flag(sys, p, &reason);
        if (p > 1)
            halo = t < 0 ? INFINITY : 2.0 * ((double)(2 * NS) * p2p_alpha(sys, c, t) + (double)bdHV * p2p_beta(sys, c, t));
        ge = t < 0 ? INFINITY : t_allreduce(sys, p, (double)dW, (double)dW / (double)p, c->alpha[t], c->beta[t]);
        /* Allgather of y_Ls after the prefix: (p-1)(alpha + (B delta |y_Ls| / p) beta) */
        if (Lp < m->G && p > 1)
            ag = t < 0 ? INFINITY : (double)(p - 1) * (c->alpha[t] + ((double)BdY / (double)p) * c->beta[t]);
        /* memory: prefix activations / p, suffix activations in full, weights replicated */
        mem = sys->gamma * ((double)delta * ((((double)tBXYp / (double)p + (double)tBXYs) +
                                              (double)(2 * s.W)) + (double)s.BI));
        break;
    }
    case OR_GPIPE: {
        /* GPipe: the per-replica batch b is cut into S segments of b/S
         * samples that flow through the s stages, forward wave then backward wave.
         * Table 2's Layer row approximates its time "by the maximum"
         * (P:1008); this family times the schedule itself (Q36): a discrete-event
         * simulation of the S segments over the s stages.  Stage i forward task
         * lasts f_i = (b/S) FW_{G_i}; it then sends y_{G_i} to stage i+1 (blocking
         * P2P: alpha + (b/S) delta |y_{G_i}| beta), so stage i is busy
         * f_i + c_i; the backward task lasts g_i = (b/S) BW_{G_i} plus the send of the
         * input gradient to stage i-1 (same message size).  Backward starts when the
         * last stage finished its forward wave (GPipe flush); each stage applies WU_{G_i}
         * after its last backward task.  Iteration time = the last WU end. */
        int64_t ns = c->n_stages;
        int64_t S = c->S;
        if (d[0] != 1) FAIL(E_INVAL, "gpipe dims must be 1");
        if (S < 1) FAIL(E_INVAL, "gpipe needs S >= 1");
        p = ns;
        B = b;
        stage_t st;
        int rc = stage_terms(m, c, b, &st);
        if (rc) return rc;
        int ts = tier_or_flag(sys, ns, &reason);
        if (ts < 0) {
            comp = INFINITY;
        } else {
            double fq[OR_MAX_STAGES], gq[OR_MAX_STAGES], uq[OR_MAX_STAGES], cq[OR_MAX_STAGES];
            double mb = (double)b / (double)S;
            int64_t beg = 0;
            for (int i = 0; i < ns; i++) {
                int64_t F = 0, Bw = 0, U = 0;
                for (int64_t l = beg; l < c->stage_end[i]; l++) {
                    F += m->rows[l].fw;
                    Bw += m->rows[l].bw;
                    U += m->rows[l].wu;
                }
                fq[i] = (mb * (double)F) * tau;
                gq[i] = (mb * (double)Bw) * tau;
                uq[i] = (double)U * tau;
                cq[i] = 0.0;
                if (i < ns - 1)
                    cq[i] = p2p_alpha(sys, c, ts) + (mb * (double)(delta * m->rows[c->stage_end[i] - 1].y)) * p2p_beta(sys, c, ts);
                beg = c->stage_end[i];
            }
            /* forward wave: segment j enters stage i when stage i is free and stage i-1
             * has delivered it (stage 0 holds the input) */
            double freeq[OR_MAX_STAGES];
            for (int i = 0; i < ns; i++) freeq[i] = 0.0;
            for (int64_t j = 0; j < S; j++) {
                double ready = 0.0;
                for (int i = 0; i < ns; i++) {
                    double start = freeq[i] > ready ? freeq[i] : ready;
                    double dur = i < ns - 1 ? fq[i] + cq[i] : fq[i];
                    freeq[i] = start + dur;
                    ready = freeq[i];
                }
            }
            double t_f = freeq[ns - 1];
            /* backward wave, last stage first, after the flush */
            for (int i = 0; i < ns; i++) freeq[i] = t_f;
            for (int64_t j = 0; j < S; j++) {
                double ready = t_f;
                for (int i = (int)ns - 1; i >= 0; i--) {
                    double start = freeq[i] > ready ? freeq[i] : ready;
                    double dur = i > 0 ? gq[i] + cq[i - 1] : gq[i];
                    freeq[i] = start + dur;
                    ready = freeq[i];
                }
            }
            /* weight update per stage after its last backward task */
            double end = 0.0;
            for (int i = 0; i < ns; i++) {
                double e = freeq[i] + uq[i];
                if (e > end) end = e;
            }
            comp = end;
        }
        mem = sys->gamma * ((double)delta * (double)st.memI);   /* Table 2 Layer row memory */
        if (S > b) reason |= OR_R_SEGMENTS;   /* Q9 */
        break;
    }
    default:
        FAIL(E_INVAL, "bad family");
    }
    (void)tmp;
    o->t_comp = comp;
    o->t_ge = ge;
    o->t_fb_ag = ag;
    o->t_fb_ar = ar;
    o->t_halo = halo;
    o->t_p2p = p2p;
    o->t_iter = ((((comp + ge) + ag) + ar) + halo) + p2p;
    o->I = (double)m->D / (double)B;                  /* Table 1: I = D/B */
    o->t_epoch = o->t_iter * o->I;
    o->mem = mem;
    if (!(mem <= c->cap)) reason |= OR_R_MEMORY;       /* capacity, P:73, P:781-782 (Q31) */
    o->B = B;
    o->p = p;
    o->reason = reason;
    o->feasible = reason == 0;
    return 0;
}

/* ---------------------------------------------------------------- literal fold mode
 * Table 2 exactly as printed: every Sigma_l is an fp64 left fold over per-layer
 * real-valued terms (FW_l = fw_l * tau per sample, per-layer memory, per-layer comm).
 * Differs from or_eval only in rounding order; tests require <= 1e-12 relative. */
int or_eval_fold(const or_model *models, const or_system *sys, const or_config *c, or_pred *o)
{
    int rc = or_eval(models, sys, c, o);   /* structure, feasibility, B, p */
    if (rc) return rc;
    const or_model *m = &models[c->model];
    const double tau = 1.0 / c->flops;
    const double dl = (double)sys->delta;
    const int64_t b = c->b;
    const int32_t *d = c->dims;
    int64_t B = o->B, p = o->p;
    int64_t pc = 1, pu = 1, pa = 1, pw = 1;
    int fam = c->family;
    if (fam == OR_DATA || fam == OR_DATA_LW) { pc = p; pa = p; }
    if (fam == OR_SPATIAL || fam == OR_DS) { pc = p; pa = p; }
    if (fam == OR_FILTER || fam == OR_CHANNEL) { pc = p; pu = p; pw = p; }
    if (fam == OR_DF) { pc = p; pu = d[1]; pa = d[0]; pw = d[1]; }
    if (fam == OR_SPATIAL_AG) {
        /* per-row fold: rows before Ls divided by p (compute, activations), the rest in full */
        int64_t Lp = c->Ls < m->G ? c->Ls : m->G;
        double comp = 0.0, mem = 0.0;
        for (int64_t l = 0; l < m->G; l++) {
            const or_layer *r = &m->rows[l];
            double pp = l < Lp ? (double)p : 1.0;
            comp += ((double)B / pp) * ((double)r->fw * tau + (double)r->bw * tau);
            mem += dl * ((2.0 * (double)B) * (double)(r->x + r->y) / pp + 2.0 * (double)r->w + (double)r->bi);
        }
        for (int64_t l = 0; l < m->G; l++) comp += (double)m->rows[l].wu * tau;
        o->t_comp = comp;
        o->mem = sys->gamma * mem;
        if (o->t_halo != 0.0 && isfinite(o->t_halo)) {
            int32_t split[3] = {d[1], d[2], d[3]};
            int t = tier_of(sys, p);
            double sum = 0.0;
            for (int64_t l = 0; l < Lp; l++) {
                const or_layer *r = &m->rows[l];
                if (r->kind != OR_CONV && r->kind != OR_POOL) continue;
                double hv = (double)(or_halo_elements(r, split, 0) + or_halo_elements(r, split, 1));
                sum += 2.0 * p2p_alpha(sys, c, t) + (double)b * dl * p2p_beta(sys, c, t) * hv;
            }
            o->t_halo = 2.0 * sum;
        }
        if (o->t_fb_ag != 0.0 && isfinite(o->t_fb_ag)) {
            int t = tier_of(sys, p);
            o->t_fb_ag = (double)(p - 1) * (c->alpha[t] + (double)B * (double)m->rows[Lp - 1].y / (double)p * dl * c->beta[t]);
        }
    }
    if (fam == OR_SERIAL || fam == OR_DATA || fam == OR_DATA_LW || fam == OR_SPATIAL || fam == OR_DS ||
        fam == OR_FILTER || fam == OR_CHANNEL || fam == OR_DF || fam == OR_LAYERPURE) {
        int64_t Bc = fam == OR_LAYERPURE ? b : B;
        double comp = 0.0;
        for (int64_t l = 0; l < m->G; l++)
            comp += ((double)Bc / (double)pc) * ((double)m->rows[l].fw * tau + (double)m->rows[l].bw * tau);
        for (int64_t l = 0; l < m->G; l++) comp += ((double)m->rows[l].wu * tau) / (double)pu;
        o->t_comp = comp;
    }
    if (fam != OR_PIPELINE && fam != OR_LAYERPURE && fam != OR_PD && fam != OR_GPIPE && fam != OR_SPATIAL_AG) {
        double mem = 0.0;
        for (int64_t l = 0; l < m->G; l++) {
            const or_layer *r = &m->rows[l];
            mem += dl * ((2.0 * (double)B) * (double)(r->x + r->y) / (double)pa +
                         2.0 * (double)r->w / (double)pw + (double)r->bi);
        }
        o->mem = sys->gamma * mem;
    }
    if ((fam == OR_FILTER || fam == OR_CHANNEL || fam == OR_DF) && o->t_fb_ag != 0.0 && isfinite(o->t_fb_ag)) {
        int64_t pg = fam == OR_DF ? d[1] : p;
        int t = tier_of(sys, pg);
        int64_t last = -1;
        for (int64_t l = 0; l < m->G; l++) if (m->rows[l].flags & OR_FLAG_COMM) last = l;
        double sum = 0.0;
        for (int64_t l = 0; l < m->G; l++) {
            if (!(m->rows[l].flags & OR_FLAG_COMM) || l == last) continue;
            sum += c->alpha[t] + ((double)B * (double)m->rows[l].y / (double)p) * dl * c->beta[t];
        }
        o->t_fb_ag = (double)(pg - 1) * sum;
        o->t_fb_ar = (sys->filter_rs ? 1.0 : 2.0) * (double)(pg - 1) * sum;
    }
    if ((fam == OR_SPATIAL || fam == OR_DS) && o->t_halo != 0.0 && isfinite(o->t_halo)) {
        int32_t split[3] = {d[1], d[2], d[3]};
        int t = tier_of(sys, (int64_t)d[1] * d[2] * d[3]);
        double sum = 0.0;
        for (int64_t l = 0; l < m->G && l < c->Ls; l++) {
            const or_layer *r = &m->rows[l];
            if (r->kind != OR_CONV && r->kind != OR_POOL) continue;
            double hv = (double)(or_halo_elements(r, split, 0) + or_halo_elements(r, split, 1));
            sum += 2.0 * p2p_alpha(sys, c, t) + (double)b * dl * p2p_beta(sys, c, t) * hv;
        }
        o->t_halo = 2.0 * sum;
    }
    if (fam == OR_PIPELINE || fam == OR_PD || fam == OR_LAYERPURE) {
        /* per-group times FW_{G_i} = sum_{l in g_i} FW_l in fp64, then maxima */
        double mF = 0, mB = 0, mU = 0, memx = 0, sumP2P = 0;
        int ts = tier_of(sys, c->n_stages);
        int64_t beg = 0;
        for (int i = 0; i < c->n_stages; i++) {
            double F = 0, Bw = 0, U = 0, mm = 0;
            for (int64_t l = beg; l < c->stage_end[i]; l++) {
                const or_layer *r = &m->rows[l];
                F += (double)r->fw * tau;
                Bw += (double)r->bw * tau;
                U += (double)r->wu * tau;
                mm += dl * (2.0 * (double)b * (double)(r->x + r->y) + 2.0 * (double)r->w + (double)r->bi);
            }
            mF = F > mF ? F : mF;
            mB = Bw > mB ? Bw : mB;
            mU = U > mU ? U : mU;
            memx = mm > memx ? mm : memx;
            if (i < c->n_stages - 1 && ts >= 0)
                sumP2P += p2p_alpha(sys, c, ts) + dl * (double)b * (double)m->rows[c->stage_end[i] - 1].y * p2p_beta(sys, c, ts);
            beg = c->stage_end[i];
        }
        o->mem = sys->gamma * memx;
        if (fam == OR_LAYERPURE) {
            if (c->n_stages > 1 && ts >= 0) o->t_p2p = 2.0 * sumP2P;
        } else {
            o->t_comp = (double)(c->n_stages + c->S - 1) / (double)c->S * (double)b * (mF + mB) + mU;
        }
    }
    if (fam == OR_LAYERWISE) {
        /* per-row fold: each row with its own strategy's divisors; Allgather / transition
         * terms one message at a time */
        const uint64_t mask = c->i_part;
        int64_t last_comm = -1, first_comm = -1, ncomm = 0;
        for (int64_t l = 0; l < m->G; l++)
            if (m->rows[l].flags & OR_FLAG_COMM) { if (first_comm < 0) first_comm = l; last_comm = l; }
        int cur = first_comm >= 0 ? (int)(mask & 1) : 0;
        double comp = 0.0, mem = 0.0, agf = 0.0, tr = 0.0;
        int t = tier_of(sys, p);
        const double a = t >= 0 ? c->alpha[t] : 0.0, be = t >= 0 ? c->beta[t] : 0.0;
        for (int64_t l = 0; l < m->G; l++) {
            const or_layer *r = &m->rows[l];
            if (r->flags & OR_FLAG_COMM) {
                int sf = (int)((mask >> ncomm) & 1);
                if (ncomm > 0 && sf != cur) {
                    double one = a + (double)b * (double)m->rows[l - 1].y * dl * be;
                    tr += sf ? 2.0 * one : one;
                }
                cur = sf;
                ncomm++;
                if (cur && l != last_comm) agf += a + ((double)B * (double)r->y / (double)p) * dl * be;
            }
            comp += ((double)B / (double)p) * ((double)r->fw * tau + (double)r->bw * tau);
            comp += ((double)r->wu * tau) / (cur ? (double)p : 1.0);
            mem += dl * ((2.0 * (double)B) * (double)(r->x + r->y) / (cur ? 1.0 : (double)p) +
                         2.0 * (double)r->w / (cur ? (double)p : 1.0) + (double)r->bi);
        }
        o->t_comp = comp;
        o->mem = sys->gamma * mem;
        if (p > 1 && t >= 0 && o->t_fb_ag != 0.0) {
            o->t_fb_ag = (double)(p - 1) * agf + (double)(p - 1) * tr;
            o->t_fb_ar = (sys->filter_rs ? 1.0 : 2.0) * (double)(p - 1) * agf;
        }
    }
    o->t_iter = ((((o->t_comp + o->t_ge) + o->t_fb_ag) + o->t_fb_ar) + o->t_halo) + o->t_p2p;
    o->t_epoch = o->t_iter * o->I;
    return 0;
}

/* ---------------------------------------------------------------- batch drivers */
typedef struct {
    const or_model *models;
    int n_models;
    const or_system *sys;
    const or_spec *spec;
    /* dense / many */
    const uint64_t *idx_list;
    uint64_t first;
    int64_t lo, hi;
    double *t_iter, *mem, *key;
    uint32_t *reason32;
    uint8_t *reason8;
    /* topk */
    int32_t k;
    or_hit *hits;
    int32_t n_hits;
    uint64_t count;
    int rc;
    char err[256];
} job_t;

static int hit_less(double ka, uint64_t ia, double kb, uint64_t ib)
{
    return ka < kb || (ka == kb && ia < ib);
}

static void topk_insert(or_hit *h, int32_t *n, int32_t k, double key, uint64_t idx)
{
    if (*n == k && !hit_less(key, idx, h[k - 1].key, h[k - 1].idx)) return;
    int32_t pos = *n < k ? *n : k - 1;
    while (pos > 0 && hit_less(key, idx, h[pos - 1].key, h[pos - 1].idx)) {
        h[pos] = h[pos - 1];
        pos--;
    }
    h[pos].key = key;
    h[pos].idx = idx;
    if (*n < k) (*n)++;
}

static void *job_run(void *arg)
{
    job_t *j = (job_t *)arg;
    for (int64_t i = j->lo; i < j->hi; i++) {
        uint64_t idx = j->idx_list ? j->idx_list[i] : j->first + (uint64_t)i;
        or_config c;
        or_pred pr;
        int rc = or_decode(j->models, j->n_models, j->sys, j->spec, idx, &c);
        if (!rc) rc = or_eval(j->models, j->sys, &c, &pr);
        if (rc) {
            j->rc = rc;
            snprintf(j->err, sizeof j->err, "%s", g_err);
            return NULL;
        }
        if (j->hits) {
            if (pr.feasible) {
                j->count++;
                topk_insert(j->hits, &j->n_hits, j->k, pr.t_epoch, idx);
            }
            continue;
        }
        if (j->t_iter) j->t_iter[i] = pr.t_iter;
        if (j->mem) j->mem[i] = pr.mem;
        if (j->key) j->key[i] = pr.t_epoch;
        if (j->reason32) j->reason32[i] = pr.reason;
        if (j->reason8) j->reason8[i] = (uint8_t)pr.reason;
    }
    return NULL;
}

static int n_threads(int req)
{
    if (req > 0) return req;
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

static int run_jobs(job_t *proto, int64_t n, int nthreads, job_t **out_jobs, int *out_nt)
{
    int nt = n_threads(nthreads);
    if (nt > n && n > 0) nt = (int)n;
    if (nt < 1) nt = 1;
    job_t *jobs = calloc((size_t)nt, sizeof(job_t));
    pthread_t *th = calloc((size_t)nt, sizeof(pthread_t));
    for (int t = 0; t < nt; t++) {
        jobs[t] = *proto;
        jobs[t].lo = n * t / nt;
        jobs[t].hi = n * (t + 1) / nt;
        if (proto->hits) jobs[t].hits = calloc((size_t)proto->k, sizeof(or_hit));
        pthread_create(&th[t], NULL, job_run, &jobs[t]);
    }
    int rc = 0;
    for (int t = 0; t < nt; t++) {
        pthread_join(th[t], NULL);
        if (jobs[t].rc && !rc) {
            rc = jobs[t].rc;
            snprintf(g_err, sizeof g_err, "%s", jobs[t].err);
        }
    }
    free(th);
    *out_jobs = jobs;
    *out_nt = nt;
    return rc;
}

int or_eval_many(const or_model *models, int n_models, const or_system *sys,
                 const or_spec *spec, const uint64_t *idx, int64_t n,
                 double *t_iter, double *mem, uint32_t *reason, double *key, int nthreads)
{
    job_t p = {0};
    p.models = models; p.n_models = n_models; p.sys = sys; p.spec = spec;
    p.idx_list = idx; p.t_iter = t_iter; p.mem = mem; p.reason32 = reason; p.key = key;
    job_t *jobs; int nt;
    int rc = run_jobs(&p, n, nthreads, &jobs, &nt);
    free(jobs);
    return rc;
}

int or_sweep_dense(const or_model *models, int n_models, const or_system *sys,
                   const or_spec *spec, uint64_t first, uint64_t count,
                   double *t_iter, double *mem, uint32_t *bits, uint8_t *reason, int nthreads)
{
    uint64_t N;
    int rc = or_sweep_size(models, n_models, sys, spec, &N);
    if (rc) return rc;
    if (first > N || count > N - first) FAIL(E_RANGE, "range outside the sweep");
    uint32_t *r32 = malloc(sizeof(uint32_t) * (count ? count : 1));
    job_t p = {0};
    p.models = models; p.n_models = n_models; p.sys = sys; p.spec = spec;
    p.first = first; p.t_iter = t_iter; p.mem = mem; p.reason32 = r32;
    job_t *jobs; int nt;
    rc = run_jobs(&p, (int64_t)count, nthreads, &jobs, &nt);
    free(jobs);
    if (!rc) {
        if (bits) memset(bits, 0, sizeof(uint32_t) * ((count + 31) / 32));
        for (uint64_t i = 0; i < count; i++) {
            if (bits && r32[i] == 0) bits[i / 32] |= 1u << (i % 32);
            if (reason) reason[i] = (uint8_t)r32[i];
        }
    }
    free(r32);
    return rc;
}

int or_topk(const or_model *models, int n_models, const or_system *sys,
            const or_spec *spec, uint64_t first, uint64_t count, int32_t k,
            or_hit *hits, uint64_t *n_feasible, int nthreads)
{
    if (k < 1) FAIL(E_INVAL, "k < 1");
    uint64_t N;
    int rc = or_sweep_size(models, n_models, sys, spec, &N);
    if (rc) return rc;
    if (first > N || count > N - first) FAIL(E_RANGE, "range outside the sweep");
    job_t p = {0};
    p.models = models; p.n_models = n_models; p.sys = sys; p.spec = spec;
    p.first = first; p.k = k; p.hits = (or_hit *)1;
    job_t *jobs; int nt;
    rc = run_jobs(&p, (int64_t)count, nthreads, &jobs, &nt);
    int32_t n = 0;
    uint64_t cnt = 0;
    for (int i = 0; i < k; i++) { hits[i].idx = UINT64_MAX; hits[i].key = INFINITY; }
    for (int t = 0; t < nt; t++) {
        for (int i = 0; i < jobs[t].n_hits; i++) topk_insert(hits, &n, k, jobs[t].hits[i].key, jobs[t].hits[i].idx);
        cnt += jobs[t].count;
        free(jobs[t].hits);
    }
    free(jobs);
    *n_feasible = cnt;
    return rc;
}
