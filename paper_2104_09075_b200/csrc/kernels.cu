// kernels.cu -- sm_100a kernels of libparadl: model prep, the persistent sweep kernels
// (one template instance per strategy family x {reduce, dense}), the top-k merge, and
// the single-configuration explain/decode kernel.
//
// Hot path: a2 image staging (one TMA bulk copy per CTA) -> a3 decode
// (mixed radix + partition unranking once per tile, odometer in between) -> a4/a5/a6
// per-configuration cost (Table 2; Appendix) with
// structure-level terms hoisted out of the alpha/beta inner radices -> a7 feasibility ->
// a8 warp-ballot top-k / count, or a9 coalesced dense writes.
//
// Bit-exactness contract with the oracle: every real-valued term is the fp64 expression
// tree of DESIGN.md §2.3, evaluated with __dadd_rn/__dmul_rn/__ddiv_rn (never
// contracted into FMA; the library is also built with --fmad=false) and
// round-to-nearest int64 -> double conversions.  Integer sums are exact int64.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "paradl_internal.h"

namespace paradl {

// ------------------------------------------------------------------ fp64 helpers
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double i2d(int64_t x) { return __ll2double_rn(x); }

template <class T>
__device__ __forceinline__ const T *at(const uint8_t *base, uint32_t off) {
    return reinterpret_cast<const T *>(base + off);
}

// ------------------------------------------------------------------ a2: TMA bulk staging
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// One elected thread issues cp.async.bulk global->shared copies of the whole image,
// completing on an mbarrier; every thread waits on the barrier's phase 0.
__device__ void stage_image(uint8_t *dst, const uint8_t *src, uint32_t bytes, uint64_t *mbar) {
    const uint32_t bar = smem_u32(mbar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                     : "memory");
        const uint32_t chunk = 32768;
        for (uint32_t off = 0; off < bytes; off += chunk) {
            uint32_t n = bytes - off < chunk ? bytes - off : chunk;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(dst + off)),
                "l"(src + off), "r"(n), "r"(bar)
                : "memory");
        }
    }
    __syncthreads();
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(bar), "r"(0u)
            : "memory");
    }
}

// ------------------------------------------------------------------ image views
struct View {
    const uint8_t *img;
    const ImgHdr *H;
    const SubHdr *S;
    const ModelHdr *M;
    const uint8_t *mb;   // model block base
};

__device__ __forceinline__ View make_view(const uint8_t *img, int sub) {
    View v;
    v.img = img;
    v.H = at<ImgHdr>(img, 0);
    v.S = at<SubHdr>(img, v.H->sub_off[sub]);
    v.mb = img + v.H->model_off[v.S->model];
    v.M = reinterpret_cast<const ModelHdr *>(v.mb);
    return v;
}

__device__ __forceinline__ int tier_of(const ImgHdr *H, int64_t span) {
    for (int t = 0; t < H->n_tiers; t++)
        if (H->max_pes[t] >= span) return t;
    return -1;
}

__device__ __forceinline__ int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ int64_t ceil_log2_64(int64_t n) {
    int64_t l = 0;
    while ((int64_t(1) << l) < n) l++;
    return l;
}

// ------------------------------------------------------------------ a3: decode state
struct Lane {
    uint32_t d[kDigits];
    uint64_t part;    // partition rank (COMB) or mask (MASK)
    int32_t ns;       // stage count
};

// Lexicographic unranking of cut tuples inside the stage-count block.
__device__ void unrank_comb(const View &v, uint64_t r, Lane &L, uint16_t *cuts, int cs) {
    const SubHdr *S = v.S;
    const uint64_t *sblk = at<uint64_t>(v.img, S->off_sblk);
    const uint64_t *binom = at<uint64_t>(v.img, S->off_binom);
    const int stride = S->binom_stride;
    int j = 0;
    while (r >= sblk[j + 1]) j++;
    const int s = S->s_min + j;
    uint64_t rr = r - sblk[j];
    const int k = s - 1, n = S->G - 1;
    int val = 0;
    for (int q = 1; q <= k; q++) {
        val++;
        for (;;) {
            uint64_t c = binom[(n - val) * stride + (k - q)];
            if (rr < c) break;
            rr -= c;
            val++;
        }
        cuts[(q - 1) * cs] = (uint16_t)val;
    }
    L.ns = s;
}

// Lexicographic successor of the cut tuple; next stage count after the last tuple.
__device__ void succ_comb(const View &v, Lane &L, uint16_t *cuts, int cs) {
    const int n = v.S->G - 1;
    int k = L.ns - 1;
    int i = k - 1;
    while (i >= 0 && (int)cuts[i * cs] == n - (k - 1 - i)) i--;
    if (i >= 0) {
        int val = cuts[i * cs] + 1;
        for (int t = i; t < k; t++) cuts[t * cs] = (uint16_t)(val + (t - i));
    } else {
        L.ns++;
        if (L.ns > v.S->s_max) L.ns = v.S->s_min;
        k = L.ns - 1;
        for (int t = 0; t < k; t++) cuts[t * cs] = (uint16_t)(t + 1);
    }
}

__device__ void decode(const View &v, uint64_t u, Lane &L, uint16_t *cuts, int cs) {
    const SubHdr *S = v.S;
#pragma unroll
    for (int i = 0; i < kDigits; i++) {
        if (i == D_PART) {
            uint64_t np = S->part_n;
            L.part = u % np;
            u /= np;
        } else {
            uint32_t r = S->radix[i];
            L.d[i] = (uint32_t)(u % r);
            u /= r;
        }
    }
    L.ns = 1;
    if (S->part_mode == PARADL_PART_COMB) unrank_comb(v, L.part, L, cuts, cs);
    else if (S->part_mode == PARADL_PART_MASK) L.ns = __popcll(L.part) + 1;
}

// Adds the lane stride (mixed-radix digits inc[]) to the digit vector; returns the
// slowest digit that changed (-1: none).
__device__ __forceinline__ int advance(const LaunchArgs &a, const View &v, Lane &L, uint16_t *cuts,
                                       int cs) {
    const SubHdr *S = v.S;
    uint32_t c = 0;
    int lvl = -1;
#pragma unroll
    for (int i = 0; i < kDigits; i++) {
        if (i == D_PART) {
            uint64_t add = a.inc_part + c;
            if (add == 0) {
                if (i > a.inc_top) return lvl;
                continue;
            }
            lvl = i;
            uint64_t np = L.part + add;
            c = 0;
            bool wrap = np >= S->part_n;
            if (wrap) {
                np -= S->part_n;
                c = 1;
            }
            if (S->part_mode == PARADL_PART_COMB) {
                if (add == 1 && !wrap) succ_comb(v, L, cuts, cs);
                else unrank_comb(v, np, L, cuts, cs);
            } else if (S->part_mode == PARADL_PART_MASK) {
                L.ns = __popcll(np) + 1;
            }
            L.part = np;
        } else {
            uint32_t add = a.inc[i] + c;
            if (add == 0) {
                if (i > a.inc_top) return lvl;
                continue;
            }
            lvl = i;
            uint32_t nv = L.d[i] + add;
            c = nv >= S->radix[i];
            if (c) nv -= S->radix[i];
            L.d[i] = nv;
        }
    }
    return lvl;
}

// ------------------------------------------------------------------ a6: stage terms
struct StageT {
    int64_t maxF, maxB, maxU, maxW, maxY, sumY, memI;
};

// Per-stage sums FW_{G_i} = sum_{l in g_i} FW_l by prefix differences; maxima
// as in Table 2's Layer row.  b = per-replica batch (memory, Q6).
__device__ void stage_terms(const View &v, const Lane &L, const uint16_t *cuts, int cs, int64_t b,
                            StageT &st) {
    const ModelHdr *M = v.M;
    const int64_t *PF = at<int64_t>(v.mb, M->off_pf);
    const int64_t *PB = at<int64_t>(v.mb, M->off_pb);
    const int64_t *PU = at<int64_t>(v.mb, M->off_pu);
    const int64_t *PW = at<int64_t>(v.mb, M->off_pw);
    const int64_t *PX = at<int64_t>(v.mb, M->off_pxy);
    const int64_t *PI = at<int64_t>(v.mb, M->off_pbi);
    const int64_t *Y = at<int64_t>(v.mb, M->off_y);
    const int G = M->G;
    st.maxF = st.maxB = st.maxU = st.maxW = st.maxY = st.sumY = st.memI = 0;
    const int64_t twob = 2 * b;
    int beg = 0;
    uint64_t mask = L.part;
    const bool is_mask = v.S->part_mode == PARADL_PART_MASK;
    for (int i = 0; i < L.ns; i++) {
        int end;
        if (i == L.ns - 1) {
            end = G;
        } else if (is_mask) {
            end = __ffsll((long long)mask);   // bit j set <=> cut after row j+1
            mask &= mask - 1;
        } else {
            end = cuts[i * cs];
        }
        int64_t F = PF[end] - PF[beg], B = PB[end] - PB[beg], U = PU[end] - PU[beg];
        int64_t Wt = PW[end] - PW[beg], XY = PX[end] - PX[beg], BI = PI[end] - PI[beg];
        st.maxF = F > st.maxF ? F : st.maxF;
        st.maxB = B > st.maxB ? B : st.maxB;
        st.maxU = U > st.maxU ? U : st.maxU;
        st.maxW = Wt > st.maxW ? Wt : st.maxW;
        int64_t mem = twob * XY + 2 * Wt + BI;
        st.memI = mem > st.memI ? mem : st.memI;
        if (i < L.ns - 1) {
            int64_t y = Y[end - 1];
            st.maxY = y > st.maxY ? y : st.maxY;
            st.sumY += y;
        }
        beg = end;
    }
}

// ------------------------------------------------------------------ a4/a5: structure terms
// Allreduce term in hoisted form c * (alpha + s * beta_hat) (ring P:556 / tree P:559).
struct ARt {
    double c, s;
    int t;
    bool on;
};

__device__ __forceinline__ ARt make_ar(const ImgHdr *H, int64_t n, double m, double seg, int t) {
    ARt r;
    r.t = t;
    r.on = n != 1;
    if (H->tree_thr > 0.0 && m < H->tree_thr) {
        r.c = i2d(2 * (ceil_log2_64(n) + H->tree_chunks));
        r.s = ddiv(m, i2d(2 * (int64_t)H->tree_chunks));
    } else {
        r.c = i2d(2 * (n - 1));
        r.s = seg;
    }
    return r;
}

struct Mid {
    double comp, I, mem;
    uint32_t reason;
    int64_t B, p;
    ARt ge, ge2;          // GE (data/spatial/df/pd), ds: reduce-to-leader (ge) + leaders (ge2)
    double phi;           // df inter-group contention multiplier on beta
    double ag_c, ag_na, ag_s;
    int ag_t;
    bool ag_on;           // filter/channel/df Allgather phase (Allreduce = 2x)
    double h_na, h_s;
    int h_t;
    bool h_on;            // spatial/ds halo 2 (na alpha + s beta)
    double pp_c, pp_na, pp_s;
    int pp_t;
    bool pp_on;           // pipeline c (alpha + s beta) / layer-pure 2 (na alpha + s beta)
};

// comp row of Table 2: ((B FB)/p_c) tau + (WU/p_u) tau
__device__ __forceinline__ double comp_term(int64_t BFB, int64_t WU, int64_t pc, int64_t pu, double tau) {
    return dadd(dmul(ddiv(i2d(BFB), i2d(pc)), tau), dmul(ddiv(i2d(WU), i2d(pu)), tau));
}
// mem row of Table 2: gamma (delta ((2B XY)/p_a + (2W)/p_w + BI))
__device__ __forceinline__ double mem_term(const ImgHdr *H, int64_t twoBXY, int64_t W, int64_t BI,
                                           int64_t pa, int64_t pw) {
    return dmul(H->gamma, dmul(i2d(H->delta), dadd(dadd(ddiv(i2d(twoBXY), i2d(pa)), ddiv(i2d(2 * W), i2d(pw))),
                                                   i2d(BI))));
}

__device__ __forceinline__ uint32_t flag_tier(int t) { return t < 0 ? (uint32_t)PARADL_R_TIER : 0u; }

// Spatial set Sp = Conv/Pool rows among the first Ls rows; halo volume
// (Q15); per-axis limits (Q13) and SplitTooFine.
__device__ uint32_t spatial_terms(const View &v, int32_t Ls, const int32_t split[3], int64_t &NS,
                                  int64_t &HV) {
    const RowGeo *geo = at<RowGeo>(v.mb, v.M->off_geo);
    const int G = v.M->G;
    uint32_t reason = 0;
    NS = 0;
    HV = 0;
    const int lim = Ls < G ? Ls : G;
    for (int l = 0; l < lim; l++) {
        const RowGeo &r = geo[l];
        if (r.kind != PARADL_CONV && r.kind != PARADL_POOL) continue;
        NS++;
        for (int a = 0; a < 3; a++) {
            if (split[a] <= 1) continue;
            const int64_t h = r.K[a] / 2;
            if (split[a] > r.X[a]) reason |= PARADL_R_SCALING;
            if (ceil_div64(r.X[a], split[a]) < h || ceil_div64(r.Y[a], split[a]) < h) reason |= PARADL_R_SPLIT;
            if (h == 0) continue;
            const int64_t nnb = split[a] > 2 ? 2 : 1;
            int64_t cx = 1, cy = 1;
            for (int o = 0; o < 3; o++) {
                if (o == a) continue;
                cx *= ceil_div64(r.X[o], split[o]);
                cy *= ceil_div64(r.Y[o], split[o]);
            }
            HV += (int64_t)r.C * h * cx * nnb + (int64_t)r.F * h * cy * nnb;
        }
    }
    return reason;
}

template <int FAM>
__device__ void compute_mid(const View &v, const Lane &L, const StageT &st, Mid &m) {
    const ImgHdr *H = v.H;
    const SubHdr *S = v.S;
    const ModelHdr *M = v.M;
    const double cap = at<double>(v.img, S->off_cap)[L.d[D_CAP]];
    const double R = at<double>(v.img, S->off_flops)[L.d[D_FLOPS]];
    const double tau = ddiv(1.0, R);
    const int64_t b = at<int64_t>(v.img, S->off_b)[L.d[D_B]];
    const int32_t *dm = at<int32_t>(v.img, S->off_dims) + 4 * L.d[D_DIMS];
    const int64_t delta = H->delta;
    const int64_t dW = delta * M->W;
    uint32_t reason = 0;
    m.ge.on = m.ge2.on = m.ag_on = m.h_on = m.pp_on = false;
    m.phi = 1.0;
    int64_t B = b, p = 1;
    if (FAM == PARADL_SERIAL) {   // Table 2 Serial row
        m.comp = comp_term(B * M->FB, M->WU, 1, 1, tau);
        m.mem = mem_term(H, 2 * B * M->XY, M->W, M->BI, 1, 1);
    } else if (FAM == PARADL_DATA) {   // Data row
        p = dm[0];
        B = b * p;
        m.comp = comp_term(B * M->FB, M->WU, p, 1, tau);
        const int t = tier_of(H, p);
        reason |= flag_tier(t);
        m.ge = make_ar(H, p, i2d(dW), ddiv(i2d(dW), i2d(p)), t);
        m.mem = mem_term(H, 2 * B * M->XY, M->W, M->BI, p, 1);
        if (p > B) reason |= PARADL_R_SCALING;
    } else if (FAM == PARADL_SPATIAL || FAM == PARADL_DS) {   // Spatial row; ds (Q16)
        const int64_t p1 = dm[0];
        const int32_t split[3] = {dm[1], dm[2], dm[3]};
        const int64_t p2 = (int64_t)dm[1] * dm[2] * dm[3];
        p = p1 * p2;
        B = b * p1;
        m.comp = comp_term(B * M->FB, M->WU, p, 1, tau);
        const int32_t Ls = at<int32_t>(v.img, S->off_Ls)[L.d[D_LS]];
        int64_t NS, HV;
        reason |= spatial_terms(v, Ls, split, NS, HV);
        const int ti = tier_of(H, p2), to = tier_of(H, p);
        reason |= flag_tier(ti) | flag_tier(to);
        m.h_on = p2 > 1;
        m.h_na = i2d(2 * NS);
        m.h_s = i2d(b * delta * HV);
        m.h_t = ti;
        if (FAM == PARADL_SPATIAL) {
            m.ge = make_ar(H, p, i2d(dW), ddiv(i2d(dW), i2d(p)), to);
        } else {
            m.ge = make_ar(H, p2, i2d(dW), ddiv(i2d(dW), i2d(p2)), ti);   // reduce to leader
            m.ge2 = make_ar(H, p1, i2d(dW), ddiv(i2d(dW), i2d(p1)), to);  // Allreduce among leaders
        }
        m.mem = mem_term(H, 2 * B * M->XY, M->W, M->BI, p, 1);
    } else if (FAM == PARADL_FILTER || FAM == PARADL_CHANNEL) {   // Filter / Channel rows
        p = dm[0];
        B = b;
        m.comp = comp_term(B * M->FB, M->WU, p, p, tau);
        const int t = tier_of(H, p);
        reason |= flag_tier(t);
        m.ag_on = p > 1;
        m.ag_c = i2d(p - 1);
        m.ag_na = i2d(M->NC);
        m.ag_s = ddiv(i2d(B * delta * M->YC), i2d(p));
        m.ag_t = t;
        m.mem = mem_term(H, 2 * B * M->XY, M->W, M->BI, 1, p);
        if (FAM == PARADL_FILTER ? (p > M->Fmin) : (p > M->Cmin2)) reason |= PARADL_R_SCALING;
    } else if (FAM == PARADL_DF) {   // Data+Filter row, contention phi
        const int64_t p1 = dm[0], p2 = dm[1];
        p = p1 * p2;
        B = b * p1;
        m.comp = comp_term(B * M->FB, M->WU, p, p2, tau);
        const int ti = tier_of(H, p2), to = tier_of(H, p);
        reason |= flag_tier(ti) | flag_tier(to);
        m.ag_on = p2 > 1;
        m.ag_c = i2d(p2 - 1);
        m.ag_na = i2d(M->NC);
        m.ag_s = ddiv(i2d(B * delta * M->YC), i2d(p));
        m.ag_t = ti;
        m.phi = p2 > 1 ? H->phi_df : 1.0;
        m.ge = make_ar(H, p1, ddiv(i2d(dW), i2d(p2)), ddiv(i2d(dW), i2d(p)), to);
        m.mem = mem_term(H, 2 * B * M->XY, M->W, M->BI, p1, p2);
        if (p2 > M->Fmin) reason |= PARADL_R_SCALING;
    } else {   // PIPELINE, LAYERPURE, PD (Q17)
        const int64_t ns = L.ns;
        const int64_t Sg = at<int32_t>(v.img, S->off_S)[L.d[D_S]];
        const int64_t pd = FAM == PARADL_PD ? dm[0] : 1;
        p = ns * pd;
        B = b * pd;
        const int ts = tier_of(H, ns);
        reason |= flag_tier(ts);
        if (FAM == PARADL_LAYERPURE) {
            m.comp = comp_term(b * M->FB, M->WU, 1, 1, tau);
            m.pp_on = ns > 1;
            m.pp_na = i2d(ns - 1);
            m.pp_s = i2d(delta * b * st.sumY);
            m.pp_t = ts;
        } else {
            const double bS = ddiv(i2d(b), i2d(Sg));
            const double cseg = dmul(i2d(ns + Sg - 1), bS);
            m.comp = dadd(dmul(dmul(cseg, i2d(st.maxF + st.maxB)), tau), dmul(i2d(st.maxU), tau));
            m.pp_on = ns > 1;
            m.pp_c = i2d(2 * (ns + Sg - 2));
            m.pp_s = dmul(bS, i2d(delta * st.maxY));
            m.pp_t = ts;
            if (FAM == PARADL_PD) {
                const int tp = tier_of(H, p);
                reason |= flag_tier(tp);
                const double mW = i2d(delta * st.maxW);
                m.ge = make_ar(H, pd, mW, ddiv(mW, i2d(pd)), tp);
            }
        }
        m.mem = dmul(H->gamma, dmul(i2d(delta), i2d(st.memI)));
        if (Sg < 1 || Sg > b) reason |= PARADL_R_SEGMENTS;
    }
    m.I = ddiv(i2d(M->D), i2d(B));   // Table 1: I = D/B
    if (!(m.mem <= cap)) reason |= PARADL_R_MEMORY;
    m.reason = reason;
    m.B = B;
    m.p = p;
}

struct Phases {
    double comp, ge, ag, ar, halo, p2p;
};

// alpha/beta-dependent part and the t_iter fold ((((comp+GE)+AG)+AR)+Halo)+P2P.
// EXPLAIN: also report phases, with +inf for a phase whose tier is missing.
template <int FAM, bool EXPLAIN>
__device__ __forceinline__ double inner(const Mid &m, const double *arow, const double *brow, Phases *ph) {
    double ge = 0.0, ag = 0.0, ar = 0.0, halo = 0.0, p2p = 0.0;
    double t = m.comp;
    if (!EXPLAIN && (m.reason & PARADL_R_TIER)) return CUDART_INF;
    auto ar_eval = [&](const ARt &r, double phi, bool use_phi) -> double {
        if (!r.on) return 0.0;
        if (EXPLAIN && r.t < 0) return CUDART_INF;
        const double bh = use_phi ? dmul(brow[r.t], phi) : brow[r.t];
        return dmul(r.c, dadd(arow[r.t], dmul(r.s, bh)));
    };
    if (FAM == PARADL_DATA || FAM == PARADL_SPATIAL || FAM == PARADL_PD) {
        ge = ar_eval(m.ge, 1.0, false);
        if (m.ge.on) t = dadd(t, ge);
    }
    if (FAM == PARADL_DS) {
        ge = dadd(ar_eval(m.ge, 1.0, false), ar_eval(m.ge2, 1.0, false));
        t = dadd(t, ge);
    }
    if (FAM == PARADL_DF) {
        ge = ar_eval(m.ge, m.phi, true);
        if (m.ge.on) t = dadd(t, ge);
    }
    if (FAM == PARADL_FILTER || FAM == PARADL_CHANNEL || FAM == PARADL_DF) {
        if (m.ag_on) {
            if (EXPLAIN && m.ag_t < 0) ag = CUDART_INF;
            else ag = dmul(m.ag_c, dadd(dmul(m.ag_na, arow[m.ag_t]), dmul(m.ag_s, brow[m.ag_t])));
            ar = dmul(2.0, ag);
            t = dadd(dadd(t, ag), ar);
        }
    }
    if (FAM == PARADL_SPATIAL || FAM == PARADL_DS) {
        if (m.h_on) {
            if (EXPLAIN && m.h_t < 0) halo = CUDART_INF;
            else halo = dmul(2.0, dadd(dmul(m.h_na, arow[m.h_t]), dmul(m.h_s, brow[m.h_t])));
            t = dadd(t, halo);
        }
    }
    if (FAM == PARADL_PIPELINE || FAM == PARADL_PD) {
        if (m.pp_on) {
            if (EXPLAIN && m.pp_t < 0) p2p = CUDART_INF;
            else p2p = dmul(m.pp_c, dadd(arow[m.pp_t], dmul(m.pp_s, brow[m.pp_t])));
            t = dadd(t, p2p);
        }
    }
    if (FAM == PARADL_LAYERPURE) {
        if (m.pp_on) {
            if (EXPLAIN && m.pp_t < 0) p2p = CUDART_INF;
            else p2p = dmul(2.0, dadd(dmul(m.pp_na, arow[m.pp_t]), dmul(m.pp_s, brow[m.pp_t])));
            t = dadd(t, p2p);
        }
    }
    if (EXPLAIN) {
        ph->comp = m.comp;
        ph->ge = ge;
        ph->ag = ag;
        ph->ar = ar;
        ph->halo = halo;
        ph->p2p = p2p;
    }
    return t;
}

// ------------------------------------------------------------------ a8: warp top-k
__device__ __forceinline__ bool hit_less(double ka, uint64_t ia, double kb, uint64_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// Sorted list of up to 64 (key, idx) entries held in registers across the warp:
// lane l owns entries l (a) and l + 32 (b).  th = entry k-1 (the admission threshold).
struct WarpTopK {
    double ka, kb, thk;
    uint64_t ia, ib, thi;
    int k;

    __device__ void init(int kk) {
        k = kk;
        ka = kb = thk = CUDART_INF;
        ia = ib = thi = ~0ull;
    }
    // whole warp, uniform (key, idx)
    __device__ void insert(double key, uint64_t idx) {
        const int lane = threadIdx.x & 31;
        const unsigned full = 0xffffffffu;
        int pos = __popc(__ballot_sync(full, hit_less(ka, ia, key, idx))) +
                  __popc(__ballot_sync(full, hit_less(kb, ib, key, idx)));
        if (pos >= k) return;
        double pak = __shfl_up_sync(full, ka, 1), pbk = __shfl_up_sync(full, kb, 1);
        uint64_t pai = __shfl_up_sync(full, ia, 1), pbi = __shfl_up_sync(full, ib, 1);
        double a31k = __shfl_sync(full, ka, 31);
        uint64_t a31i = __shfl_sync(full, ia, 31);
        if (lane == 0) {
            pbk = a31k;
            pbi = a31i;
        }
        if (lane > pos) {
            ka = pak;
            ia = pai;
        } else if (lane == pos) {
            ka = key;
            ia = idx;
        }
        const int j = lane + 32;
        if (j > pos) {
            kb = pbk;
            ib = pbi;
        } else if (j == pos) {
            kb = key;
            ib = idx;
        }
        const int src = (k - 1) & 31;
        double tka = __shfl_sync(full, ka, src), tkb = __shfl_sync(full, kb, src);
        uint64_t tia = __shfl_sync(full, ia, src), tib = __shfl_sync(full, ib, src);
        if (k - 1 < 32) {
            thk = tka;
            thi = tia;
        } else {
            thk = tkb;
            thi = tib;
        }
    }
    // whole warp; per-lane candidate (valid, key, idx)
    __device__ __forceinline__ void offer(bool valid, double key, uint64_t idx) {
        const unsigned full = 0xffffffffu;
        bool cand = valid && key <= thk && (key < thk || idx < thi);
        unsigned msk = __ballot_sync(full, cand);
        while (msk) {
            const int src = __ffs(msk) - 1;
            msk &= msk - 1;
            double kk = __shfl_sync(full, key, src);
            uint64_t ii = __shfl_sync(full, idx, src);
            if (hit_less(kk, ii, thk, thi)) insert(kk, ii);
        }
    }
};

// ------------------------------------------------------------------ the sweep kernel
struct SmemExtra {
    uint16_t cuts[kMaxCuts][kThreads];
    paradl_hit lists[kWarps][PARADL_MAX_TOPK];
};

template <int FAM, bool DENSE>
__global__ void __launch_bounds__(kThreads) sweep_kernel(const LaunchArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t mbar;
    __shared__ unsigned long long s_count;
    if (threadIdx.x == 0) s_count = 0;
    stage_image(smem, a.img, a.img_bytes, &mbar);
    SmemExtra *ex = reinterpret_cast<SmemExtra *>(smem + a.img_bytes);
    const View v = make_view(smem, a.sub);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint16_t *cuts = &ex->cuts[0][threadIdx.x];
    const int cs = kThreads;
    const int NT = v.H->n_tiers;
    const double *alpha_tab = at<double>(v.img, v.S->off_alpha);
    const double *beta_tab = at<double>(v.img, v.S->off_beta);
    const uint64_t gbase = v.S->offset;   // global index of local index 0
    const uint64_t TS = 32ull * a.steps;
    constexpr bool PIPE = FAM == PARADL_PIPELINE || FAM == PARADL_LAYERPURE || FAM == PARADL_PD;

    WarpTopK tk;
    tk.init(a.k);
    unsigned long long cnt = 0;

    for (;;) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(a.tile_counter, 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        const uint64_t tile = t * (uint64_t)a.n_shards + (uint64_t)a.shard;
        if (tile >= a.n_tiles) break;
        const uint64_t u0 = a.lo + tile * TS;
        const uint64_t uend = (u0 + TS < a.hi) ? u0 + TS : a.hi;

        Lane L;
        StageT st;
        Mid m;
        uint64_t u = u0 + lane;
        bool active = u < uend;
        if (active) {
            decode(v, u, L, cuts, cs);
            if (PIPE) stage_terms(v, L, cuts, cs, at<int64_t>(v.img, v.S->off_b)[L.d[D_B]], st);
            compute_mid<FAM>(v, L, st, m);
        }
        uint32_t carry = 0;
        uint64_t wlast = 0;
        bool have_carry = false;
        for (uint64_t s0 = u0; s0 < uend; s0 += 32) {
            active = u < uend;
            double key = CUDART_INF, t_it = CUDART_INF;
            bool feas = false;
            if (active) {
                const double *arow = alpha_tab + (size_t)L.d[D_ALPHA] * NT;
                const double *brow = beta_tab + (size_t)L.d[D_BETA] * NT;
                if (DENSE || m.reason == 0) {
                    t_it = inner<FAM, false>(m, arow, brow, nullptr);
                    key = dmul(t_it, m.I);
                }
                feas = m.reason == 0;
            }
            const uint64_t gidx = gbase + u;
            if (!DENSE) {
                cnt += (active && feas) ? 1u : 0u;
                tk.offer(active && feas, key, gidx);
            } else {
                const uint64_t o = gidx - a.first;
                if (active) {
                    if (a.t_iter) a.t_iter[o] = t_it;
                    if (a.mem) a.mem[o] = m.mem;
                    if (a.reason) a.reason[o] = (uint8_t)m.reason;
                }
                if (a.bits) {
                    const unsigned bits = __ballot_sync(0xffffffffu, active && feas);
                    if (lane == 0) {
                        const uint64_t pos0 = gbase + s0 - a.first;   // bit position of this step's lane 0
                        const uint32_t sh = (uint32_t)(pos0 & 31);
                        const uint64_t w = pos0 >> 5;
                        const uint32_t lo = bits << sh;
                        const uint32_t hi = sh ? (bits >> (32 - sh)) : 0u;
                        const uint32_t word = lo | (have_carry ? carry : 0u);
                        // exclusive iff every bit of word w maps into this tile's range
                        const uint64_t wg0 = a.first + (w << 5);
                        const bool excl = have_carry || sh == 0;
                        const bool inside = wg0 >= gbase + u0 && wg0 + 32 <= gbase + uend;
                        if (excl && inside) a.bits[w] = word;
                        else if (word) atomicOr(&a.bits[w], word);
                        carry = hi;
                        have_carry = sh != 0;
                        wlast = w + 1;
                    }
                }
            }
            // advance every lane by 32 indices
            u += 32;
            if (u < uend) {
                const int lvl = advance(a, v, L, cuts, cs);
                if (lvl >= D_LS) {
                    if (PIPE && lvl >= D_PART)
                        stage_terms(v, L, cuts, cs, at<int64_t>(v.img, v.S->off_b)[L.d[D_B]], st);
                    compute_mid<FAM>(v, L, st, m);
                }
            }
        }
        if (DENSE && a.bits && lane == 0 && have_carry && carry) atomicOr(&a.bits[wlast], carry);
    }

    if (!DENSE) {
        // CTA merge: warps publish their lists; warp 0 inserts the others into its own.
        paradl_hit *mine = ex->lists[warp];
        mine[lane].idx = tk.ia;
        mine[lane].key_epoch_s = tk.ka;
        mine[lane + 32].idx = tk.ib;
        mine[lane + 32].key_epoch_s = tk.kb;
        atomicAdd(&s_count, cnt);
        __syncthreads();
        if (warp == 0) {
            for (int w = 1; w < kWarps; w++) {
                for (int e = 0; e < a.k; e += 32) {
                    const int j = e + lane;
                    const bool ok = j < a.k;
                    const double kk = ok ? ex->lists[w][j].key_epoch_s : CUDART_INF;
                    const uint64_t ii = ok ? ex->lists[w][j].idx : ~0ull;
                    tk.offer(ok && ii != ~0ull, kk, ii);
                }
            }
            paradl_hit *out = a.cta_lists + (size_t)blockIdx.x * a.k;
            if (lane < a.k) {
                out[lane].idx = tk.ia;
                out[lane].key_epoch_s = tk.ka;
            }
            if (lane + 32 < a.k) {
                out[lane + 32].idx = tk.ib;
                out[lane + 32].key_epoch_s = tk.kb;
            }
            if (lane == 0) atomicAdd(a.count, s_count);
        }
    }
}

// ------------------------------------------------------------------ merge kernel
// Merges n_lists sorted-or-not lists of k hits and sums n_counts counts.
__global__ void __launch_bounds__(1024) merge_kernel(const paradl_hit *lists, int64_t n_lists, int32_t k,
                                                      const unsigned long long *counts, int32_t n_counts,
                                                      paradl_hit *out, unsigned long long *count_out) {
    __shared__ paradl_hit s_lists[32][PARADL_MAX_TOPK];
    __shared__ unsigned long long s_cnt;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    unsigned long long c = 0;
    for (int i = threadIdx.x; i < n_counts; i += blockDim.x) c += counts[i];
    atomicAdd(&s_cnt, c);
    WarpTopK tk;
    tk.init(k);
    const int64_t n = n_lists * (int64_t)k;
    const int nw = blockDim.x >> 5;
    for (int64_t base = (int64_t)warp * 32; base < n; base += (int64_t)nw * 32) {
        const int64_t j = base + lane;
        const bool ok = j < n;
        const double kk = ok ? lists[j].key_epoch_s : CUDART_INF;
        const uint64_t ii = ok ? lists[j].idx : ~0ull;
        tk.offer(ok && ii != ~0ull, kk, ii);
    }
    s_lists[warp][lane].idx = tk.ia;
    s_lists[warp][lane].key_epoch_s = tk.ka;
    s_lists[warp][lane + 32].idx = tk.ib;
    s_lists[warp][lane + 32].key_epoch_s = tk.kb;
    __syncthreads();
    if (warp == 0) {
        for (int w = 1; w < nw; w++)
            for (int e = 0; e < k; e += 32) {
                const int j = e + lane;
                const bool ok = j < k;
                const double kk = ok ? s_lists[w][j].key_epoch_s : CUDART_INF;
                const uint64_t ii = ok ? s_lists[w][j].idx : ~0ull;
                tk.offer(ok && ii != ~0ull, kk, ii);
            }
        if (lane < k) {
            out[lane].idx = tk.ia;
            out[lane].key_epoch_s = tk.ka;
        }
        if (lane + 32 < k) {
            out[lane + 32].idx = tk.ib;
            out[lane + 32].key_epoch_s = tk.kb;
        }
        if (lane == 0) *count_out = s_cnt;
    }
}

// ------------------------------------------------------------------ explain / decode
template <int FAM>
__device__ void explain_one(const View &v, const Lane &L, const uint16_t *cuts, paradl_config *cfg,
                            paradl_prediction *pr) {
    StageT st = {};
    const int64_t b = at<int64_t>(v.img, v.S->off_b)[L.d[D_B]];
    constexpr bool PIPE = FAM == PARADL_PIPELINE || FAM == PARADL_LAYERPURE || FAM == PARADL_PD;
    if (PIPE) stage_terms(v, L, cuts, 1, b, st);
    Mid m;
    compute_mid<FAM>(v, L, st, m);
    const int NT = v.H->n_tiers;
    const double *arow = at<double>(v.img, v.S->off_alpha) + (size_t)L.d[D_ALPHA] * NT;
    const double *brow = at<double>(v.img, v.S->off_beta) + (size_t)L.d[D_BETA] * NT;
    Phases ph;
    const double t = inner<FAM, true>(m, arow, brow, &ph);
    pr->t_comp = ph.comp;
    pr->t_ge = ph.ge;
    pr->t_fb_ag = ph.ag;
    pr->t_fb_ar = ph.ar;
    pr->t_halo = ph.halo;
    pr->t_p2p = ph.p2p;
    pr->t_iter = t;
    pr->I = m.I;
    pr->t_epoch = dmul(t, m.I);
    pr->mem = m.mem;
    pr->reason = m.reason;
    pr->feasible = m.reason == 0;
    cfg->B = m.B;
    cfg->p = m.p;
}

__global__ void explain_kernel(const uint8_t *img, int32_t sub, uint64_t local, paradl_config *cfg,
                               paradl_prediction *pr) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const View v = make_view(img, sub);
    uint16_t cuts[kMaxCuts + 1];
    Lane L;
    decode(v, local, L, cuts, 1);
    const SubHdr *S = v.S;
    cfg->sub = sub;
    cfg->family = S->family;
    cfg->model_id = S->model;
    cfg->n_stages = L.ns;
    cfg->i_cap = L.d[D_CAP];
    cfg->i_flops = L.d[D_FLOPS];
    cfg->i_b = L.d[D_B];
    cfg->i_S = L.d[D_S];
    cfg->i_dims = L.d[D_DIMS];
    cfg->i_Ls = L.d[D_LS];
    cfg->i_alpha = L.d[D_ALPHA];
    cfg->i_beta = L.d[D_BETA];
    cfg->i_part = L.part;
    cfg->cap = at<double>(img, S->off_cap)[L.d[D_CAP]];
    cfg->flops = at<double>(img, S->off_flops)[L.d[D_FLOPS]];
    cfg->b = at<int64_t>(img, S->off_b)[L.d[D_B]];
    cfg->S = at<int32_t>(img, S->off_S)[L.d[D_S]];
    cfg->Ls = at<int32_t>(img, S->off_Ls)[L.d[D_LS]];
    for (int a = 0; a < 4; a++) cfg->dims[a] = at<int32_t>(img, S->off_dims)[4 * L.d[D_DIMS] + a];
    const int NT = v.H->n_tiers;
    for (int t = 0; t < PARADL_MAX_TIERS; t++) {
        cfg->alpha[t] = t < NT ? at<double>(img, S->off_alpha)[(size_t)L.d[D_ALPHA] * NT + t] : 0.0;
        cfg->beta[t] = t < NT ? at<double>(img, S->off_beta)[(size_t)L.d[D_BETA] * NT + t] : 0.0;
    }
    {
        const int G = v.M->G;
        uint64_t mask = L.part;
        for (int i = 0; i < PARADL_MAX_STAGES; i++) cfg->stage_end[i] = 0;
        for (int i = 0; i < L.ns && i < PARADL_MAX_STAGES; i++) {
            int end;
            if (i == L.ns - 1) end = G;
            else if (S->part_mode == PARADL_PART_MASK) {
                end = __ffsll((long long)mask);
                mask &= mask - 1;
            } else end = cuts[i];
            cfg->stage_end[i] = end;
        }
    }
    switch (S->family) {
    case PARADL_SERIAL: explain_one<PARADL_SERIAL>(v, L, cuts, cfg, pr); break;
    case PARADL_DATA: explain_one<PARADL_DATA>(v, L, cuts, cfg, pr); break;
    case PARADL_SPATIAL: explain_one<PARADL_SPATIAL>(v, L, cuts, cfg, pr); break;
    case PARADL_FILTER: explain_one<PARADL_FILTER>(v, L, cuts, cfg, pr); break;
    case PARADL_CHANNEL: explain_one<PARADL_CHANNEL>(v, L, cuts, cfg, pr); break;
    case PARADL_DF: explain_one<PARADL_DF>(v, L, cuts, cfg, pr); break;
    case PARADL_DS: explain_one<PARADL_DS>(v, L, cuts, cfg, pr); break;
    case PARADL_PIPELINE: explain_one<PARADL_PIPELINE>(v, L, cuts, cfg, pr); break;
    case PARADL_LAYERPURE: explain_one<PARADL_LAYERPURE>(v, L, cuts, cfg, pr); break;
    case PARADL_PD: explain_one<PARADL_PD>(v, L, cuts, cfg, pr); break;
    default: break;
    }
}

// ------------------------------------------------------------------ model prep
// Derives the model block (row geometry, prefix arrays, Table 2 sums) from the rows.
__global__ void prep_model_kernel(const paradl_layer *rows, int32_t G, int64_t D, uint8_t *blk, ModelHdr lay) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    ModelHdr *M = reinterpret_cast<ModelHdr *>(blk);
    RowGeo *geo = reinterpret_cast<RowGeo *>(blk + lay.off_geo);
    int64_t *PF = reinterpret_cast<int64_t *>(blk + lay.off_pf);
    int64_t *PB = reinterpret_cast<int64_t *>(blk + lay.off_pb);
    int64_t *PU = reinterpret_cast<int64_t *>(blk + lay.off_pu);
    int64_t *PW = reinterpret_cast<int64_t *>(blk + lay.off_pw);
    int64_t *PX = reinterpret_cast<int64_t *>(blk + lay.off_pxy);
    int64_t *PI = reinterpret_cast<int64_t *>(blk + lay.off_pbi);
    int64_t *Y = reinterpret_cast<int64_t *>(blk + lay.off_y);
    *M = lay;
    M->G = G;
    M->D = D;
    PF[0] = PB[0] = PU[0] = PW[0] = PX[0] = PI[0] = 0;
    int first_comm = -1, last_comm = -1;
    int64_t Fmin = INT64_MAX;
    for (int l = 0; l < G; l++) {
        const paradl_layer &r = rows[l];
        RowGeo &g = geo[l];
        g.kind = r.kind;
        g.flags = (int32_t)r.flags;
        g.C = (int32_t)r.C;
        g.F = (int32_t)r.F;
        for (int a = 0; a < 3; a++) {
            g.X[a] = (int32_t)r.X[a];
            g.Y[a] = (int32_t)r.Y[a];
            g.K[a] = (int32_t)r.K[a];
        }
        g.pad = 0;
        PF[l + 1] = PF[l] + r.fw;
        PB[l + 1] = PB[l] + r.bw;
        PU[l + 1] = PU[l] + r.wu;
        PW[l + 1] = PW[l] + r.w;
        PX[l + 1] = PX[l] + r.x + r.y;
        PI[l + 1] = PI[l] + r.bi;
        Y[l] = r.y;
        if (r.flags & PARADL_FLAG_COMM) {
            if (first_comm < 0) first_comm = l;
            last_comm = l;
            if (r.F < Fmin) Fmin = r.F;
        }
    }
    int64_t YC = 0, NC = 0, Cmin2 = INT64_MAX;
    for (int l = 0; l < G; l++) {
        const paradl_layer &r = rows[l];
        if (!(r.flags & PARADL_FLAG_COMM)) continue;
        if (l != last_comm) {
            YC += r.y;
            NC += 1;
        }
        if (l != first_comm && r.C < Cmin2) Cmin2 = r.C;
    }
    M->FB = PF[G] + PB[G];
    M->WU = PU[G];
    M->W = PW[G];
    M->BI = PI[G];
    M->XY = PX[G];
    M->YC = YC;
    M->NC = NC;
    M->Fmin = Fmin;
    M->Cmin2 = Cmin2;
}

// ------------------------------------------------------------------ FP64 peak microbenchmark
// 8 independent DFMA chains per thread; counts executed DFMA instructions.
__global__ void __launch_bounds__(256) fp64_bench_kernel(int iters, double *sink) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
           a7 = a0 + 7;
    const double m = 0.999999, c = 1e-12;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int j = 0; j < 16; j++) {
            asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a0) : "d"(m), "d"(c));
            asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a1) : "d"(m), "d"(c));
            asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a2) : "d"(m), "d"(c));
            asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a3) : "d"(m), "d"(c));
            asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a4) : "d"(m), "d"(c));
            asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a5) : "d"(m), "d"(c));
            asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a6) : "d"(m), "d"(c));
            asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a7) : "d"(m), "d"(c));
        }
    }
    const double r = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (r == 12345.678) sink[threadIdx.x] = r;
}

cudaError_t launch_fp64_bench(int n_sm, int iters, double *d_sink, cudaStream_t st, int *threads_out) {
    const int grid = n_sm * 8;
    fp64_bench_kernel<<<grid, 256, 0, st>>>(iters, d_sink);
    *threads_out = grid * 256;
    return cudaGetLastError();
}

// ------------------------------------------------------------------ launchers
template <int FAM, bool DENSE>
static void *kernel_ptr() {
    return (void *)sweep_kernel<FAM, DENSE>;
}

static void *sweep_fn(int family, bool dense) {
#define PARADL_CASE(F)                                                              \
    case F:                                                                         \
        return dense ? kernel_ptr<F, true>() : kernel_ptr<F, false>();
    switch (family) {
        PARADL_CASE(PARADL_SERIAL)
        PARADL_CASE(PARADL_DATA)
        PARADL_CASE(PARADL_SPATIAL)
        PARADL_CASE(PARADL_FILTER)
        PARADL_CASE(PARADL_CHANNEL)
        PARADL_CASE(PARADL_DF)
        PARADL_CASE(PARADL_DS)
        PARADL_CASE(PARADL_PIPELINE)
        PARADL_CASE(PARADL_LAYERPURE)
        PARADL_CASE(PARADL_PD)
    default: return nullptr;
    }
#undef PARADL_CASE
}

size_t sweep_smem_extra() { return sizeof(SmemExtra); }

int max_blocks_per_sm(int family, bool dense, size_t smem) {
    void *fn = sweep_fn(family, dense);
    if (!fn) return 0;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kThreads, smem) != cudaSuccess) return 0;
    return nb;
}

cudaError_t launch_sweep(int family, bool dense, const LaunchArgs &a, int grid, size_t smem, cudaStream_t st) {
    void *fn = sweep_fn(family, dense);
    if (!fn) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    void *args[] = {const_cast<LaunchArgs *>(&a)};
    return cudaLaunchKernel(fn, dim3(grid), dim3(kThreads), args, smem, st);
}

cudaError_t launch_merge(const paradl_hit *lists, int64_t n_lists, int32_t k, const unsigned long long *counts,
                         int32_t n_counts, paradl_hit *out, unsigned long long *count_out, cudaStream_t st) {
    merge_kernel<<<1, 1024, 0, st>>>(lists, n_lists, k, counts, n_counts, out, count_out);
    return cudaGetLastError();
}

cudaError_t launch_explain(const uint8_t *img, uint32_t, int32_t sub, uint64_t local, paradl_config *d_cfg,
                           paradl_prediction *d_pred, cudaStream_t st) {
    explain_kernel<<<1, 32, 0, st>>>(img, sub, local, d_cfg, d_pred);
    return cudaGetLastError();
}

cudaError_t launch_prep_model(const paradl_layer *d_rows, int32_t G, int64_t D, uint8_t *d_block,
                              const ModelHdr &layout, cudaStream_t st) {
    prep_model_kernel<<<1, 32, 0, st>>>(d_rows, G, D, d_block, layout);
    return cudaGetLastError();
}

}  // namespace paradl
