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
#include <cstdio>

#include <mutex>

#include "paradl_internal.h"

namespace paradl {

// tuning knobs (experiments build variants with -D; defaults are the measured best)
#ifndef PARADL_RELAXED_BOUND
#define PARADL_RELAXED_BOUND 1
#endif
#ifndef PARADL_MINB
#define PARADL_MINB 2
#endif
#ifndef PARADL_PIPE_MINB
#define PARADL_PIPE_MINB PARADL_MINB
#endif
#ifndef PARADL_COMB_MINB
#define PARADL_COMB_MINB PARADL_MINB   // mode-3 resident CTAs per SM the register budget targets
#endif
#ifndef PARADL_COMB_UNROLL
#define PARADL_COMB_UNROLL 2
#endif
constexpr int kCombUnroll = PARADL_COMB_UNROLL;   // mode-3 p_d loop unroll (A/B knob)
#ifndef PARADL_PIPE_KEYS
#define PARADL_PIPE_KEYS 16
#endif

// Device-side bounds checks of the checked build (-DPARADL_CHECKS=1, tools/checked_build.py):
// a failed check traps, so the call returns PARADL_ECUDA and the test that made it fails.
// (compute-sanitizer is not available on the GPU pool.)
#ifndef PARADL_CHECKS
#define PARADL_CHECKS 0
#endif
#if PARADL_CHECKS
#define PCHECK(c)                                                                                   \
    do {                                                                                            \
        if (!(c)) {                                                                                 \
            printf("PARADL_CHECKS: %s failed at %s:%d (block %d thread %d)\n", #c, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                              \
            __trap();                                                                               \
        }                                                                                           \
    } while (0)
#else
#define PCHECK(c) \
    do {          \
    } while (0)
#endif

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
    for (int t = 0; t < H->n_ctiers; t++)
        if (H->max_pes[t] >= span) return t;
    return -1;
}

// alpha/beta column of the point-to-point copy of tier t (Q40); t < 0 stays < 0
__device__ __forceinline__ int p2p_tier(const ImgHdr *H, int t) { return t < 0 ? t : t + H->p2p_off; }

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
    int lo = 1;   // smallest value the next cut can take
    for (int q = 1; q <= k; q++) {
        // tuples whose cut q is >= m (the later cuts free): A(m) = sum_{v >= m} C(n - v, j)
        // = C(n - m + 1, j + 1) (hockey stick), j = k - q cuts after it.  Cut q is the largest
        // m with A(lo) - A(m) <= rr -- the count of tuples skipped by a linear scan that
        // subtracts C(n - v, j) for v = lo, lo + 1, ... -- found by bisection.
        const int j = k - q;
        int val;
        if (j == 0) {
            val = lo + (int)rr;   // C(n - v, 0) = 1 per value
            rr = 0;
        } else {
            const uint64_t Alo = binom[(n - lo + 1) * stride + j + 1];
            int a = lo, b = n - j + 1;   // P(a) holds, P(b) does not (b is past the last value)
            while (b - a > 1) {
                const int m = (a + b) >> 1;
                if (Alo - binom[(n - m + 1) * stride + j + 1] <= rr) a = m;
                else b = m;
            }
            val = a;
            rr -= Alo - binom[(n - a + 1) * stride + j + 1];
        }
        PCHECK(val >= 1 && val <= n && (q == 1 || val > cuts[(q - 2) * cs]));
        cuts[(q - 1) * cs] = (uint16_t)val;
        lo = val + 1;
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
    if ((u >> 32) == 0 && (S->part_n >> 32) == 0) {
        // 32-bit mixed-radix decode (most sub-sweeps): ~5x cheaper than 64-bit division
        uint32_t w = (uint32_t)u;
#pragma unroll
        for (int i = 0; i < kDigits; i++) {
            const uint32_t r = i == D_PART ? (uint32_t)S->part_n : S->radix[i];
            const uint32_t q = w / r;
            const uint32_t d = w - q * r;
            if (i == D_PART) L.part = d;
            else L.d[i] = d;
            w = q;
        }
    } else {
        // 64-bit divisions only while the quotient still needs them (a few fast digits of
        // a >= 2^32 index; radix-1 digits cost nothing)
#pragma unroll
        for (int i = 0; i < kDigits; i++) {
            if (i == D_PART) {
                uint64_t np = S->part_n;
                L.part = u % np;
                u /= np;
            } else {
                const uint32_t r = S->radix[i];
                if (r == 1) {
                    L.d[i] = 0;
                } else if ((u >> 32) == 0) {
                    const uint32_t w = (uint32_t)u, q = w / r;
                    L.d[i] = w - q * r;
                    u = q;
                } else {
                    L.d[i] = (uint32_t)(u % r);
                    u /= r;
                }
            }
        }
    }
    L.ns = 1;
    if (S->part_mode == PARADL_PART_COMB) unrank_comb(v, L.part, L, cuts, cs);
    else if (S->part_mode == PARADL_PART_MASK) L.ns = __popcll(L.part) + 1;
#if PARADL_CHECKS
    for (int i = 0; i < kDigits; i++) PCHECK(i == D_PART || L.d[i] < S->radix[i]);
    PCHECK(L.part < S->part_n || S->part_n == 0);
    PCHECK(S->part_mode != PARADL_PART_COMB || (L.ns >= S->s_min && L.ns <= S->s_max));
#endif
}

// Adds the lane stride (mixed-radix digits inc[]) to the digit vector; returns the
// slowest digit that changed (-1: none).
__device__ __forceinline__ int advance(const WorkItem &a, const View &v, Lane &L, uint16_t *cuts,
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
// stage_span folds stages i0..i1-1 (stage i ends at cut i, the last one at G; COMB cuts) that
// start at row beg into st; all terms are exact int64 maxima / sums, so any split of the
// stage list composes to the same StageT.
__device__ __forceinline__ void stage_span(const View &v, const uint16_t *cuts, int cs, int64_t twob, int ns,
                                           int i0, int i1, int beg, StageT &st) {
    const ModelHdr *M = v.M;
    const int64_t *PF = at<int64_t>(v.mb, M->off_pf);
    const int64_t *PB = at<int64_t>(v.mb, M->off_pb);
    const int64_t *PU = at<int64_t>(v.mb, M->off_pu);
    const int64_t *PW = at<int64_t>(v.mb, M->off_pw);
    const int64_t *PX = at<int64_t>(v.mb, M->off_pxy);
    const int64_t *PI = at<int64_t>(v.mb, M->off_pbi);
    const int64_t *Y = at<int64_t>(v.mb, M->off_y);
    // prefix values at the stage start, carried from the previous stage end
    int64_t bF = PF[beg], bB = PB[beg], bU = PU[beg], bW = PW[beg], bX = PX[beg], bI = PI[beg];
    for (int i = i0; i < i1; i++) {
        const int end = i == ns - 1 ? M->G : cuts[i * cs];
        const int64_t eF = PF[end], eB = PB[end], eU = PU[end], eW = PW[end], eX = PX[end], eI = PI[end];
        const int64_t F = eF - bF, B = eB - bB, U = eU - bU;
        const int64_t Wt = eW - bW, XY = eX - bX, BI = eI - bI;
        bF = eF, bB = eB, bU = eU, bW = eW, bX = eX, bI = eI;
        st.maxF = F > st.maxF ? F : st.maxF;
        st.maxB = B > st.maxB ? B : st.maxB;
        st.maxU = U > st.maxU ? U : st.maxU;
        st.maxW = Wt > st.maxW ? Wt : st.maxW;
        const int64_t mem = twob * XY + 2 * Wt + BI;
        st.memI = mem > st.memI ? mem : st.memI;
        if (i < ns - 1) {
            const int64_t y = Y[end - 1];
            st.maxY = y > st.maxY ? y : st.maxY;
            st.sumY += y;
        }
    }
}

__device__ void stage_terms(const View &v, const Lane &L, const uint16_t *cuts, int cs, int64_t b,
                            StageT &st) {
    st.maxF = st.maxB = st.maxU = st.maxW = st.maxY = st.sumY = st.memI = 0;
    if (v.S->part_mode != PARADL_PART_MASK) {
        stage_span(v, cuts, cs, 2 * b, L.ns, 0, L.ns, 0, st);
        return;
    }
    const ModelHdr *M = v.M;
    const int64_t *PF = at<int64_t>(v.mb, M->off_pf);
    const int64_t *PB = at<int64_t>(v.mb, M->off_pb);
    const int64_t *PU = at<int64_t>(v.mb, M->off_pu);
    const int64_t *PW = at<int64_t>(v.mb, M->off_pw);
    const int64_t *PX = at<int64_t>(v.mb, M->off_pxy);
    const int64_t *PI = at<int64_t>(v.mb, M->off_pbi);
    const int64_t *Y = at<int64_t>(v.mb, M->off_y);
    const int G = M->G;
    const int64_t twob = 2 * b;
    uint64_t mask = L.part;
    int64_t bF = PF[0], bB = PB[0], bU = PU[0], bW = PW[0], bX = PX[0], bI = PI[0];
    for (int i = 0; i < L.ns; i++) {
        int end;
        if (i == L.ns - 1) {
            end = G;
        } else {
            end = __ffsll((long long)mask);   // bit j set <=> cut after row j+1
            mask &= mask - 1;
        }
        const int64_t eF = PF[end], eB = PB[end], eU = PU[end], eW = PW[end], eX = PX[end], eI = PI[end];
        const int64_t F = eF - bF, B = eB - bB, U = eU - bU;
        const int64_t Wt = eW - bW, XY = eX - bX, BI = eI - bI;
        bF = eF, bB = eB, bU = eU, bW = eW, bX = eX, bI = eI;
        st.maxF = F > st.maxF ? F : st.maxF;
        st.maxB = B > st.maxB ? B : st.maxB;
        st.maxU = U > st.maxU ? U : st.maxU;
        st.maxW = Wt > st.maxW ? Wt : st.maxW;
        const int64_t mem = twob * XY + 2 * Wt + BI;
        st.memI = mem > st.memI ? mem : st.memI;
        if (i < L.ns - 1) {
            const int64_t y = Y[end - 1];
            st.maxY = y > st.maxY ? y : st.maxY;
            st.sumY += y;
        }
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
    double ag_c, ag_na, ag_s, ar_mult;
    int ag_t;
    bool ag_on;           // filter/channel/df Allgather phase (Allreduce = 2x)
    double h_na, h_s;
    int h_t;
    bool h_on;            // spatial/ds halo 2 (na alpha + s beta)
    double pp_c, pp_na, pp_s;
    int pp_t;
    bool pp_on;           // pipeline c (alpha + s beta) / layer-pure 2 (na alpha + s beta)
    double *gp;           // GPIPE: this lane's stage table f[i], g[i], m[i], u[i] at gp[(4i+k)*gps]
    int gps, gS, gns;     // table stride, segments S, stage count s
    const double *lwt;    // DATA_LW: the work item's [n_dims][lwn][2] table of (c_l, s_l); row of
    int lwn;              // the current dims value after compute_mid; lwn weighted layers
    // memoised divisions (same operands -> same IEEE result; recomputed when an operand changes)
    double R_memo, tau_memo;
    int64_t B_memo;
    double I_memo;
    int64_t bS_b, bS_S;
    double bS_memo;
    // LAYERWISE: the strategy assignment's row sums, kept while the mask repeats (the dims,
    // b and slower digits change the products only)
    uint64_t lw_mask;
    int64_t lw_WUF, lw_WF, lw_XYF, lw_NCF, lw_YCF, lw_nT, lw_YT, lw_FminF;
    int32_t lw_ncomm, lw_nF;
    __device__ void reset_memo() {
        R_memo = -1.0;
        B_memo = -1;
        bS_b = bS_S = -1;
        lw_mask = ~0ull;
    }
};

// comp row of Table 2: ((B FB)/p_c) tau + (WU/p_u) tau
// x / 1.0 == x exactly, so a division by 1 is skipped
// and x / 2^k is x * 2^-k exactly (integer numerators: the quotient is 0 or >= 2^-62, never
// subnormal), so only a non-power-of-two divisor pays a true IEEE division
__device__ __forceinline__ double div_i(int64_t num, int64_t den) {
    if (den == 1) return i2d(num);
    if ((den & (den - 1)) == 0) {
        const int k = 63 - __clzll(den);
        return dmul(i2d(num), __hiloint2double((1023 - k) << 20, 0));
    }
    return ddiv(i2d(num), i2d(den));
}
// a division taken only when a memoised operand changes: out of line, so the compiler
// cannot if-convert it into every call
__device__ __noinline__ double ddiv_rare(double a, double b) { return ddiv(a, b); }
__device__ __forceinline__ double comp_term(int64_t BFB, int64_t WU, int64_t pc, int64_t pu, double tau) {
    return dadd(dmul(div_i(BFB, pc), tau), dmul(div_i(WU, pu), tau));
}
// mem row of Table 2: gamma (delta ((2B XY)/p_a + (2W)/p_w + BI))
__device__ __forceinline__ double mem_term(const ImgHdr *H, int64_t twoBXY, int64_t W, int64_t BI,
                                           int64_t pa, int64_t pw) {
    return dmul(H->gamma, dmul(i2d(H->delta), dadd(dadd(div_i(twoBXY, pa), div_i(2 * W, pw)), i2d(BI))));
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
__device__ void compute_mid(const View &v, const Lane &L, const StageT &st, Mid &m, const HaloEntry *halo = nullptr) {
    const ImgHdr *H = v.H;
    const SubHdr *S = v.S;
    const ModelHdr *M = v.M;
    const double cap = at<double>(v.img, S->off_cap)[L.d[D_CAP]];
    const double R = at<double>(v.img, S->off_flops)[L.d[D_FLOPS]];
    if (R != m.R_memo) {
        m.R_memo = R;
        m.tau_memo = ddiv_rare(1.0, R);
    }
    const double tau = m.tau_memo;
    const int64_t b = at<int64_t>(v.img, S->off_b)[L.d[D_B]];
    const int32_t *dm = at<int32_t>(v.img, S->off_dims) + 4 * L.d[D_DIMS];
    const int64_t delta = H->delta;
    const int64_t dW = delta * M->W;
    uint32_t reason = 0;
    m.ge.on = m.ge2.on = m.ag_on = m.h_on = m.pp_on = false;
    m.ar_mult = H->ar_mult;
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
        m.ge = make_ar(H, p, i2d(dW), div_i(dW, p), t);
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
        if (halo) {
            const HaloEntry &he = halo[L.d[D_DIMS] * S->radix[D_LS] + L.d[D_LS]];
            NS = he.NS;
            HV = he.HV;
            reason |= he.reason;
        } else {
            reason |= spatial_terms(v, Ls, split, NS, HV);
        }
        const int ti = tier_of(H, p2), to = tier_of(H, p);
        reason |= flag_tier(ti) | flag_tier(to);
        m.h_on = p2 > 1;
        m.h_na = i2d(2 * NS);
        m.h_s = i2d(b * delta * HV);
        m.h_t = p2p_tier(H, ti);
        if (FAM == PARADL_DS) m.phi = p1 > 1 ? H->phi_ds : 1.0;   // concurrent reduce-to-leader (Q40)
        if (FAM == PARADL_SPATIAL) {
            m.ge = make_ar(H, p, i2d(dW), div_i(dW, p), to);
        } else {
            m.ge = make_ar(H, p2, i2d(dW), div_i(dW, p2), ti);   // reduce to leader
            m.ge2 = make_ar(H, p1, i2d(dW), div_i(dW, p1), to);  // Allreduce among leaders
        }
        m.mem = mem_term(H, 2 * B * M->XY, M->W, M->BI, p, 1);
    } else if (FAM == PARADL_DATA_LW) {   // Data row, one Allreduce per weighted layer (Q37)
        p = dm[0];
        B = b * p;
        m.comp = comp_term(B * M->FB, M->WU, p, 1, tau);
        const int t = tier_of(H, p);
        reason |= flag_tier(t);
        m.pp_t = t;
        m.lwt += (size_t)L.d[D_DIMS] * m.lwn * 2;
        m.mem = mem_term(H, 2 * B * M->XY, M->W, M->BI, p, 1);
        if (p > B) reason |= PARADL_R_SCALING;
    } else if (FAM == PARADL_SPATIAL_AG) {
        // Spatial on rows [0, Ls), Allgather of y_Ls, rows [Ls, G) replicated (Q35):
        // comp = ((B FB_pre / p) tau + (B FB_suf) tau) + WU tau; GE = AR(p, delta W);
        // AG = (p-1)(alpha + (B delta |y_Ls| / p) beta); halo as Spatial over the prefix;
        // mem = gamma (delta (((2B XY_pre)/p + 2B XY_suf) + 2W) + BI)
        const int32_t split[3] = {dm[1], dm[2], dm[3]};
        p = (int64_t)dm[1] * dm[2] * dm[3];
        B = b;
        const int32_t Ls = at<int32_t>(v.img, S->off_Ls)[L.d[D_LS]];
        const int Lp = Ls < M->G ? Ls : M->G;
        const int64_t *PF = at<int64_t>(v.mb, M->off_pf);
        const int64_t *PB = at<int64_t>(v.mb, M->off_pb);
        const int64_t *PX = at<int64_t>(v.mb, M->off_pxy);
        const int64_t *Y = at<int64_t>(v.mb, M->off_y);
        const int64_t FBp = PF[Lp] + PB[Lp], XYp = PX[Lp];
        m.comp = dadd(dadd(dmul(div_i(B * FBp, p), tau), dmul(i2d(B * (M->FB - FBp)), tau)), dmul(i2d(M->WU), tau));
        int64_t NS, HV;
        if (halo) {
            const HaloEntry &he = halo[L.d[D_DIMS] * S->radix[D_LS] + L.d[D_LS]];
            NS = he.NS;
            HV = he.HV;
            reason |= he.reason;
        } else {
            reason |= spatial_terms(v, Ls, split, NS, HV);
        }
        const int t = tier_of(H, p);
        reason |= flag_tier(t);
        m.h_on = p > 1;
        m.h_na = i2d(2 * NS);
        m.h_s = i2d(b * delta * HV);
        m.h_t = p2p_tier(H, t);
        m.ge = make_ar(H, p, i2d(dW), div_i(dW, p), t);
        m.ag_on = Lp < M->G && p > 1;
        m.ag_c = i2d(p - 1);
        m.ag_na = 1.0;
        m.ag_s = div_i(B * delta * Y[Lp - 1], p);
        m.ag_t = t;
        m.mem = dmul(H->gamma, dmul(i2d(delta), dadd(dadd(dadd(div_i(2 * B * XYp, p), i2d(2 * B * (M->XY - XYp))),
                                                          i2d(2 * M->W)),
                                                     i2d(M->BI))));
    } else if (FAM == PARADL_GPIPE) {
        // GPipe schedule (Q36): per-stage f = ((b/S) FW_i) tau, g = ((b/S) BW_i) tau,
        // m = (b/S) delta |y_i| (boundary message, c_i = alpha + m beta), u = WU_i tau, written
        // to the lane's stage table; the schedule itself runs per (alpha, beta) in gpipe_time()
        const int ns = L.ns;
        const int64_t Sg = at<int32_t>(v.img, S->off_S)[L.d[D_S]];
        p = ns;
        B = b;
        const int ts = tier_of(H, ns);
        reason |= flag_tier(ts);
        if (b != m.bS_b || Sg != m.bS_S) {
            m.bS_b = b;
            m.bS_S = Sg;
            m.bS_memo = div_i(b, Sg);
        }
        m.comp = 0.0;
        m.pp_t = p2p_tier(H, ts);
        m.gS = (int)Sg;
        m.gns = ns;
        m.mem = dmul(H->gamma, dmul(i2d(delta), i2d(st.memI)));
        if (Sg > b) reason |= PARADL_R_SEGMENTS;
    } else if (FAM == PARADL_LAYERWISE) {
        // Per-layer strategy (Q39): bit j of the partition digit
        // makes the j-th COMM row filter-parallel (else data-parallel) over the same p PEs;
        // other rows follow the COMM row before them.  Exact int64 sums over the rows by
        // prefix differences: WU, W, XY of the data (D) and filter (F) rows, the filter COMM
        // rows' Allgather messages (NC_F, YC_F; the model's last COMM row excluded, Q10) and
        // limit (min F), the strategy changes (n_T messages of Y_T b-sample elements).
        p = dm[0];
        B = b * p;
        const RowGeo *geo = at<RowGeo>(v.mb, M->off_geo);
        const int64_t *PU = at<int64_t>(v.mb, M->off_pu);
        const int64_t *PW = at<int64_t>(v.mb, M->off_pw);
        const int64_t *PX = at<int64_t>(v.mb, M->off_pxy);
        const int64_t *Y = at<int64_t>(v.mb, M->off_y);
        const uint64_t mask = L.part;
        const int G = M->G;
        if (mask != m.lw_mask) {
            m.lw_mask = mask;
            int last_comm = -1, first_comm = -1;
            for (int l = 0; l < G; l++)
                if (geo[l].flags & PARADL_FLAG_COMM) {
                    if (first_comm < 0) first_comm = l;
                    last_comm = l;
                }
            int cur = first_comm >= 0 ? (int)(mask & 1) : 0;
            int64_t WUF = 0, WF = 0, XYF = 0, NCF = 0, YCF = 0, nT = 0, YT = 0, FminF = INT64_MAX;
            int ncomm = 0, nF = 0;
            for (int l = 0; l < G; l++) {
                if (geo[l].flags & PARADL_FLAG_COMM) {
                    const int sf = (int)((mask >> ncomm) & 1);
                    if (ncomm > 0 && sf != cur) {
                        nT += sf ? 2 : 1;
                        YT += sf ? 2 * Y[l - 1] : Y[l - 1];
                    }
                    cur = sf;
                    ncomm++;
                    if (cur) {
                        nF++;
                        FminF = min(FminF, (int64_t)geo[l].F);
                        if (l != last_comm) {
                            NCF++;
                            YCF += Y[l];
                        }
                    }
                }
                if (cur) {
                    WUF += PU[l + 1] - PU[l];
                    WF += PW[l + 1] - PW[l];
                    XYF += PX[l + 1] - PX[l];
                }
            }
            m.lw_WUF = WUF, m.lw_WF = WF, m.lw_XYF = XYF, m.lw_NCF = NCF, m.lw_YCF = YCF;
            m.lw_nT = nT, m.lw_YT = YT, m.lw_FminF = FminF, m.lw_ncomm = ncomm, m.lw_nF = nF;
        }
        const int64_t WUF = m.lw_WUF, WF = m.lw_WF, XYF = m.lw_XYF, NCF = m.lw_NCF, YCF = m.lw_YCF;
        const int64_t nT = m.lw_nT, YT = m.lw_YT, FminF = m.lw_FminF;
        const int ncomm = m.lw_ncomm, nF = m.lw_nF;
        const int64_t WUD = M->WU - WUF, WD = M->W - WF, XYD = M->XY - XYF;
        // comp = ((B FB)/p) tau + (WU_D + WU_F/p) tau
        m.comp = dadd(dmul(div_i(B * M->FB, p), tau), dmul(dadd(i2d(WUD), div_i(WUF, p)), tau));
        const int t = tier_of(H, p);
        reason |= flag_tier(t);
        m.ge.c = m.ge.s = 0.0;   // no data row (every COMM row filter-parallel): no gradient Allreduce
        m.ge.t = t;
        if (!(ncomm > 0 && nF == ncomm)) m.ge = make_ar(H, p, i2d(delta * WD), div_i(delta * WD, p), t);
        m.ag_on = p > 1 && (nF > 0 || nT > 0);
        m.ag_c = i2d(p - 1);
        m.ag_na = i2d(NCF);
        m.ag_s = div_i(B * delta * YCF, p);
        m.ag_t = t;
        m.pp_on = m.ag_on;   // strategy changes: (p - 1)(n_T alpha + (b delta Y_T) beta)
        m.pp_c = m.ag_c;
        m.pp_na = i2d(nT);
        m.pp_s = i2d(b * delta * YT);
        m.pp_t = t;
        m.mem = dmul(H->gamma, dmul(i2d(delta), dadd(dadd(dadd(div_i(2 * B * XYD, p), i2d(2 * B * XYF)),
                                                          dadd(i2d(2 * WD), div_i(2 * WF, p))),
                                                     i2d(M->BI))));
        if (nF > 0 && p > FminF) reason |= PARADL_R_SCALING;
    } else if (FAM == PARADL_FILTER || FAM == PARADL_CHANNEL) {   // Filter / Channel rows
        p = dm[0];
        B = b;
        m.comp = comp_term(B * M->FB, M->WU, p, p, tau);
        const int t = tier_of(H, p);
        reason |= flag_tier(t);
        m.ag_on = p > 1;
        m.ag_c = i2d(p - 1);
        m.ag_na = i2d(M->NC);
        m.ag_s = div_i(B * delta * M->YC, p);
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
        m.ag_s = div_i(B * delta * M->YC, p);
        m.ag_t = ti;
        m.phi = p2 > 1 ? H->phi_df : 1.0;
        m.ge = make_ar(H, p1, div_i(dW, p2), div_i(dW, p), to);
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
            m.pp_t = p2p_tier(H, ts);
        } else {
            if (b != m.bS_b || Sg != m.bS_S) {
                m.bS_b = b;
                m.bS_S = Sg;
                m.bS_memo = div_i(b, Sg);
            }
            const double bS = m.bS_memo;
            const double cseg = dmul(i2d(ns + Sg - 1), bS);
            m.comp = dadd(dmul(dmul(cseg, i2d(st.maxF + st.maxB)), tau), dmul(i2d(st.maxU), tau));
            m.pp_on = ns > 1;
            m.pp_c = i2d(2 * (ns + Sg - 2));
            m.pp_s = dmul(bS, i2d(delta * st.maxY));
            m.pp_t = p2p_tier(H, ts);
            if (FAM == PARADL_PD) {
                const int tp = tier_of(H, p);
                reason |= flag_tier(tp);
                const double mW = i2d(delta * st.maxW);
                m.ge = make_ar(H, pd, mW, div_i(delta * st.maxW, pd), tp);
                m.phi = ns > 1 ? H->phi_pd : 1.0;   // the s stage Allreduces at once (Q40)
            }
        }
        m.mem = dmul(H->gamma, dmul(i2d(delta), i2d(st.memI)));
        if (Sg < 1 || Sg > b) reason |= PARADL_R_SEGMENTS;
    }
    if (B != m.B_memo) {
        m.B_memo = B;
        m.I_memo = div_i(M->D, B);   // Table 1: I = D/B
    }
    m.I = m.I_memo;
    if (!(m.mem <= cap)) reason |= PARADL_R_MEMORY;
    m.reason = reason;
    m.B = B;
    m.p = p;
}

// GPIPE stage table of the lane (after compute_mid<PARADL_GPIPE>, which set m.bS_memo = b/S
// and m.tau_memo): per stage i, f = ((b/S) FW_i) tau, g = ((b/S) BW_i) tau, m = (b/S)(delta
// |y_i|) for i < s-1 (else 0), u = WU_i tau; stage sums by prefix differences (exact int64).
__device__ void gpipe_fill(const View &v, const Lane &L, const uint16_t *cuts, int cs, Mid &m) {
    const ModelHdr *M = v.M;
    const int64_t *PF = at<int64_t>(v.mb, M->off_pf);
    const int64_t *PB = at<int64_t>(v.mb, M->off_pb);
    const int64_t *PU = at<int64_t>(v.mb, M->off_pu);
    const int64_t *Y = at<int64_t>(v.mb, M->off_y);
    const int64_t delta = v.H->delta;
    const double mb = m.bS_memo, tau = m.tau_memo;
    const bool maskm = v.S->part_mode == PARADL_PART_MASK;
    uint64_t mask = L.part;
    int beg = 0;
    for (int i = 0; i < L.ns; i++) {
        int end;
        if (i == L.ns - 1) end = M->G;
        else if (maskm) {
            end = __ffsll((long long)mask);   // bit j set <=> cut after row j+1
            mask &= mask - 1;
        } else end = cuts[i * cs];
        double *q = m.gp + (size_t)(4 * i) * m.gps;
        q[0] = dmul(dmul(mb, i2d(PF[end] - PF[beg])), tau);
        q[m.gps] = dmul(dmul(mb, i2d(PB[end] - PB[beg])), tau);
        q[2 * m.gps] = i < L.ns - 1 ? dmul(mb, i2d(delta * Y[end - 1])) : 0.0;
        q[3 * m.gps] = dmul(i2d(PU[end] - PU[beg]), tau);
        beg = end;
    }
}

// The GPipe schedule (Q36) for NC (alpha, beta) pairs of the stage tier,
// evaluated as NC interleaved chains (ILP): S segments flow through the NS stages; forward
// stage i is busy f_i + c_i (blocking send of y_i, c_i = alpha + m_i beta), backward stage i
// is busy g_i + c_{i-1}; backward starts at the forward makespan; stage i applies WU after its
// last backward segment.  Each task starts at max(stage free, input delivered) -- the oracle's
// event simulation, whose additions this performs operand for operand.  The maxima the
// oracle takes against a value known to be smaller are skipped (max returns an operand
// exactly): stage 0 forward is ready at 0 <= its free time; segment 0 finds every stage free
// before its input arrives (free = 0 forward, = t_f <= ready backward); the last stage's
// backward input is ready at t_f <= its free time.
#ifndef PARADL_GP_QUAD
#define PARADL_GP_QUAD 2
#endif
constexpr uint32_t kGpQuad = PARADL_GP_QUAD;   // GPipe configurations per schedule call
#ifndef PARADL_LW_QUAD
#define PARADL_LW_QUAD 4
#endif
constexpr uint32_t kLwQuad = PARADL_LW_QUAD;   // DATA_LW configurations per interleaved fold

// max of two non-negative, non-NaN doubles as one compare + two 32-bit selects (fmax adds
// NaN handling: a third ALU instruction per max on sm_100a, which has no DMNMX)
__device__ __forceinline__ double dmax_nn(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double dmin_nn(double a, double b) { return a < b ? a : b; }

template <int NS, int NC>
__device__ __forceinline__ void gp_chains(const double *q, int gs, int S, const double *a, const double *be,
                                          double *t) {
    double dfw[NC][NS], dbw[NC][NS], fr[NC][NS];
#pragma unroll
    for (int i = 0; i < NS; i++) {
        const double f = q[(4 * i) * gs], g = q[(4 * i + 1) * gs];
#pragma unroll
        for (int c = 0; c < NC; c++) {
            dfw[c][i] = f;
            dbw[c][i] = g;
        }
    }
#pragma unroll
    for (int i = 0; i + 1 < NS; i++) {
        const double mi = q[(4 * i + 2) * gs];
#pragma unroll
        for (int c = 0; c < NC; c++) {
            const double ci = dadd(a[c], dmul(mi, be[c]));
            dfw[c][i] = dadd(dfw[c][i], ci);
            dbw[c][i + 1] = dadd(dbw[c][i + 1], ci);
        }
    }
    // forward wave, segment 0 then 1..S-1
#pragma unroll
    for (int c = 0; c < NC; c++) {
        fr[c][0] = dfw[c][0];
#pragma unroll
        for (int i = 1; i < NS; i++) fr[c][i] = dadd(fr[c][i - 1], dfw[c][i]);
    }
    for (int j = 1; j < S; j++) {
#pragma unroll
        for (int c = 0; c < NC; c++) {
            fr[c][0] = dadd(fr[c][0], dfw[c][0]);
#pragma unroll
            for (int i = 1; i < NS; i++) fr[c][i] = dadd(dmax_nn(fr[c][i], fr[c][i - 1]), dfw[c][i]);
        }
    }
    // backward wave (GPipe flush at t_f = fr[NS-1]), segment 0 then 1..S-1
#pragma unroll
    for (int c = 0; c < NC; c++) {
        fr[c][NS - 1] = dadd(fr[c][NS - 1], dbw[c][NS - 1]);
#pragma unroll
        for (int i = NS - 2; i >= 0; i--) fr[c][i] = dadd(fr[c][i + 1], dbw[c][i]);
    }
    for (int j = 1; j < S; j++) {
#pragma unroll
        for (int c = 0; c < NC; c++) {
            fr[c][NS - 1] = dadd(fr[c][NS - 1], dbw[c][NS - 1]);
#pragma unroll
            for (int i = NS - 2; i >= 0; i--) fr[c][i] = dadd(dmax_nn(fr[c][i], fr[c][i + 1]), dbw[c][i]);
        }
    }
    // weight update after each stage's last backward segment
#pragma unroll
    for (int i = 0; i < NS; i++) {
        const double u = q[(4 * i + 3) * gs];
#pragma unroll
        for (int c = 0; c < NC; c++) {
            const double e = dadd(fr[c][i], u);
            t[c] = i == 0 ? e : dmax_nn(t[c], e);   // the oracle's max(0, e_0) = e_0 (e_0 >= 0)
        }
    }
}

#ifndef PARADL_GP_INLINE
#define PARADL_GP_INLINE 1
#endif
#if PARADL_GP_INLINE
#define PARADL_GP_ATTR __forceinline__
#else
#define PARADL_GP_ATTR __noinline__
#endif
// NC configurations at once: up to 4 stages as NC interleaved chains; beyond that (more
// registers per chain) as NC/2-wide halves
template <int NC>
__device__ PARADL_GP_ATTR void gpipe_eval(const double *q, int gs, int ns, int S, const double *a, const double *be,
                                        double *t) {
    constexpr int H = NC > 2 ? 2 : NC;
    switch (ns) {
    case 1: gp_chains<1, NC>(q, gs, S, a, be, t); break;
    case 2: gp_chains<2, NC>(q, gs, S, a, be, t); break;
    case 3: gp_chains<3, NC>(q, gs, S, a, be, t); break;
    case 4: gp_chains<4, NC>(q, gs, S, a, be, t); break;
    default:
#pragma unroll 1
        for (int h = 0; h < NC; h += H) {
            switch (ns) {
            case 5: gp_chains<5, H>(q, gs, S, a + h, be + h, t + h); break;
            case 6: gp_chains<6, H>(q, gs, S, a + h, be + h, t + h); break;
            case 7: gp_chains<7, H>(q, gs, S, a + h, be + h, t + h); break;
            default: gp_chains<kGpMax, H>(q, gs, S, a + h, be + h, t + h); break;
            }
        }
        break;
    }
}

__device__ __forceinline__ double gpipe_time(const Mid &m, double a, double be) {
    double t[1];
    gpipe_eval<1>(m.gp, m.gps, m.gns, m.gS, &a, &be, t);
    return t[0];
}

// NC interleaved folds (independent configurations, same table): ILP for the serial chain
template <int NC>
__device__ __forceinline__ void lw_ge_n(const double *tab, int n, const double *a, const double *be, double *ge) {
#pragma unroll
    for (int c = 0; c < NC; c++) ge[c] = 0.0;
    for (int j = 0; j < n; j++) {
        const double2 q = *reinterpret_cast<const double2 *>(tab + 2 * j);
#pragma unroll
        for (int c = 0; c < NC; c++) ge[c] = dadd(ge[c], dmul(q.x, dadd(a[c], dmul(q.y, be[c]))));
    }
}

// DATA_LW gradient exchange: left fold over the weighted layers of c_l (alpha + s_l beta),
// the per-message Allreduce of the table built by build_memo (ring or tree per message)
__device__ __forceinline__ double lw_ge(const double *tab, int n, double a, double be) {
    double ge = 0.0;
    int j = 0;
    for (; j + 2 <= n; j += 2) {   // two loads of (c, s) pairs per step; the fold stays in order
        const double4 q = *reinterpret_cast<const double4 *>(tab + 2 * j);
        ge = dadd(ge, dmul(q.x, dadd(a, dmul(q.y, be))));
        ge = dadd(ge, dmul(q.z, dadd(a, dmul(q.w, be))));
    }
    if (j < n) ge = dadd(ge, dmul(tab[2 * j], dadd(a, dmul(tab[2 * j + 1], be))));
    return ge;
}

struct Phases {
    double comp, ge, ag, ar, halo, p2p;
};

// alpha/beta-dependent part and the t_iter fold ((((comp+GE)+AG)+AR)+Halo)+P2P.
// EXPLAIN: also report phases, with +inf for a phase whose tier is missing.
template <int FAM, bool EXPLAIN, bool CHECK_TIER = true>
__device__ __forceinline__ double inner(const Mid &m, const double *arow, const double *brow, Phases *ph) {
    double ge = 0.0, ag = 0.0, ar = 0.0, halo = 0.0, p2p = 0.0;
    double t = m.comp;
    if (!EXPLAIN && CHECK_TIER && (m.reason & PARADL_R_TIER)) return CUDART_INF;
    if (FAM == PARADL_DATA_LW) {
        ge = (EXPLAIN && m.pp_t < 0) ? CUDART_INF : lw_ge(m.lwt, m.lwn, arow[max(m.pp_t, 0)], brow[max(m.pp_t, 0)]);
        t = dadd(t, ge);
        if (EXPLAIN) {
            ph->comp = m.comp;
            ph->ge = ge;
            ph->ag = ph->ar = ph->halo = ph->p2p = 0.0;
        }
        return t;
    }
    if (FAM == PARADL_GPIPE) {
        t = (EXPLAIN && m.pp_t < 0) ? CUDART_INF : gpipe_time(m, arow[max(m.pp_t, 0)], brow[max(m.pp_t, 0)]);
        if (EXPLAIN) {
            ph->comp = t;
            ph->ge = ph->ag = ph->ar = ph->halo = ph->p2p = 0.0;
        }
        return t;
    }
    auto ar_eval = [&](const ARt &r, double phi, bool use_phi) -> double {
        if (!r.on) return 0.0;
        if (EXPLAIN && r.t < 0) return CUDART_INF;
        const double bh = use_phi ? dmul(brow[r.t], phi) : brow[r.t];
        return dmul(r.c, dadd(arow[r.t], dmul(r.s, bh)));
    };
    if (FAM == PARADL_DATA || FAM == PARADL_SPATIAL || FAM == PARADL_SPATIAL_AG) {
        ge = ar_eval(m.ge, 1.0, false);
        if (m.ge.on) t = dadd(t, ge);
    }
    if (FAM == PARADL_PD) {
        ge = ar_eval(m.ge, m.phi, true);
        if (m.ge.on) t = dadd(t, ge);
    }
    if (FAM == PARADL_SPATIAL_AG && m.ag_on) {   // boundary Allgather
        if (EXPLAIN && m.ag_t < 0) ag = CUDART_INF;
        else ag = dmul(m.ag_c, dadd(arow[m.ag_t], dmul(m.ag_s, brow[m.ag_t])));
        t = dadd(t, ag);
    }
    if (FAM == PARADL_DS) {
        ge = dadd(ar_eval(m.ge, m.phi, true), ar_eval(m.ge2, 1.0, false));
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
            ar = dmul(m.ar_mult, ag);
            t = dadd(dadd(t, ag), ar);
        }
    }
    if (FAM == PARADL_LAYERWISE) {
        ge = ar_eval(m.ge, 1.0, false);
        if (m.ge.on) t = dadd(t, ge);
        if (m.ag_on) {
            double agf, tr;
            if (EXPLAIN && m.ag_t < 0) agf = tr = CUDART_INF;
            else {
                agf = dmul(m.ag_c, dadd(dmul(m.ag_na, arow[m.ag_t]), dmul(m.ag_s, brow[m.ag_t])));
                tr = dmul(m.pp_c, dadd(dmul(m.pp_na, arow[m.pp_t]), dmul(m.pp_s, brow[m.pp_t])));
            }
            ag = dadd(agf, tr);
            ar = dmul(m.ar_mult, agf);
            t = dadd(dadd(t, ag), ar);
        }
    }
    if (FAM == PARADL_SPATIAL || FAM == PARADL_DS || FAM == PARADL_SPATIAL_AG) {
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

// Branch-free form of inner() for the sweep's hot loop: absent phases carry zero
// coefficients (t + 0*x == t exactly for finite x), tiers are clamped to a valid row.
// Only used where no tier is missing (reduce mode evaluates feasible configs only;
// dense mode checks PARADL_R_TIER first), so results equal inner() bit for bit.
__device__ __forceinline__ void fastify(Mid &m) {
    if (!m.ge.on) m.ge.c = m.ge.s = 0.0;
    if (!m.ge2.on) m.ge2.c = m.ge2.s = 0.0;
    if (!m.ag_on) m.ag_c = m.ag_na = m.ag_s = 0.0;
    if (!m.h_on) m.h_na = m.h_s = 0.0;
    if (!m.pp_on) m.pp_c = m.pp_na = m.pp_s = 0.0;
    m.ge.t = max(m.ge.t, 0);
    m.ge2.t = max(m.ge2.t, 0);
    m.ag_t = max(m.ag_t, 0);
    m.h_t = max(m.h_t, 0);
    m.pp_t = max(m.pp_t, 0);
}

// The alpha/beta-dependent part split into alpha-derived values (one alpha row), beta-slot
// values (products s*beta, invariant over alpha) and their combination.  The operations
// and their order are exactly those of inner(); splitting only decides which results are
// computed once and reused.
struct AlphaV {
    double ge, ge2, ag, h, pp;
};
struct SlotV {
    double ge, ge2, ag, h, pp;
};

template <int FAM>
__device__ __forceinline__ void alpha_vals(const Mid &m, const double *arow, AlphaV &a) {
    if (FAM == PARADL_DATA || FAM == PARADL_SPATIAL || FAM == PARADL_PD || FAM == PARADL_DS || FAM == PARADL_DF ||
        FAM == PARADL_SPATIAL_AG || FAM == PARADL_LAYERWISE)
        a.ge = arow[m.ge.t];
    if (FAM == PARADL_LAYERWISE) {
        a.ag = dmul(m.ag_na, arow[m.ag_t]);
        a.pp = dmul(m.pp_na, arow[m.pp_t]);
    }
    if (FAM == PARADL_DS) a.ge2 = arow[m.ge2.t];
    if (FAM == PARADL_FILTER || FAM == PARADL_CHANNEL || FAM == PARADL_DF) a.ag = dmul(m.ag_na, arow[m.ag_t]);
    if (FAM == PARADL_SPATIAL_AG) a.ag = arow[m.ag_t];
    if (FAM == PARADL_SPATIAL || FAM == PARADL_DS || FAM == PARADL_SPATIAL_AG) a.h = dmul(m.h_na, arow[m.h_t]);
    if (FAM == PARADL_PIPELINE || FAM == PARADL_PD) a.pp = arow[m.pp_t];
    if (FAM == PARADL_LAYERPURE) a.pp = dmul(m.pp_na, arow[m.pp_t]);
}

template <int FAM>
__device__ __forceinline__ void slot_vals(const Mid &m, const double *brow, SlotV &v) {
    if (FAM == PARADL_DATA || FAM == PARADL_SPATIAL || FAM == PARADL_SPATIAL_AG || FAM == PARADL_LAYERWISE)
        v.ge = dmul(m.ge.s, brow[m.ge.t]);
    if (FAM == PARADL_PD || FAM == PARADL_DS) v.ge = dmul(m.ge.s, dmul(brow[m.ge.t], m.phi));
    if (FAM == PARADL_LAYERWISE) {
        v.ag = dmul(m.ag_s, brow[m.ag_t]);
        v.pp = dmul(m.pp_s, brow[m.pp_t]);
    }
    if (FAM == PARADL_DF) v.ge = dmul(m.ge.s, dmul(brow[m.ge.t], m.phi));
    if (FAM == PARADL_DS) v.ge2 = dmul(m.ge2.s, brow[m.ge2.t]);
    if (FAM == PARADL_FILTER || FAM == PARADL_CHANNEL || FAM == PARADL_DF || FAM == PARADL_SPATIAL_AG)
        v.ag = dmul(m.ag_s, brow[m.ag_t]);
    if (FAM == PARADL_SPATIAL || FAM == PARADL_DS || FAM == PARADL_SPATIAL_AG) v.h = dmul(m.h_s, brow[m.h_t]);
    if (FAM == PARADL_PIPELINE || FAM == PARADL_PD || FAM == PARADL_LAYERPURE) v.pp = dmul(m.pp_s, brow[m.pp_t]);
}

template <int FAM>
__device__ __forceinline__ double combine(const Mid &m, const AlphaV &a, const SlotV &v) {
    double t = m.comp;
    if (FAM == PARADL_DATA || FAM == PARADL_SPATIAL || FAM == PARADL_PD || FAM == PARADL_DF || FAM == PARADL_SPATIAL_AG)
        t = dadd(t, dmul(m.ge.c, dadd(a.ge, v.ge)));
    if (FAM == PARADL_SPATIAL_AG) t = dadd(t, dmul(m.ag_c, dadd(a.ag, v.ag)));
    if (FAM == PARADL_LAYERWISE) {
        t = dadd(t, dmul(m.ge.c, dadd(a.ge, v.ge)));
        const double agf = dmul(m.ag_c, dadd(a.ag, v.ag));
        t = dadd(dadd(t, dadd(agf, dmul(m.pp_c, dadd(a.pp, v.pp)))), dmul(m.ar_mult, agf));
    }
    if (FAM == PARADL_DS) t = dadd(t, dadd(dmul(m.ge.c, dadd(a.ge, v.ge)), dmul(m.ge2.c, dadd(a.ge2, v.ge2))));
    if (FAM == PARADL_FILTER || FAM == PARADL_CHANNEL || FAM == PARADL_DF) {
        const double ag = dmul(m.ag_c, dadd(a.ag, v.ag));
        t = dadd(dadd(t, ag), dmul(m.ar_mult, ag));
    }
    if (FAM == PARADL_SPATIAL || FAM == PARADL_DS || FAM == PARADL_SPATIAL_AG) t = dadd(t, dmul(2.0, dadd(a.h, v.h)));
    if (FAM == PARADL_PIPELINE || FAM == PARADL_PD) t = dadd(t, dmul(m.pp_c, dadd(a.pp, v.pp)));
    if (FAM == PARADL_LAYERPURE) t = dadd(t, dmul(2.0, dadd(a.pp, v.pp)));
    return t;
}

template <int FAM>
__device__ __forceinline__ double inner_fast(const Mid &m, const double *arow, const double *brow) {
    if constexpr (FAM == PARADL_GPIPE) return gpipe_time(m, arow[m.pp_t], brow[m.pp_t]);
    if constexpr (FAM == PARADL_DATA_LW) return dadd(m.comp, lw_ge(m.lwt, m.lwn, arow[m.pp_t], brow[m.pp_t]));
    AlphaV a;
    SlotV v;
    alpha_vals<FAM>(m, arow, a);
    slot_vals<FAM>(m, brow, v);
    return combine<FAM>(m, a, v);
}

// ------------------------------------------------------------------ a8: warp top-k
__device__ __forceinline__ bool hit_less(double ka, uint64_t ia, double kb, uint64_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// Sorted list of up to 64 (key, idx) entries of one warp, kept in shared memory (the CTA's
// merge buffer): lane l owns entries l (a) and l + 32 (b) and only ever touches those two, so
// the warp's own program order is the only ordering needed.  insert / batch load the two
// entries into registers, work on them with shuffles and store them back; the hot loops
// carry only th = entry k-1 (the admission threshold) and the admission bound.
struct WarpTopK {
    paradl_hit *L;   // this warp's 64 entries (shared memory)
    double thk;
    uint64_t thi;
    int k;
    // Admission bound shared by every warp of the call: the k-th key of ANY full warp list
    // bounds the global k-th key (that warp alone holds k entries <= it), so configs with a
    // larger key can never enter the global top-k.  Kept as the bit pattern of a
    // non-negative double (monotone as uint64) under atomicMin; ~0 = none yet.
    double adm;
    unsigned long long *gbound;
    unsigned long long gnext;   // bound loaded at the previous refresh (software-pipelined load)

    __device__ void init(int kk, paradl_hit *list, unsigned long long *g = nullptr) {
        const int lane = threadIdx.x & 31;
        k = kk;
        thk = adm = CUDART_INF;
        thi = ~0ull;
        gbound = g;
        gnext = ~0ull;
        L = list;
        L[lane].idx = L[lane + 32].idx = ~0ull;
        L[lane].key_epoch_s = L[lane + 32].key_epoch_s = CUDART_INF;
        __syncwarp();
    }
    __device__ __forceinline__ void load(double &ka, uint64_t &ia, double &kb, uint64_t &ib) const {
        const int lane = threadIdx.x & 31;
        ka = L[lane].key_epoch_s;
        ia = L[lane].idx;
        kb = L[lane + 32].key_epoch_s;
        ib = L[lane + 32].idx;
    }
    __device__ __forceinline__ void store(double ka, uint64_t ia, double kb, uint64_t ib) {
        const int lane = threadIdx.x & 31;
        L[lane].key_epoch_s = ka;
        L[lane].idx = ia;
        L[lane + 32].key_epoch_s = kb;
        L[lane + 32].idx = ib;
    }
    // adopt the shared bound loaded at the previous call and issue the next load, so the
    // global-memory latency overlaps the work in between (whole warp; broadcast load)
    // (blocking while this warp has no bound at all, e.g. short-lived warps of small launches)
    __device__ __forceinline__ static unsigned long long load_bound(const unsigned long long *p) {
#if PARADL_RELAXED_BOUND
        unsigned long long v;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
        return v;
#else
        return *(volatile const unsigned long long *)p;
#endif
    }
    __device__ __forceinline__ void refresh() {
        if (!gbound) return;
        unsigned long long g = gnext;
        if (adm == CUDART_INF) g = load_bound(gbound);
        gnext = load_bound(gbound);
        if (g != ~0ull) adm = dmin_nn(adm, dmin_nn(thk, __longlong_as_double((long long)g)));
    }
    // after thk changed: tighten adm and publish a full list's threshold
    __device__ __forceinline__ void publish() {
        if (thk < adm) {
            adm = thk;
            if (gbound && thk < CUDART_INF && (threadIdx.x & 31) == 0)
                atomicMin(gbound, (unsigned long long)__double_as_longlong(thk));
        }
    }
    // whole warp, uniform (key, idx)
    __device__ void insert(double key, uint64_t idx) {
        const int lane = threadIdx.x & 31;
        const unsigned full = 0xffffffffu;
        double ka, kb;
        uint64_t ia, ib;
        load(ka, ia, kb, ib);
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
        store(ka, ia, kb, ib);
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
        publish();
    }
    // compare-exchange with lane^j: keep the smaller (keep_min) or the larger entry
    __device__ __forceinline__ static void cx(double &k, uint64_t &i, int j, bool keep_min) {
        const double ok = __shfl_xor_sync(0xffffffffu, k, j);
        const uint64_t oi = __shfl_xor_sync(0xffffffffu, i, j);
        const bool other_less = hit_less(ok, oi, k, i);
        if (keep_min == other_less) {
            k = ok;
            i = oi;
        }
    }
    // ascending bitonic sort of one entry per lane
    __device__ __forceinline__ static void sort32(double &k, uint64_t &i) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int s = 2; s <= 32; s <<= 1)
#pragma unroll
            for (int j = s >> 1; j > 0; j >>= 1) cx(k, i, j, ((lane & s) == 0) == ((lane & j) == 0));
    }
    // ascending sort of a bitonic sequence held one entry per lane
    __device__ __forceinline__ static void merge32(double &k, uint64_t &i) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) cx(k, i, j, (lane & j) == 0);
    }
    // batch insertion of up to 32 candidates (sentinels elsewhere): the 64 smallest of
    // list(a,b) + C are a + the 32 smallest of b + C (every a <= every b)
    __device__ void batch(double ck, uint64_t ci) {
        const int lane = threadIdx.x & 31;
        const unsigned full = 0xffffffffu;
        double ka, kb;
        uint64_t ia, ib;
        load(ka, ia, kb, ib);
        sort32(ck, ci);
        const double rk = __shfl_sync(full, ck, 31 - lane);
        const uint64_t ri = __shfl_sync(full, ci, 31 - lane);
        if (hit_less(rk, ri, kb, ib)) {
            kb = rk;
            ib = ri;
        }
        merge32(kb, ib);
        const double bk = __shfl_sync(full, kb, 31 - lane);
        const uint64_t bi = __shfl_sync(full, ib, 31 - lane);
        if (hit_less(bk, bi, ka, ia)) {   // lower half keeps the min, upper half the max
            kb = ka;
            ib = ia;
            ka = bk;
            ia = bi;
        } else {
            kb = bk;
            ib = bi;
        }
        merge32(ka, ia);
        merge32(kb, ib);
        store(ka, ia, kb, ib);
        const int src = (k - 1) & 31;
        const double tka = __shfl_sync(full, ka, src), tkb = __shfl_sync(full, kb, src);
        const uint64_t tia = __shfl_sync(full, ia, src), tib = __shfl_sync(full, ib, src);
        if (k - 1 < 32) {
            thk = tka;
            thi = tia;
        } else {
            thk = tkb;
            thi = tib;
        }
        publish();
    }
    // whole warp; per-lane candidate (valid, key, idx).  The insertion code is large, so it
    // lives in one out-of-line function (state passed by value) instead of being inlined at
    // every call site: short-lived launches are otherwise instruction-cache bound.
    __device__ __forceinline__ void offer(bool valid, double key, uint64_t idx);
    // inline variant for call sites that are few (lane-blocked inner loops)
    __device__ __forceinline__ void offer_inl(bool valid, double key, uint64_t idx) {
        const bool cand = valid && key <= adm && key <= thk && (key < thk || idx < thi);
        const unsigned msk = __ballot_sync(0xffffffffu, cand);
        if (msk) offer_slow(cand, msk, key, idx);
    }
    __device__ __forceinline__ void offer_slow(bool cand, unsigned msk, double key, uint64_t idx) {
        const unsigned full = 0xffffffffu;
        if (__popc(msk) >= 6) {
            batch(cand ? key : CUDART_INF, cand ? idx : ~0ull);
            return;
        }
        while (msk) {
            const int src = __ffs(msk) - 1;
            msk &= msk - 1;
            double kk = __shfl_sync(full, key, src);
            uint64_t ii = __shfl_sync(full, idx, src);
            if (hit_less(kk, ii, thk, thi)) insert(kk, ii);
        }
    }
};

__device__ __noinline__ WarpTopK topk_offer_slow(WarpTopK t, bool cand, unsigned msk, double key, uint64_t idx) {
    t.offer_slow(cand, msk, key, idx);
    return t;
}

__device__ __forceinline__ void WarpTopK::offer(bool valid, double key, uint64_t idx) {
    const bool cand = valid && key <= adm && key <= thk && (key < thk || idx < thi);
    const unsigned msk = __ballot_sync(0xffffffffu, cand);
    if (msk) *this = topk_offer_slow(*this, cand, msk, key, idx);
}

// ------------------------------------------------------------------ beta-slot run (reduce mode)
// Evaluates `run` consecutive lane steps inside one alpha/beta block when n_beta = 32*M:
// lane step r visits beta = base + 32*slot, slot cycling 0..M-1, alpha advancing after
// slot M-1.  idx0 = global index of the lane's first configuration of the run.  On exit
// (alpha_i, beta_i) is the lane's last evaluated configuration.
template <int FAM, int M, int NTC = 0>
__device__ __forceinline__ void run_slots(const Mid &m, WarpTopK &tk, const double *alpha_tab, const double *beta_tab,
                                          int NT_, uint32_t &alpha_i, uint32_t &beta_i, uint32_t run, uint64_t idx0) {
    // NTC > 0: the tier count is a compile-time constant (alpha rows at immediate offsets)
    const int NT = NTC > 0 ? NTC : NT_;
    const unsigned full = 0xffffffffu;
    const uint32_t base = beta_i & 31u;
    SlotV sv[M];
#pragma unroll
    for (int i = 0; i < M; i++) slot_vals<FAM>(m, beta_tab + (size_t)(base + 32u * i) * NT, sv[i]);
    uint32_t slot = beta_i >> 5;
    uint32_t r = 0;
    uint32_t a = alpha_i;
    uint32_t last_a = a, last_slot = slot;
    // phase: finish a partially visited alpha row (M == 2, starting at slot 1)
    if (M == 2 && slot == 1) {
        AlphaV av;
        alpha_vals<FAM>(m, alpha_tab + (size_t)a * NT, av);
        const double key = dmul(combine<FAM>(m, av, sv[M - 1]), m.I);
        if (__any_sync(full, key <= tk.adm)) tk.offer(true, key, idx0);
        last_a = a;
        last_slot = 1;
        r = 1;
        a++;
    }
    // R = KEYS/M whole alpha rows per iteration: KEYS independent dependency chains (16 for
    // the light families, 8 where more comm terms would spill); the admission test is one
    // ballot per key (no min/select sequence)
    constexpr int KEYS = FAM == PARADL_PIPELINE                                ? PARADL_PIPE_KEYS
                         : (FAM == PARADL_DATA || FAM == PARADL_LAYERPURE) ? 16
                         : (FAM == PARADL_SPATIAL || FAM == PARADL_DS || FAM == PARADL_DF ||
                            FAM == PARADL_SPATIAL_AG || FAM == PARADL_LAYERWISE)                  ? 4
                                                                                                  : 8;
    constexpr int R = KEYS / M;
    const double *ap = alpha_tab + (size_t)a * NT;
    while (r + R * M <= run) {
        double key[R * M];
#pragma unroll
        for (int q = 0; q < R; q++) {
            AlphaV av;
            alpha_vals<FAM>(m, ap + q * NT, av);
#pragma unroll
            for (int i = 0; i < M; i++) key[q * M + i] = dmul(combine<FAM>(m, av, sv[i]), m.I);
        }
        // admission screen on the high words (integer min; key <= adm implies hi(key) <=
        // hi(adm) for non-negative doubles), one vote per R*M keys; offer() is exact
        int hk = __double2hiint(key[0]);
#pragma unroll
        for (int i = 1; i < R * M; i++) hk = min(hk, __double2hiint(key[i]));
        if (__any_sync(full, hk <= __double2hiint(tk.adm))) {
#pragma unroll
            for (int i = 0; i < R * M; i++) tk.offer(true, key[i], idx0 + 32ull * (r + i));
        }
        last_a = a + R - 1;
        last_slot = M - 1;
        r += R * M;
        a += R;
        ap += R * NT;
    }
    // remaining whole alpha rows
    while (r + M <= run) {
        AlphaV av;
        alpha_vals<FAM>(m, alpha_tab + (size_t)a * NT, av);
        double key[M];
        unsigned b = 0;
#pragma unroll
        for (int i = 0; i < M; i++) {
            key[i] = dmul(combine<FAM>(m, av, sv[i]), m.I);
            b |= __ballot_sync(full, key[i] <= tk.adm);
        }
        if (b) {
#pragma unroll
            for (int i = 0; i < M; i++) tk.offer(true, key[i], idx0 + 32ull * (r + i));
        }
        last_a = a;
        last_slot = M - 1;
        r += M;
        a++;
    }
    // tail (M == 2 only): slot 0 of one more row
    if (r < run) {
        AlphaV av;
        alpha_vals<FAM>(m, alpha_tab + (size_t)a * NT, av);
        const double key = dmul(combine<FAM>(m, av, sv[0]), m.I);
        if (__any_sync(full, key <= tk.adm)) tk.offer(true, key, idx0 + 32ull * r);
        last_a = a;
        last_slot = 0;
    }
    alpha_i = last_a;
    beta_i = base + 32u * last_slot;
}

// ------------------------------------------------------------------ the sweep kernel
// Block-wide ascending bitonic sort of n (power of two) hits by (key, idx) in shared memory.
__device__ void bitonic_sort_smem(paradl_hit *x, int n) {
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const paradl_hit p = x[i], q = x[ixj];
                    const bool up = (i & k) == 0;
                    const bool gt = hit_less(q.key_epoch_s, q.idx, p.key_epoch_s, p.idx);
                    if (gt == up) {
                        x[i] = q;
                        x[ixj] = p;
                    }
                }
            }
            __syncthreads();
        }
    }
}

struct __align__(16) SmemExtra {
    uint16_t cuts[kMaxCuts][kThreads];
    paradl_hit lists[kWarps][PARADL_MAX_TOPK];
    int8_t tier_by_n[PARADL_MAX_STAGES + 8];   // tier_of(n), n <= 64 (mask stage counts)
};

// Structure terms of the lane's current structure from the pipeline structure table: the
// structure index is the mixed-radix value of the digits slower than alpha.
__device__ __forceinline__ uint64_t struct_index(const View &v, const Lane &L) {
    const SubHdr *S = v.S;
    uint64_t s = L.d[D_CAP];
    s = s * S->radix[D_FLOPS] + L.d[D_FLOPS];
    s = s * S->radix[D_B] + L.d[D_B];
    s = s * S->part_n + L.part;
    s = s * S->radix[D_S] + L.d[D_S];
    s = s * S->radix[D_DIMS] + L.d[D_DIMS];
    s = s * S->radix[D_LS] + L.d[D_LS];
    return s;
}
__device__ __forceinline__ void load_rec(const WorkItem &w, uint64_t s, Mid &m) {
    PCHECK(s >= w.stab_lo);
    const PipeRec *r = w.stab + (s - w.stab_lo);
    const double4 q = *reinterpret_cast<const double4 *>(r);
    const int2 t = *reinterpret_cast<const int2 *>(&r->reason);
    m.comp = q.x;
    m.pp_c = q.y;
    m.pp_s = q.z;
    m.I = q.w;
    m.reason = (uint32_t)t.x;
    m.pp_t = t.y;
}

// One tile (32*steps consecutive configurations of work item w) for the whole warp.
// DENSE: 0 reduce (top-k / count), 1 dense writes, 2 compact writes (paradl_sweep_compact)
template <int FAM, int DENSE>
__device__ __forceinline__ void tile_body(const LaunchArgs &a, const WorkItem &w, uint64_t tile, uint8_t *smem,
                                          uint16_t *cuts, WarpTopK &tk, unsigned long long &cnt, double *dtab,
                                          const double *memo) {
    const View v = make_view(smem, w.sub);
    const int lane = threadIdx.x & 31;
    const int cs = kThreads;
    const int NT = v.H->n_tiers;
    const double *alpha_tab = at<double>(v.img, v.S->off_alpha);
    const double *beta_tab = at<double>(v.img, v.S->off_beta);
    const uint64_t gbase = v.S->offset;   // global index of local index 0
    const uint64_t TS = 32ull * w.steps;
    constexpr bool PIPE = FAM == PARADL_PIPELINE || FAM == PARADL_LAYERPURE || FAM == PARADL_PD || FAM == PARADL_GPIPE;
    constexpr bool GP = FAM == PARADL_GPIPE;
    constexpr bool REC = FAM == PARADL_PIPELINE && !DENSE;
    const uint32_t nB = v.S->radix[D_BETA];
    const uint32_t nA = v.S->radix[D_ALPHA];
    const uint32_t nAB = nA * nB;                       // host guarantees < 2^31
    const uint32_t dB = 32u % nB, dA = 32u / nB;        // lane stride 32 inside the alpha/beta block
    // beta-slot caching (M = nB / 32) needs every lane of a step in the same 32-aligned beta
    // window, i.e. a 32-aligned range start (tile starts are lo + multiples of 32)
    constexpr bool LW = FAM == PARADL_DATA_LW;
    const bool slots = !GP && !LW && (nB == 32u || nB == 64u) && (w.lo & 31u) == 0;
    const bool M2 = nB == 64u;
    const unsigned full = 0xffffffffu;
        const uint64_t u0 = w.lo + tile * TS;
        const uint64_t uend = (u0 + TS < w.hi) ? u0 + TS : w.hi;
        const uint32_t len = (uint32_t)(uend - u0);       // <= 32 * steps
        const uint32_t nsteps = (len + 31) >> 5;
        const uint32_t nfull = len >> 5;                  // steps with all 32 lanes active
        const uint64_t g0 = gbase + u0;                   // global index of the tile's first config

        Lane L;
        StageT st;
        Mid m;
        m.reset_memo();
        if (GP) {
            m.gp = dtab + threadIdx.x;
            m.gps = kThreads;
        }
        const double *lw_base = LW ? memo + w.memo_off / sizeof(double) : nullptr;
        if (LW) {
            m.lwt = lw_base;
            m.lwn = (int)(w.memo_n / (2u * v.S->radix[D_DIMS]));
        }
        // pipeline reduce tiles read the structure terms from the structure table
        const bool rec = REC && w.stab != nullptr;
        uint64_t sidx = 0;   // rec: the lane's structure index
        if ((uint32_t)lane < len) {
            decode(v, u0 + lane, L, cuts, cs);
            if (rec) {
                sidx = struct_index(v, L);
                load_rec(w, sidx, m);
            } else {
                if (PIPE) stage_terms(v, L, cuts, cs, at<int64_t>(v.img, v.S->off_b)[L.d[D_B]], st);
                if (LW) m.lwt = lw_base;
                compute_mid<FAM>(v, L, st, m, w.halo);
                if (GP) gpipe_fill(v, L, cuts, cs, m);
                fastify(m);
            }
        } else {
            L.d[D_ALPHA] = L.d[D_BETA] = 0;
            m.reason = PARADL_R_SCALING;
        }
        uint32_t alpha_i = L.d[D_ALPHA], beta_i = L.d[D_BETA];
        uint32_t carry = 0;
        bool have_carry = false;
        // compact mode: pass 1 counts the tile's feasible configurations, pass 2 writes them
        // from the tile's scanned offset (warp ballot + popc of the lanes below)
        uint32_t c_tile = 0;
        uint64_t c_pos = (DENSE == 2 && a.c_off) ? a.c_off[w.tile_base + tile] : 0;
        PCHECK(w.tile_base + tile < a.total_tiles);

        // emits one step (step index jj within the tile) for every lane
        auto emit_dense = [&](bool act, double t_it, bool feas, uint32_t jj) {
            if (DENSE == 2 && a.c_cnt) {
                c_tile += __popc(__ballot_sync(full, act && feas));
                return;
            }
            if (DENSE == 2) {
                const unsigned bb = __ballot_sync(full, act && feas);
                const uint64_t pos = c_pos + __popc(bb & ((1u << lane) - 1u));
                if (act && feas && pos < a.c_cap) {
                    a.c_idx[pos] = g0 + lane + 32ull * jj;
                    if (a.t_iter) a.t_iter[pos] = t_it;
                    if (a.mem) a.mem[pos] = m.mem;
                }
                c_pos += __popc(bb);
                return;
            }
            const uint64_t o = g0 + lane + 32ull * jj - a.first;
            if (act) {
                if (a.t_iter) a.t_iter[o] = t_it;
                if (a.mem) a.mem[o] = m.mem;
                if (a.reason) a.reason[o] = (uint8_t)m.reason;
            }
            if (a.bits) {
                const unsigned bits = __ballot_sync(full, act && feas);
                if (lane == 0) {
                    const uint64_t pos0 = g0 + 32ull * jj - a.first;   // bit position of lane 0
                    const uint32_t sh = (uint32_t)(pos0 & 31);
                    const uint64_t w = pos0 >> 5;
                    const uint32_t lo = bits << sh;
                    const uint32_t hi = sh ? (bits >> (32 - sh)) : 0u;
                    const uint32_t word = lo | (have_carry ? carry : 0u);
                    const uint64_t wg0 = a.first + (w << 5);
                    const bool excl = have_carry || sh == 0;
                    const bool inside = wg0 >= g0 && wg0 + 32 <= gbase + uend;
                    if (excl && inside) a.bits[w] = word;
                    else if (word) atomicOr(&a.bits[w], word);
                    carry = hi;
                    have_carry = sh != 0;
                }
            }
        };

        uint32_t j = 0;
        while (j < nsteps) {
            if (j >= nfull) {
                // ragged last step of the range: generic evaluation with an activity mask
                const bool act = (uint32_t)lane + 32u * j < len;
                const double *arow = alpha_tab + (size_t)alpha_i * NT;
                const double *brow = beta_tab + (size_t)beta_i * NT;
                const bool feas = act && m.reason == 0;
                if (DENSE) {
                    const double t_it = (act && !(m.reason & PARADL_R_TIER)) ? inner_fast<FAM>(m, arow, brow) : CUDART_INF;
                    emit_dense(act, t_it, feas, j);
                } else {
                    const double key = feas ? dmul(inner_fast<FAM>(m, arow, brow), m.I) : CUDART_INF;
                    cnt += feas ? 1u : 0u;
                    tk.offer(feas, key, g0 + lane + 32ull * j);
                }
                j++;
                break;
            }
            // a run: consecutive steps in which no lane leaves its alpha/beta block
            const uint32_t ab = alpha_i * nB + beta_i;
            uint32_t run = __reduce_min_sync(full, (nAB - ab + 31u) >> 5);
            run = min(run, nfull - j);
            const bool feas = m.reason == 0;
            if (!DENSE) {
                tk.refresh();
                const unsigned fb = __ballot_sync(full, feas);
                if (fb == 0u) {
                    if (run > 1) {   // no feasible lane: skip the run, closed-form advance
                        const uint32_t nab = ab + 32u * (run - 1);
                        alpha_i = nab / nB;
                        beta_i = nab - alpha_i * nB;
                    }
                } else if (fb == full && slots) {
                    // every lane feasible and n_beta = 32*M: lane's beta values are fixed, so the
                    // s*beta products are formed once per run and reused for every alpha row
                    if constexpr (!GP && !LW) {
                        if (M2 && NT == 2)
                            run_slots<FAM, 2, 2>(m, tk, alpha_tab, beta_tab, NT, alpha_i, beta_i, run, g0 + lane + 32ull * j);
                        else if (M2)
                            run_slots<FAM, 2>(m, tk, alpha_tab, beta_tab, NT, alpha_i, beta_i, run, g0 + lane + 32ull * j);
                        else if (NT == 2)
                            run_slots<FAM, 1, 2>(m, tk, alpha_tab, beta_tab, NT, alpha_i, beta_i, run, g0 + lane + 32ull * j);
                        else
                            run_slots<FAM, 1>(m, tk, alpha_tab, beta_tab, NT, alpha_i, beta_i, run, g0 + lane + 32ull * j);
                    }
                } else if ((GP || LW) && fb == full) {
                    // GPipe schedule / per-layer folds: Q (alpha, beta) configurations per call,
                    // interleaved dependency chains
                    const int ts = m.pp_t;
                    constexpr uint32_t Q = LW ? kLwQuad : kGpQuad;
                    uint32_t r = 0;
                    for (; r + Q <= run; r += Q) {
                        double av[Q], bv[Q], kv[Q];
#pragma unroll
                        for (uint32_t c = 0; c < Q; c++) {
                            av[c] = alpha_tab[(size_t)alpha_i * NT + ts];
                            bv[c] = beta_tab[(size_t)beta_i * NT + ts];
                            beta_i += dB;
                            alpha_i += dA;
                            if (beta_i >= nB) {
                                beta_i -= nB;
                                alpha_i++;
                            }
                        }
                        if constexpr (LW) {
                            lw_ge_n<(int)Q>(m.lwt, m.lwn, av, bv, kv);
#pragma unroll
                            for (uint32_t c = 0; c < Q; c++) kv[c] = dadd(m.comp, kv[c]);
                        } else {
                            gpipe_eval<Q>(m.gp, m.gps, m.gns, m.gS, av, bv, kv);
                        }
                        bool any = false;
#pragma unroll
                        for (uint32_t c = 0; c < Q; c++) {
                            kv[c] = dmul(kv[c], m.I);
                            any |= kv[c] <= tk.adm;
                        }
                        if (__any_sync(full, any)) {
#pragma unroll
                            for (uint32_t c = 0; c < Q; c++) tk.offer(true, kv[c], g0 + lane + 32ull * (j + r + c));
                        }
                    }
#pragma unroll 1
                    for (; r < run; r++) {
                        const double key = dmul(inner_fast<FAM>(m, alpha_tab + (size_t)alpha_i * NT,
                                                                beta_tab + (size_t)beta_i * NT),
                                                m.I);
                        if (__any_sync(full, key <= tk.adm)) tk.offer(true, key, g0 + lane + 32ull * (j + r));
                        beta_i += dB;
                        alpha_i += dA;
                        if (beta_i >= nB) {
                            beta_i -= nB;
                            alpha_i++;
                        }
                    }
                    {
                        const uint32_t nab = ab + 32u * (run - 1);
                        alpha_i = nab / nB;
                        beta_i = nab - alpha_i * nB;
                    }
                } else if (fb == full) {
                    // every lane feasible: branch-free evaluation, rare slow path for insertions
#pragma unroll 2
                    for (uint32_t r = 0; r < run; r++) {
                        const double key = dmul(inner_fast<FAM>(m, alpha_tab + (size_t)alpha_i * NT,
                                                                beta_tab + (size_t)beta_i * NT),
                                                m.I);
                        if (__any_sync(full, key <= tk.adm)) tk.offer(true, key, g0 + lane + 32ull * (j + r));
                        beta_i += dB;
                        alpha_i += dA;
                        if (beta_i >= nB) {
                            beta_i -= nB;
                            alpha_i++;
                        }
                    }
                    // undo the advance after the run's last step (the generic odometer takes it)
                    {
                        const uint32_t nab = ab + 32u * (run - 1);
                        alpha_i = nab / nB;
                        beta_i = nab - alpha_i * nB;
                    }
                } else {
                    for (uint32_t r = 0; r < run; r++) {
                        double key = CUDART_INF;
                        if (feas)
                            key = dmul(inner_fast<FAM>(m, alpha_tab + (size_t)alpha_i * NT,
                                                       beta_tab + (size_t)beta_i * NT),
                                       m.I);
                        if (__any_sync(full, feas && key <= tk.adm)) tk.offer(feas, key, g0 + lane + 32ull * (j + r));
                        if (r + 1 < run) {
                            beta_i += dB;
                            alpha_i += dA;
                            if (beta_i >= nB) {
                                beta_i -= nB;
                                alpha_i++;
                            }
                        }
                    }
                }
                cnt += feas ? run : 0u;
            } else {
                const bool tier_ok = !(m.reason & PARADL_R_TIER);
                for (uint32_t r = 0; r < run; r++) {
                    const double t_it = tier_ok ? inner_fast<FAM>(m, alpha_tab + (size_t)alpha_i * NT,
                                                                  beta_tab + (size_t)beta_i * NT)
                                                : CUDART_INF;
                    emit_dense(true, t_it, feas, j + r);
                    if (r + 1 < run) {
                        beta_i += dB;
                        alpha_i += dA;
                        if (beta_i >= nB) {
                            beta_i -= nB;
                            alpha_i++;
                        }
                    }
                }
            }
            j += run;
            if (rec && nAB >= 32u && j < nsteps && (uint32_t)lane + 32u * j < len) {
                // step into the next configuration (32 ahead): with a block of >= 32 the lane
                // crosses at most one structure, the next record in the table
                beta_i += dB;
                alpha_i += dA;
                if (beta_i >= nB) {
                    beta_i -= nB;
                    alpha_i++;
                }
                if (alpha_i >= nA) {
                    alpha_i -= nA;
                    sidx++;
                    load_rec(w, sidx, m);
                }
            } else if (j < nsteps && (uint32_t)lane + 32u * j < len) {
                // step into the next configuration: generic odometer (may leave the block)
                L.d[D_ALPHA] = alpha_i;
                L.d[D_BETA] = beta_i;
                const int lvl = advance(w, v, L, cuts, cs);
                if (lvl >= D_LS) {
                    if (rec) {
                        sidx = struct_index(v, L);
                        load_rec(w, sidx, m);
                    } else {
                        if (PIPE && lvl >= D_PART)
                            stage_terms(v, L, cuts, cs, at<int64_t>(v.img, v.S->off_b)[L.d[D_B]], st);
                        if (LW) m.lwt = lw_base;
                        compute_mid<FAM>(v, L, st, m, w.halo);
                        if (GP) gpipe_fill(v, L, cuts, cs, m);
                        fastify(m);
                    }
                }
                alpha_i = L.d[D_ALPHA];
                beta_i = L.d[D_BETA];
            }
        }
        if (DENSE && a.bits && lane == 0 && have_carry && carry) {
            const uint64_t pos_end = g0 + 32ull * nsteps - a.first;
            atomicOr(&a.bits[pos_end >> 5], carry);
        }
        if (DENSE == 2 && a.c_cnt && lane == 0) a.c_cnt[w.tile_base + tile] = c_tile;
    
}

// ------------------------------------------------------------------ lane-blocked tiles (pipeline families)
// For sub-sweeps whose alpha/beta block is small (e.g. cfg5: 2x2) a lane owns whole
// partitions, each with its inner S x dims x Ls x alpha x beta block.  Terms are hoisted
// per partition (stage sums), per dims value (p, tiers, GE) and per S (comp, P2P); the
// fp64 trees are those of compute_mid / inner_fast, so results are bit-identical.
// memo = the work item's smem table [n_b][n_S + n_dims]: b/S and D/(b*dims0).
struct BlkCtx {
    View v;
    const double *alpha_tab, *beta_tab, *memo;
    const int32_t *Sv, *dmv;
    uint32_t nB, nA, nL, nD, nS, nLAB;
    uint64_t Q;
    double R_memo, tau;
    double mW_tab;   // screened pd: mW the lane's ge_s table holds (NaN: none)
};

__device__ __forceinline__ BlkCtx make_blk(const WorkItem &w, uint8_t *smem, const double *memo) {
    BlkCtx C;
    C.v = make_view(smem, w.sub);
    const SubHdr *S = C.v.S;
    C.alpha_tab = at<double>(C.v.img, S->off_alpha);
    C.beta_tab = at<double>(C.v.img, S->off_beta);
    C.Sv = at<int32_t>(C.v.img, S->off_S);
    C.dmv = at<int32_t>(C.v.img, S->off_dims);
    C.memo = memo + w.memo_off / sizeof(double);
    C.nB = S->radix[D_BETA];
    C.nA = S->radix[D_ALPHA];
    C.nL = S->radix[D_LS];
    C.nD = S->radix[D_DIMS];
    C.nS = S->radix[D_S];
    C.nLAB = C.nL * C.nA * C.nB;
    C.Q = (uint64_t)C.nS * C.nD * C.nLAB;
    C.R_memo = -1.0;
    C.tau = 0.0;
    C.mW_tab = CUDART_NAN;
    return C;
}

// Evaluates one partition (stage terms st, ns stages) and its inner block for the lane;
// gblk = global index of the block's first configuration.  Whole warp (act per lane).
template <int FAM, bool COUNT = true>
__device__ __forceinline__ void eval_partition(BlkCtx &C, bool act, const Lane &L, const StageT &st, int64_t ns,
                                               uint64_t gblk, WarpTopK &tk, unsigned long long &cnt) {
    const View &v = C.v;
    const SubHdr *S = v.S;
    const ImgHdr *H = v.H;
    const ModelHdr *M = v.M;
    const unsigned full = 0xffffffffu;
    const int NT = H->n_tiers;
    const int64_t delta = H->delta;
    int64_t b = 1;
    double FBs = 0.0, Utau = 0.0, dmaxY = 0.0, mW = 0.0, comp_lp = 0.0, lp_na = 0.0, lp_s = 0.0;
    uint32_t rp = PARADL_R_SCALING;   // partition-level reason (inactive lanes: infeasible)
    int ts = 0;
    const double *mrow = C.memo;
    if (act) {
        b = at<int64_t>(v.img, S->off_b)[L.d[D_B]];
        const double cap = at<double>(v.img, S->off_cap)[L.d[D_CAP]];
        const double R = at<double>(v.img, S->off_flops)[L.d[D_FLOPS]];
        if (R != C.R_memo) {
            C.R_memo = R;
            C.tau = ddiv(1.0, R);
        }
        rp = 0;
        ts = tier_of(H, ns);
        rp |= flag_tier(ts);
        ts = max(ts, 0) + H->p2p_off;   // point-to-point column (Q40)
        const double memv = dmul(H->gamma, dmul(i2d(delta), i2d(st.memI)));
        if (!(memv <= cap)) rp |= PARADL_R_MEMORY;
        if (FAM == PARADL_LAYERPURE) {
            comp_lp = comp_term(b * M->FB, M->WU, 1, 1, C.tau);
            lp_na = ns > 1 ? i2d(ns - 1) : 0.0;
            lp_s = ns > 1 ? i2d(delta * b * st.sumY) : 0.0;
        } else {
            FBs = i2d(st.maxF + st.maxB);
            Utau = dmul(i2d(st.maxU), C.tau);
            dmaxY = i2d(delta * st.maxY);
            if (FAM == PARADL_PD) mW = i2d(delta * st.maxW);
        }
        mrow = C.memo + (size_t)L.d[D_B] * (C.nS + C.nD);
    }
    const double tau = C.tau;
    for (uint32_t iD = 0; iD < C.nD; iD++) {
        // per dims value: p = s*p_d, tiers, GE
        const int64_t pd = FAM == PARADL_PD ? C.dmv[4 * iD] : 1;
        const double I = mrow[C.nS + iD];
        uint32_t rd = rp;
        double ge_c = 0.0, ge_s = 0.0;
        int ge_t = 0;
        const double ge_phi = ns > 1 ? H->phi_pd : 1.0;   // concurrent stage Allreduces (Q40)
        if (FAM == PARADL_PD && act) {
            const int tp = tier_of(H, ns * pd);
            rd |= flag_tier(tp);
            const ARt g = make_ar(H, pd, mW, ddiv(mW, i2d(pd)), tp);
            if (g.on) {
                ge_c = g.c;
                ge_s = g.s;
            }
            ge_t = max(tp, 0);
        }
        for (uint32_t iS = 0; iS < C.nS; iS++) {
            const int64_t Sg = C.Sv[iS];
            uint32_t r = rd;
            if (Sg < 1 || Sg > b) r |= PARADL_R_SEGMENTS;
            double comp = comp_lp, pp_c = 0.0, pp_s = 0.0;
            if (FAM != PARADL_LAYERPURE && act) {
                const double bS = mrow[iS];
                const double cseg = dmul(i2d(ns + Sg - 1), bS);
                comp = dadd(dmul(dmul(cseg, FBs), tau), Utau);
                if (ns > 1) {
                    pp_c = i2d(2 * (ns + Sg - 2));
                    pp_s = dmul(bS, dmaxY);
                }
            }
            const bool feas = act && r == 0;
            if (COUNT) cnt += feas ? C.nLAB : 0u;
            if (__ballot_sync(full, feas) == 0u) continue;
            const uint64_t base = gblk + (uint64_t)(iS * C.nD + iD) * C.nLAB;
            for (uint32_t iL = 0; iL < C.nL; iL++)
                for (uint32_t ia = 0; ia < C.nA; ia++) {
                    const double *arow = C.alpha_tab + (size_t)ia * NT;
                    const double aval_pp = FAM == PARADL_LAYERPURE ? dmul(lp_na, arow[ts]) : arow[ts];
                    for (uint32_t ib = 0; ib < C.nB; ib++) {
                        const double *brow = C.beta_tab + (size_t)ib * NT;
                        double t = comp;
                        if (FAM == PARADL_PD)
                            t = dadd(t, dmul(ge_c, dadd(arow[ge_t], dmul(ge_s, dmul(brow[ge_t], ge_phi)))));
                        if (FAM == PARADL_LAYERPURE)
                            t = dadd(t, dmul(2.0, dadd(aval_pp, dmul(lp_s, brow[ts]))));
                        else
                            t = dadd(t, dmul(pp_c, dadd(aval_pp, dmul(pp_s, brow[ts]))));
                        const double key = feas ? dmul(t, I) : CUDART_INF;
                        if (__any_sync(full, key <= tk.adm))
                            tk.offer_inl(feas, key, base + (uint64_t)(iL * C.nA + ia) * C.nB + ib);
                    }
                }
        }
    }
}

// Screened evaluation of one partition's inner block (pipeline / pd, mode 1).  The keys
// are the trees of eval_partition, with every term hoisted to the loop level it depends
// on: per S value comp, pp_c, pp_s (4 S values per pass, in registers); per (alpha, beta)
// row the pipeline term P = pp_c (alpha + pp_s beta); per dims value (innermost, from the
// lane's smem table built once per partition) the GE term G = ge_c (alpha + ge_s beta).
// Per configuration t = comp + G, t = t + P, key = t * I remain.  No top-k work is done
// here: the block's smallest high word of the key bits is compared with the admission
// bound once (for non-negative doubles key <= adm implies hi(key) <= hi(adm), so the
// screen never drops a candidate), and a partition that passes is re-evaluated by
// eval_partition, which offers its configurations one by one.  Infeasible terms are set
// to +inf (key +inf, never below a finite bound); the feasible count is separable:
// (#S with 1 <= S <= b) x (#dims in a tier) x n_LAB.
// dtab: per-lane table [nD][kThreads] of ge_s; ge_c and ge_t come from the per-CTA ring
// table by (stage count, dims value) built with the memo (pd, ring only: tree_thr = 0).
// ge_s = mW / p_d: x / 2^k is exact (x = 0 or x >= 1: no underflow), so for power-of-two
// p_d the division equals the multiplication by the scale 2^-k (ring table row 0) bit for bit.
constexpr int kSB = 4;   // S values per pass
template <int FAM>
__device__ __forceinline__ void eval_partition_screened(BlkCtx &C, bool act, const Lane &L, const StageT &st,
                                                        int64_t ns, uint64_t gblk, WarpTopK &tk,
                                                        unsigned long long &cnt, double *dtab) {
    const View &v = C.v;
    const SubHdr *S = v.S;
    const ImgHdr *H = v.H;
    const unsigned full = 0xffffffffu;
    const int NT = H->n_tiers;
    const int64_t delta = H->delta;
    const double INF = CUDART_INF;
    double *gs_tab = dtab + threadIdx.x;
    const uint32_t nDp = C.nD + 1;
    const double *gc_row = C.memo + (size_t)S->radix[D_B] * (C.nS + C.nD);
    const int32_t *gt_row = reinterpret_cast<const int32_t *>(
        gc_row + (size_t)((S->part_mode == PARADL_PART_COMB ? S->s_max : S->G) + 1) * nDp);
    int64_t b = 1;
    double FBs = 0.0, Utau = 0.0, dmaxY = 0.0, part_inf = INF;
    int ts = 0;
    const double *mrow = C.memo;
    uint32_t nSok = 0, nDok = 0;
    if (act) {
        b = at<int64_t>(v.img, S->off_b)[L.d[D_B]];
        const double cap = at<double>(v.img, S->off_cap)[L.d[D_CAP]];
        const double R = at<double>(v.img, S->off_flops)[L.d[D_FLOPS]];
        if (R != C.R_memo) {
            C.R_memo = R;
            C.tau = ddiv(1.0, R);
        }
        const int tsr = tier_of(H, ns);
        ts = max(tsr, 0) + H->p2p_off;   // point-to-point column (Q40)
        const double memv = dmul(H->gamma, dmul(i2d(delta), i2d(st.memI)));
        part_inf = (tsr >= 0 && memv <= cap) ? 0.0 : INF;
        FBs = i2d(st.maxF + st.maxB);
        Utau = dmul(i2d(st.maxU), C.tau);
        dmaxY = i2d(delta * st.maxY);
        mrow = C.memo + (size_t)L.d[D_B] * (C.nS + C.nD);
        if (FAM == PARADL_PD) {
            const double mW = i2d(delta * st.maxW);
            if (mW != C.mW_tab) {   // ge_s = mW / p_d (the lane's table is kept while mW repeats)
                C.mW_tab = mW;
                for (uint32_t iD = 0; iD < C.nD; iD++) {
                    const double sc = gc_row[iD];
                    gs_tab[(size_t)iD * kThreads] = sc != 0.0 ? dmul(mW, sc) : ddiv(mW, i2d(C.dmv[4 * iD]));
                }
            }
            gc_row += (size_t)ns * nDp;
            gt_row += (size_t)ns * nDp;
            nDok = (uint32_t)gt_row[C.nD];
        } else {
            nDok = C.nD;
        }
    }
    const double tau = C.tau;
    int hmin = 0x7fffffff;
    for (uint32_t iS0 = 0; iS0 < C.nS; iS0 += kSB) {
        double comp[kSB], ppc[kSB], pps[kSB];
#pragma unroll
        for (int u = 0; u < kSB; u++) {
            comp[u] = INF;
            ppc[u] = pps[u] = 0.0;
            const uint32_t iS = iS0 + u;
            if (act && iS < C.nS) {
                const int64_t Sg = C.Sv[iS];
                const double bS = mrow[iS];
                const double cseg = dmul(i2d(ns + Sg - 1), bS);
                const bool sok = Sg >= 1 && Sg <= b;
                nSok += sok ? 1u : 0u;
                comp[u] = dadd(dadd(dmul(dmul(cseg, FBs), tau), Utau), sok ? part_inf : INF);
                if (ns > 1) {
                    ppc[u] = i2d(2 * (ns + Sg - 2));
                    pps[u] = dmul(bS, dmaxY);
                }
            }
        }
        for (uint32_t iL = 0; iL < C.nL; iL++)
            for (uint32_t ia = 0; ia < C.nA; ia++) {
                const double *arow = C.alpha_tab + (size_t)ia * NT;
                const double at_ = arow[ts];
                for (uint32_t ib = 0; ib < C.nB; ib++) {
                    const double *brow = C.beta_tab + (size_t)ib * NT;
                    const double bt_ = brow[ts];
                    double P[kSB];
#pragma unroll
                    for (int u = 0; u < kSB; u++) P[u] = dmul(ppc[u], dadd(at_, dmul(pps[u], bt_)));
                    if (FAM == PARADL_PD) {
#pragma unroll 2
                        for (uint32_t iD = 0; iD < C.nD; iD++) {
                            const double I = mrow[C.nS + iD];
                            const int gt = gt_row[iD];
                            const double G =
                                dmul(gc_row[iD], dadd(arow[gt], dmul(gs_tab[(size_t)iD * kThreads],
                                                                     dmul(brow[gt], ns > 1 ? H->phi_pd : 1.0))));
#pragma unroll
                            for (int u = 0; u < kSB; u++)
                                hmin = min(hmin, __double2hiint(dmul(dadd(dadd(comp[u], G), P[u]), I)));
                        }
                    } else {
                        for (uint32_t iD = 0; iD < C.nD; iD++) {
                            const double I = mrow[C.nS + iD];
#pragma unroll
                            for (int u = 0; u < kSB; u++)
                                hmin = min(hmin, __double2hiint(dmul(dadd(comp[u], P[u]), I)));
                        }
                    }
                }
            }
    }
    if (act && part_inf == 0.0) cnt += (unsigned long long)nSok * nDok * C.nLAB;
    const bool maybe = act && hmin <= __double2hiint(tk.adm);
    if (__any_sync(full, maybe)) eval_partition<FAM, false>(C, maybe, L, st, ns, gblk, tk, cnt);
}

// Mode 1: lane l of tile t owns partitions [t*32c + l*c, +c) of the block-aligned range;
// stage terms by prefix differences, successor between partitions.
#ifndef PARADL_INC_STAGES
#define PARADL_INC_STAGES 0
#endif
constexpr bool kIncStages = PARADL_INC_STAGES;
template <int FAM>
__device__ void tile_body_blocked(const LaunchArgs &a, const WorkItem &w, uint64_t tile, uint8_t *smem,
                                  uint16_t *cuts, WarpTopK &tk, unsigned long long &cnt, const double *memo,
                                  double *dtab) {
    BlkCtx C = make_blk(w, smem, memo);
    const int lane = threadIdx.x & 31;
    const uint64_t nblk = (w.hi - w.lo) / C.Q;
    const uint64_t c = w.steps;
    const uint64_t blk0 = (tile * 32 + lane) * c;
    const uint64_t nmine = blk0 < nblk ? min(c, nblk - blk0) : 0;
    const uint32_t iters = __reduce_max_sync(0xffffffffu, (uint32_t)nmine);
    Lane L;
    StageT st, pre;
    // COMB successors mostly move only the last cut: stages 0..ns-3 (ending at cut ns-3)
    // are then unchanged, so their folded terms `pre` are reused and only the last two
    // stages are recomputed (pre_key: ns, b digit and cut ns-3 it was built for)
    const bool comb = kIncStages && C.v.S->part_mode == PARADL_PART_COMB;
    uint64_t pre_key = ~0ull;
    if (nmine) decode(C.v, w.lo + blk0 * C.Q, L, cuts, kThreads);
    for (uint32_t it = 0; it < iters; it++) {
        const bool act = it < nmine;
        int64_t ns = 1;
        if (act) {
            const int64_t b = at<int64_t>(C.v.img, C.v.S->off_b)[L.d[D_B]];
            if (comb) {
                const int k2 = L.ns - 3;   // last stage of the reusable prefix
                const int c2 = k2 >= 0 ? cuts[k2 * kThreads] : 0;
                const uint64_t key = ((uint64_t)L.ns << 48) | ((uint64_t)L.d[D_B] << 16) | (uint64_t)c2;
                if (key != pre_key) {
                    pre_key = key;
                    pre.maxF = pre.maxB = pre.maxU = pre.maxW = pre.maxY = pre.sumY = pre.memI = 0;
                    if (k2 >= 0) stage_span(C.v, cuts, kThreads, 2 * b, L.ns, 0, k2 + 1, 0, pre);
                }
                st = pre;
                stage_span(C.v, cuts, kThreads, 2 * b, L.ns, max(k2 + 1, 0), L.ns, c2, st);
            } else {
                stage_terms(C.v, L, cuts, kThreads, b, st);
            }
            ns = L.ns;
        }
        const uint64_t gblk = C.v.S->offset + w.lo + (blk0 + it) * C.Q;
        if ((FAM == PARADL_PIPELINE || (FAM == PARADL_PD && C.v.H->tree_thr <= 0.0)) && dtab &&
            (size_t)C.nD * 8u * kThreads <= a.dtab_bytes)
            eval_partition_screened<FAM>(C, act, L, st, ns, gblk, tk, cnt, dtab);
        else
            eval_partition<FAM>(C, act, L, st, ns, gblk, tk, cnt);
        tk.refresh();
        if (it + 1 < nmine) advance(w, C.v, L, cuts, kThreads);   // next partition (inc_part = 1)
    }
}

// ------------------------------------------------------------------ mask mode with a low-bit table
// Mode 2 (MASK partitions, G >= 10): lane owns aligned blocks of 256 consecutive masks, so
// bits 8.. are fixed within a block.  Stages whose rows all lie among the first 9 rows
// depend only on the low 8 bits: their maxima come from a per-CTA table over the 256
// patterns.  Stages after the first high cut are evaluated once per block; per mask only
// the stage straddling bit 8 (from the last low cut to the first high cut) is formed.
// All quantities are exact int64 sums / maxima, so the composition equals stage_terms.
constexpr int kLowBits = 8;
constexpr int kLowBitsS = kLowBitsSorted;    // sorted mask path (kWorkMaskS): 512-mask blocks
constexpr int kLowBitsMax = kLowBitsS;
struct LowE {
    int64_t F, B, U, W, memI, maxY, sumY;
    int32_t e_last, pop;
};
static_assert(sizeof(LowE) == 64, "LowE layout");
// the same low-bit table as exact doubles (kWorkMaskD: every stage term < 2^53)
struct __align__(16) LowD {
    double F, B, U, M;
    double Ypp;   // pp_s of the low stages: b/S (delta maxY), monotone in maxY
    int32_t pop, e_last;
    double Y, pad_;
};
// per (b, stage count n) values of the screened mask path
struct __align__(16) NTab {
    double cseg, ppc, aw, bw;
};
// (kWorkMaskS) the low-bit table sorted by (e, pop) -- e = bit length of the low mask x (the row
// after its last low cut), pop = popcount(x) -- with the per-configuration factors folded in:
// Ut = U tau and Yb[t] = Ypp beta_t (P2P column of tier t).  Exact: max(a, b) x c = max(a c, b c)
// and a + max(u, v) = max(a + u, a + v) for round-to-nearest and c > 0 (monotone), so
// max(U, T_U) tau and pp_c (alpha + max(Ypp, hpps) beta) are maxima of precomputed parts.
struct __align__(16) LowS {
    double F, B, Ut, M;
    double Yb[4];
};
static_assert(sizeof(LowS) == 64, "LowS layout");
// start / size of the (e, pop) subgroups in the sorted table: e = 0 holds x = 0; e >= 1 holds
// x in [2^(e-1), 2^e) ordered by pop (1..e), each subgroup C(e-1, pop-1) masks by x ascending
struct SubTab {
    uint16_t start[kLowBitsMax + 1][kLowBitsMax + 2], cnt[kLowBitsMax + 1][kLowBitsMax + 2];
};
constexpr SubTab make_subtab() {
    SubTab t{};
    for (int e = 0; e <= kLowBitsMax; e++) {
        int start = e ? 1 << (e - 1) : 0;
        for (int pop = 0; pop <= kLowBitsMax + 1; pop++) {
            int c = 0;
            if (e == 0) c = pop == 0 ? 1 : 0;
            else if (pop >= 1 && pop <= e) {   // C(e-1, pop-1)
                long long v = 1;
                for (int j = 0; j < pop - 1; j++) v = v * (e - 1 - j) / (j + 1);
                c = (int)v;
            }
            t.start[e][pop] = (uint16_t)start;
            t.cnt[e][pop] = (uint16_t)c;
            start += c;
        }
    }
    return t;
}
__constant__ SubTab kSub = make_subtab();
// sorted position of low mask x
__device__ __forceinline__ int lows_pos(uint32_t x) {
    const int e = x ? 32 - __clz(x) : 0, pop = __popc(x);
    int r = 0;   // rank of x among the masks of its (e, pop) subgroup
    for (uint32_t y = e ? 1u << (e - 1) : 0u; y < x; y++) r += __popc(y) == pop;
    return kSub.start[e][pop] + r;
}
static_assert(sizeof(LowD) == 64, "LowD layout");

// Largest integer m with gamma (delta m) <= cap (Table 2 mem row), -1 if none:
// i2d and multiplication by a positive constant are monotone, so the predicate is a
// down-set in m and the integer compare m <= threshold decides exactly what the fp64
// compare decides (memI < 2^62 by the host's overflow bounds).
__device__ __noinline__ int64_t mem_threshold(const ImgHdr *H, double cap) {
    const double g = H->gamma, d = i2d(H->delta);
    auto ok = [&](int64_t m) { return dmul(g, dmul(d, i2d(m))) <= cap; };
    if (!ok(0)) return -1;
    int64_t lo = 0, hi = int64_t(1) << 62;
    if (ok(hi)) return hi;
    while (hi - lo > 1) {   // ok(lo), !ok(hi)
        const int64_t mid = lo + (hi - lo) / 2;
        if (ok(mid)) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Mode 2, screened (pipeline, one configuration per mask: the cfg3-ii shape; kWorkMaskD).
// Stage terms are exact doubles (host bound < 2^53), so maxima are DMNMX and no int64 ->
// fp64 conversion is left per mask.  Masks are visited grouped by e_last (the row after
// the last low cut: x in [2^(e-1), 2^e) has e_last = e), so the straddling stage
// [e_last, c_h) folded with the high stages is one register set per group.  Per mask only
// the low-table entry is combined and the key formed with the trees of eval_partition
// (FB = maxF + maxB, delta maxY and memI are exact in double, so they equal the int64
// forms converted); memory feasibility is the threshold memI <= mem_max.  Only the
// smallest high word of the block's keys is kept; a block that may hold a candidate is
// re-evaluated mask by mask through eval_partition (offers).
template <int FAM>
__device__ void tile_body_mask_d(const LaunchArgs &a, const WorkItem &w, uint64_t tile, uint8_t *smem,
                                 uint16_t *cuts, WarpTopK &tk, unsigned long long &cnt, const double *memo,
                                 const LowD *lowtab, const int8_t *tier_by_n) {
    BlkCtx C = make_blk(w, smem, memo);
    const View &v = C.v;
    const ModelHdr *M = v.M;
    const ImgHdr *H = v.H;
    const int lane = threadIdx.x & 31;
    const int G = M->G;
    const int64_t *PF = at<int64_t>(v.mb, M->off_pf);
    const int64_t *PB = at<int64_t>(v.mb, M->off_pb);
    const int64_t *PU = at<int64_t>(v.mb, M->off_pu);
    const int64_t *PW = at<int64_t>(v.mb, M->off_pw);
    const int64_t *PX = at<int64_t>(v.mb, M->off_pxy);
    const int64_t *PI = at<int64_t>(v.mb, M->off_pbi);
    const int64_t *Y = at<int64_t>(v.mb, M->off_y);
    const uint64_t span = C.Q << kLowBits;
    const uint64_t nblk = (w.hi - w.lo) / span;
    const uint64_t c = w.steps;
    const uint64_t blk0 = (tile * 32 + lane) * c;
    const uint64_t nmine = blk0 < nblk ? min(c, nblk - blk0) : 0;
    const uint32_t iters = __reduce_max_sync(0xffffffffu, (uint32_t)nmine);
    const int64_t delta = H->delta;
    const double dd = i2d(delta);
    const int64_t Sg = C.Sv[0];
    double cap_memo = CUDART_NAN, mem_max_d = -1.0;
    Lane L;
    if (nmine) decode(v, w.lo + blk0 * span, L, cuts, kThreads);
    for (uint32_t it = 0; it < iters; it++) {
        const bool act = it < nmine;
        const uint64_t hi_mask = L.part & ~(((uint64_t)1 << kLowBits) - 1);
        int64_t hF = 0, hB = 0, hU = 0, hM = 0, hY = 0;
        int c_h = G;
        int hpop = 0;
        int64_t b = 1;
        const LowD *lt = lowtab;
        int hmin = 0x7fffffff;
        uint32_t nok = 0;
        if (act) {
            b = at<int64_t>(v.img, v.S->off_b)[L.d[D_B]];
            lt = lowtab + (size_t)L.d[D_B] * (1 << kLowBits);
            uint64_t m = hi_mask;
            hpop = __popcll(m);
            if (m) {
                c_h = __ffsll((long long)m);
                m &= m - 1;
                int beg = c_h;
                hY = Y[c_h - 1];
                for (;;) {
                    const int end = m ? __ffsll((long long)m) : G;
                    m &= m - 1;
                    hF = max(hF, PF[end] - PF[beg]);
                    hB = max(hB, PB[end] - PB[beg]);
                    hU = max(hU, PU[end] - PU[beg]);
                    hM = max(hM, 2 * b * (PX[end] - PX[beg]) + 2 * (PW[end] - PW[beg]) + (PI[end] - PI[beg]));
                    if (end == G) break;
                    hY = max(hY, Y[end - 1]);
                    beg = end;
                }
            }
            const double cap = at<double>(v.img, v.S->off_cap)[L.d[D_CAP]];
            const double R = at<double>(v.img, v.S->off_flops)[L.d[D_FLOPS]];
            if (R != C.R_memo) {
                C.R_memo = R;
                C.tau = ddiv(1.0, R);
            }
            if (!(cap == cap_memo)) {
                cap_memo = cap;
                mem_max_d = i2d(mem_threshold(H, cap));
            }
            const double tau = C.tau;
            const double *mrow = C.memo + (size_t)L.d[D_B] * (C.nS + C.nD);
            const double bS = mrow[0], I = mrow[C.nS];
            const bool seg_ok = Sg >= 1 && Sg <= b;
            const double hFd = i2d(hF), hBd = i2d(hB), hUd = i2d(hU), hMd = i2d(hM);
            const double hpps = dmul(bS, dmul(dd, i2d(hY)));
            const uint32_t nb = v.S->radix[D_B];
            const NTab *nt = reinterpret_cast<const NTab *>(C.memo + (size_t)nb * (C.nS + C.nD)) +
                             (size_t)L.d[D_B] * kMaskTabN;
            const int64_t cF = PF[c_h], cB = PB[c_h], cU = PU[c_h], cW = PW[c_h], cX = PX[c_h], cI = PI[c_h];
            for (int e = 0; e <= kLowBits; e++) {
                const int x0 = e ? 1 << (e - 1) : 0, x1 = e ? 1 << e : 1;
                const double TF = fmax(i2d(cF - PF[e]), hFd), TB = fmax(i2d(cB - PB[e]), hBd);
                const double TU = fmax(i2d(cU - PU[e]), hUd);
                const double TM = fmax(i2d(2 * b * (cX - PX[e]) + 2 * (cW - PW[e]) + (cI - PI[e])), hMd);
                // memI = max(low, T) <= mem_max  <=>  both are
                const bool grp_ok = seg_ok && TM <= mem_max_d;
#pragma unroll 2
                for (int x = x0; x < x1; x++) {
                    const double2 *qp = reinterpret_cast<const double2 *>(lt + x);
                    const double2 qFB = qp[0], qUM = qp[1], qY = qp[2];
                    // maxima of non-NaN values as compare-select (fmax adds NaN handling); pp_s is
                    // a monotone function of maxY, so it is the max of the two precomputed parts
                    const double maxF = qFB.x > TF ? qFB.x : TF, maxB = qFB.y > TB ? qFB.y : TB;
                    const double maxU = qUM.x > TU ? qUM.x : TU, pps = qY.x > hpps ? qY.x : hpps;
                    const int ns = __double2loint(qY.y) + hpop + 1;   // LowD.pop
                    const NTab tq = nt[ns];
                    const bool feas = grp_ok & (qUM.y <= mem_max_d) & (tier_by_n[ns] >= 0);
                    const double comp = dadd(dmul(dmul(tq.cseg, dadd(maxF, maxB)), tau), dmul(maxU, tau));
                    const double key = dmul(dadd(comp, dmul(tq.ppc, dadd(tq.aw, dmul(pps, tq.bw)))), I);
                    nok += feas ? 1u : 0u;
                    hmin = min(hmin, feas ? __double2hiint(key) : 0x7fffffff);
                }
            }
        }
        cnt += nok;
        const bool maybe = act && hmin <= __double2hiint(tk.adm);
        if (__any_sync(0xffffffffu, maybe)) {
            const uint64_t gbase = v.S->offset + w.lo + (blk0 + it) * span;
            for (uint32_t x = 0; x < (1u << kLowBits); x++) {
                StageT st;
                int64_t ns = 1;
                if (maybe) {
                    const LowD q = lt[x];
                    const int beg = q.e_last;
                    st.maxF = max(max((int64_t)__double2ll_rn(q.F), PF[c_h] - PF[beg]), hF);
                    st.maxB = max(max((int64_t)__double2ll_rn(q.B), PB[c_h] - PB[beg]), hB);
                    st.maxU = max(max((int64_t)__double2ll_rn(q.U), PU[c_h] - PU[beg]), hU);
                    st.maxW = 0;   // pd only
                    st.sumY = 0;   // layer-pure only
                    st.memI = max(max((int64_t)__double2ll_rn(q.M),
                                      2 * b * (PX[c_h] - PX[beg]) + 2 * (PW[c_h] - PW[beg]) + (PI[c_h] - PI[beg])),
                                  hM);
                    st.maxY = max((int64_t)__double2ll_rn(q.Y), hY);
                    ns = q.pop + hpop + 1;
                }
                eval_partition<FAM, false>(C, maybe, L, st, ns, gbase + (uint64_t)x * C.Q, tk, cnt);
            }
        }
        tk.refresh();
        if (it + 1 < nmine) advance(w, v, L, cuts, kThreads);   // next block: inc_part = 256
    }
}

// Mode 2, sorted (kWorkMaskS: pipeline masks, one configuration per mask, one flops value, the
// cfg3-ii shape).  Lanes own blocks of 2^kLowBitsS = 512 masks; the only per-CTA table is the
// (e, pop)-sorted LowS (U tau and Ypp beta_t folded in, §5.1).  Per (e, pop) subgroup the stage
// count, its tier and NTab row and the high part's P2P term are registers; per mask 7 fp64
// operations (t_iter; x I once per block on the smallest t) and 5 compares.  A block whose screen passes (0.2 % of the work in cfg3-ii) forms
// each mask's low stage terms from the prefix sums and re-evaluates it through eval_partition.
template <int FAM>
__device__ void tile_body_mask_s(const LaunchArgs &a, const WorkItem &w, uint64_t tile, uint8_t *smem,
                                 uint16_t *cuts, WarpTopK &tk, unsigned long long &cnt, const double *memo,
                                 const LowS *lows, const int8_t *tier_by_n) {
    constexpr int LB = kLowBitsS;
    BlkCtx C = make_blk(w, smem, memo);
    const View &v = C.v;
    const ModelHdr *M = v.M;
    const ImgHdr *H = v.H;
    const int lane = threadIdx.x & 31;
    const int G = M->G;
    const int64_t *PF = at<int64_t>(v.mb, M->off_pf);
    const int64_t *PB = at<int64_t>(v.mb, M->off_pb);
    const int64_t *PU = at<int64_t>(v.mb, M->off_pu);
    const int64_t *PW = at<int64_t>(v.mb, M->off_pw);
    const int64_t *PX = at<int64_t>(v.mb, M->off_pxy);
    const int64_t *PI = at<int64_t>(v.mb, M->off_pbi);
    const int64_t *Y = at<int64_t>(v.mb, M->off_y);
    const uint64_t span = C.Q << LB;   // Q == 1
    const uint64_t nblk = (w.hi - w.lo) / span;
    const uint64_t c = w.steps;
    const uint64_t blk0 = (tile * 32 + lane) * c;
    const uint64_t nmine = blk0 < nblk ? min(c, nblk - blk0) : 0;
    const uint32_t iters = __reduce_max_sync(0xffffffffu, (uint32_t)nmine);
    const double dd = i2d(H->delta);
    const int64_t Sg = C.Sv[0];
    const uint32_t nb = v.S->radix[D_B];
    double cap_memo = CUDART_NAN, mem_max_d = -1.0;
    Lane L;
    if (nmine) decode(v, w.lo + blk0 * span, L, cuts, kThreads);
    for (uint32_t it = 0; it < iters; it++) {
        const bool act = it < nmine;
        const uint64_t hi_mask = L.part & ~(((uint64_t)1 << LB) - 1);
        int64_t hF = 0, hB = 0, hU = 0, hM = 0, hY = 0;
        int c_h = G;
        int hpop = 0;
        int64_t b = 1;
        int hmin = 0x7fffffff, th = 0x7fffffff;
        uint32_t nok = 0;
        if (act) {
            b = at<int64_t>(v.img, v.S->off_b)[L.d[D_B]];
            uint64_t m = hi_mask;
            hpop = __popcll(m);
            if (m) {   // stages after the first high cut (exact int64)
                c_h = __ffsll((long long)m);
                m &= m - 1;
                int beg = c_h;
                hY = Y[c_h - 1];
                for (;;) {
                    const int end = m ? __ffsll((long long)m) : G;
                    m &= m - 1;
                    hF = max(hF, PF[end] - PF[beg]);
                    hB = max(hB, PB[end] - PB[beg]);
                    hU = max(hU, PU[end] - PU[beg]);
                    hM = max(hM, 2 * b * (PX[end] - PX[beg]) + 2 * (PW[end] - PW[beg]) + (PI[end] - PI[beg]));
                    if (end == G) break;
                    hY = max(hY, Y[end - 1]);
                    beg = end;
                }
            }
            const double cap = at<double>(v.img, v.S->off_cap)[L.d[D_CAP]];
            const double R = at<double>(v.img, v.S->off_flops)[L.d[D_FLOPS]];
            if (R != C.R_memo) {
                C.R_memo = R;
                C.tau = ddiv(1.0, R);
            }
            if (!(cap == cap_memo)) {
                cap_memo = cap;
                mem_max_d = i2d(mem_threshold(H, cap));
            }
            const double tau = C.tau;
            const double *mrow = C.memo + (size_t)L.d[D_B] * (C.nS + C.nD);
            const double bS = mrow[0], I = mrow[C.nS];
            const bool seg_ok = Sg >= 1 && Sg <= b;
            const double hFd = i2d(hF), hBd = i2d(hB), hUd = i2d(hU), hMd = i2d(hM);
            const double hpps = dmul(bS, dmul(dd, i2d(hY)));
            const NTab *nt = reinterpret_cast<const NTab *>(C.memo + (size_t)nb * (C.nS + C.nD)) +
                             (size_t)L.d[D_B] * kMaskTabN;
            const LowS *lsb = lows + ((size_t)L.d[D_B] << LB);
            const uint32_t *fc = reinterpret_cast<const uint32_t *>(lows + ((size_t)nb << LB)) +
                                 (size_t)L.d[D_B] * (LB + 1) * (LB + 2);
            const int64_t cF = PF[c_h], cB = PB[c_h], cU = PU[c_h], cW = PW[c_h], cX = PX[c_h], cI = PI[c_h];
            for (int e = 0; e <= LB; e++) {
                // straddling stage (e, c_h] folded with the high stages
                const double TF = fmax(i2d(cF - PF[e]), hFd), TB = fmax(i2d(cB - PB[e]), hBd);
                const double TUt = dmul(fmax(i2d(cU - PU[e]), hUd), tau);
                const double TM = fmax(i2d(2 * b * (cX - PX[e]) + 2 * (cW - PW[e]) + (cI - PI[e])), hMd);
                const bool grp_ok = seg_ok && TM <= mem_max_d;   // memI = max(low, T) <= mem_max <=> both
                for (int pop = e ? 1 : 0; pop <= e; pop++) {
                    const int ns = pop + hpop + 1;
                    const NTab tq = nt[ns];
                    const int tr = tier_by_n[ns];
                    const bool ok = grp_ok && tr >= 0;
                    const int tt = max(tr, 0);
                    // an infeasible subgroup (memory of the high / straddling part, tier, S > b)
                    // gets P_h = +inf: every key is +inf; memory-infeasible entries carry F = +inf
                    const double Ph = ok ? dmul(tq.ppc, dadd(tq.aw, dmul(hpps, tq.bw))) : CUDART_INF;
                    nok += ok ? fc[e * (LB + 2) + pop] : 0u;
                    const int j0 = kSub.start[e][pop], j1 = j0 + kSub.cnt[e][pop];
#pragma unroll 2
                    for (int j = j0; j < j1; j++) {
                        const double2 *qp = reinterpret_cast<const double2 *>(lsb + j);
                        const double2 qFB = qp[0], qUM = qp[1];
                        const double yb = lsb[j].Yb[tt];
                        const double maxF = qFB.x > TF ? qFB.x : TF, maxB = qFB.y > TB ? qFB.y : TB;
                        const double mUt = qUM.x > TUt ? qUM.x : TUt;
                        const double Pl = dmul(tq.ppc, dadd(tq.aw, yb));
                        const double p2p = Pl > Ph ? Pl : Ph;
                        const double comp = dadd(dmul(dmul(tq.cseg, dadd(maxF, maxB)), tau), mUt);
                        th = min(th, __double2hiint(dadd(comp, p2p)));
                    }
                }
            }
            // key = t I is monotone in t: every key of the block is at least D(t_lo I)
            hmin = __double2hiint(dmul(__hiloint2double(th, 0), I));
        }
        cnt += nok;
        const bool maybe = act && hmin <= __double2hiint(tk.adm);
        if (__any_sync(0xffffffffu, maybe)) {
            const uint64_t gbase = v.S->offset + w.lo + (blk0 + it) * span;
            for (uint32_t x = 0; x < (1u << LB); x++) {
                StageT st;
                int64_t ns = 1;
                if (maybe) {
                    // low stages of mask x (cuts among the first LB + 1 rows), then the straddling
                    // stage (e_last, c_h] and the high maxima: exact int64, = stage_terms
                    int64_t lF = 0, lB = 0, lU = 0, lM = 0, lY = 0;
                    int beg = 0;
                    uint32_t mm = x;
                    while (mm) {
                        const int end = __ffs(mm);
                        mm &= mm - 1;
                        lF = max(lF, PF[end] - PF[beg]);
                        lB = max(lB, PB[end] - PB[beg]);
                        lU = max(lU, PU[end] - PU[beg]);
                        lM = max(lM, 2 * b * (PX[end] - PX[beg]) + 2 * (PW[end] - PW[beg]) + (PI[end] - PI[beg]));
                        lY = max(lY, Y[end - 1]);
                        beg = end;
                    }
                    st.maxF = max(max(lF, PF[c_h] - PF[beg]), hF);
                    st.maxB = max(max(lB, PB[c_h] - PB[beg]), hB);
                    st.maxU = max(max(lU, PU[c_h] - PU[beg]), hU);
                    st.maxW = 0;   // pd only
                    st.sumY = 0;   // layer-pure only
                    st.memI = max(max(lM, 2 * b * (PX[c_h] - PX[beg]) + 2 * (PW[c_h] - PW[beg]) + (PI[c_h] - PI[beg])), hM);
                    st.maxY = max(lY, hY);
                    ns = __popc(x) + hpop + 1;
                }
                eval_partition<FAM, false>(C, maybe, L, st, ns, gbase + (uint64_t)x * C.Q, tk, cnt);
            }
        }
        tk.refresh();
        if (it + 1 < nmine) advance(w, v, L, cuts, kThreads);   // next block: inc_part = 512
    }
}

template <int FAM>
__device__ void tile_body_mask(const LaunchArgs &a, const WorkItem &w, uint64_t tile, uint8_t *smem,
                               uint16_t *cuts, WarpTopK &tk, unsigned long long &cnt, const double *memo,
                               const LowE *lowtab) {
    BlkCtx C = make_blk(w, smem, memo);
    const View &v = C.v;
    const ModelHdr *M = v.M;
    const int lane = threadIdx.x & 31;
    const int G = M->G;
    const int64_t *PF = at<int64_t>(v.mb, M->off_pf);
    const int64_t *PB = at<int64_t>(v.mb, M->off_pb);
    const int64_t *PU = at<int64_t>(v.mb, M->off_pu);
    const int64_t *PW = at<int64_t>(v.mb, M->off_pw);
    const int64_t *PX = at<int64_t>(v.mb, M->off_pxy);
    const int64_t *PI = at<int64_t>(v.mb, M->off_pbi);
    const int64_t *Y = at<int64_t>(v.mb, M->off_y);
    const uint64_t span = C.Q << kLowBits;                 // configs per 256-mask block
    const uint64_t nblk = (w.hi - w.lo) / span;
    const uint64_t c = w.steps;
    const uint64_t blk0 = (tile * 32 + lane) * c;
    const uint64_t nmine = blk0 < nblk ? min(c, nblk - blk0) : 0;
    const uint32_t iters = __reduce_max_sync(0xffffffffu, (uint32_t)nmine);
    Lane L;
    if (nmine) decode(v, w.lo + blk0 * span, L, cuts, kThreads);
    for (uint32_t it = 0; it < iters; it++) {
        const bool act = it < nmine;
        // high part of this block: stages after the first high cut
        const uint64_t hi_mask = L.part & ~(((uint64_t)1 << kLowBits) - 1);
        int64_t hF = 0, hB = 0, hU = 0, hW = 0, hM = 0, hY = 0, hS = 0;
        int c_h = G;
        int hpop = 0;
        int64_t b = 1;
        const LowE *lt = lowtab;
        if (act) {
            b = at<int64_t>(v.img, v.S->off_b)[L.d[D_B]];
            lt = lowtab + (size_t)L.d[D_B] * (1 << kLowBits);
            uint64_t m = hi_mask;
            hpop = __popcll(m);
            if (m) {
                c_h = __ffsll((long long)m);
                m &= m - 1;
                int beg = c_h;
                hY = Y[c_h - 1];
                hS = Y[c_h - 1];
                for (;;) {
                    int end;
                    if (m) {
                        end = __ffsll((long long)m);
                        m &= m - 1;
                    } else {
                        end = G;
                    }
                    const int64_t F = PF[end] - PF[beg], Bw = PB[end] - PB[beg], U = PU[end] - PU[beg];
                    const int64_t Wt = PW[end] - PW[beg], XY = PX[end] - PX[beg], BI = PI[end] - PI[beg];
                    hF = max(hF, F);
                    hB = max(hB, Bw);
                    hU = max(hU, U);
                    hW = max(hW, Wt);
                    hM = max(hM, 2 * b * XY + 2 * Wt + BI);
                    if (end == G) break;
                    hY = max(hY, Y[end - 1]);
                    hS += Y[end - 1];
                    beg = end;
                }
            }
        }
        const uint64_t gbase = v.S->offset + w.lo + (blk0 + it) * span;
        for (uint32_t x = 0; x < (1u << kLowBits); x++) {
            StageT st;
            int64_t ns = 1;
            if (act) {
                const LowE e = lt[x];
                const int beg = e.e_last;
                const int64_t F = PF[c_h] - PF[beg], Bw = PB[c_h] - PB[beg], U = PU[c_h] - PU[beg];
                const int64_t Wt = PW[c_h] - PW[beg], XY = PX[c_h] - PX[beg], BI = PI[c_h] - PI[beg];
                st.maxF = max(max(e.F, F), hF);
                st.maxB = max(max(e.B, Bw), hB);
                st.maxU = max(max(e.U, U), hU);
                st.maxW = max(max(e.W, Wt), hW);
                st.memI = max(max(e.memI, 2 * b * XY + 2 * Wt + BI), hM);
                st.maxY = max(e.maxY, hY);
                st.sumY = e.sumY + hS;
                ns = e.pop + hpop + 1;
            }
            eval_partition<FAM>(C, act, L, st, ns, gbase + (uint64_t)x * C.Q, tk, cnt);
        }
        tk.refresh();
        if (it + 1 < nmine) advance(w, v, L, cuts, kThreads);   // next block: inc_part = 256
    }
}

// ------------------------------------------------------------------ mode 3: COMB partitions, incremental
// Lane-blocked pipeline / pd sweeps over combination-mode partitions (the cfg5 shape: ~6.3e8
// partitions x S x p_d x alpha x beta), ring collectives, at most 2 alpha and 2 beta rows.
//
// Stage terms.  A lane walks consecutive partitions, and the
// lexicographic successor mostly moves only the last cut c = c_{s-1}: stages 0..s-3 are then
// unchanged, so their maxima `pre` (and the prefix values at a = c_{s-2}) are kept, and only
// stage s-2 = rows (a, c] and the last stage (c, G] are formed from the prefix values at c --
// seven shared-memory loads and exact int64 differences / maxima, whatever s is.  Any other
// successor (an earlier cut moves, the stage count or a slower digit changes) recomputes
// `pre` from the cut list; every term is an exact integer maximum, so the split composes to
// the same StageT as stage_terms().
//
// Keys.  The fp64 trees are eval_partition's, operation for operation, with each subtree
// formed at the loop level it depends on: per partition FB = D(maxF + maxB), U tau, D(delta
// maxY), D(delta maxW); per S (4 per pass) comp = ((cseg FB) tau + U tau) (+inf when S > b or
// the partition is infeasible) and the pipeline term P = pp_c (alpha + (bS D(delta maxY))
// beta) for the <= 2 x 2 alpha/beta rows; per p_d value the GE term G = ge_c (alpha + ge_s
// beta) with ge_s = D(delta maxW) / p_d (x 2^-k exactly for a power of two); per
// configuration t = comp + G, t = t + P (t_iter, exact); the screen forms key = t I once per
// p_d value from the smallest t (below).  The (b, stage count, S) and (b, stage
// count, p_d) constants -- cseg, pp_c, b/S, ge_c, I = D/(b p_d), the tiers' alpha/beta -- come
// from per-CTA tables built with the memo (build_memo).  With one alpha (beta) row the second
// is a duplicate of the first: duplicate keys cannot change a minimum.
//
// Selection.  Only a lower bound of the high word of the partition's keys is kept (key <= adm
// implies hi(key) <= hi(adm) for non-negative doubles; D(t I) is monotone in t, so the 16 keys
// of one p_d value are at least D(t_lo I) with t_lo <= min t); a partition that may hold a candidate is
// re-evaluated by eval_partition (offers, exact).  Memory feasibility is the integer
// threshold memI <= mem_threshold(cap), exactly the fp64 compare (mem_threshold).  The feasible
// count is separable: (#S <= b) x (#p_d with a tier) x n_LAB per feasible partition.
struct __align__(16) CmbN {   // per stage count n: P2P tier alpha/beta rows, dims with a tier
    double a0, a1, b0, b1;
    int32_t ndok, ok, pad0, pad1;
};
struct __align__(16) CmbS {   // per (b, n, S): (n + S - 1)(b/S), 2 (n + S - 2) or 0, b/S, S <= b
    double cseg, ppc, bS;
    int32_t sok, pad;
};
struct __align__(16) CmbD {   // per (b, n, dims): ring GE coefficient (+inf: no tier), D/(b p_d),
    double gc, I, a0, a1, b0, b1, scale;   // GE tier alpha/beta rows, 2^-k for p_d = 2^k (else 0)
    int32_t pd, div;                       // div: p_d not a power of two -> IEEE division
};
static_assert(sizeof(CmbN) == 48 && sizeof(CmbS) == 32 && sizeof(CmbD) == 64, "comb table layout");

// Per-lane stage state of tile_body_comb in shared memory (column per thread, int64):
// pre = maxima over stages 0..s-3 and the prefix values at a = c_{s-2}; pre2 = maxima over
// stages 0..s-4 and the prefix values at c_{s-3} (the "mid" successor, which moves c_{s-2},
// rebuilds pre from pre2 plus one stage).  Maxima: F, B, U, W, memI, Y; prefixes: F, B, U, W, XY, BI.
enum { LS_PRE = 0, LS_APRE = 6, LS_PRE2 = 12, LS_BPRE = 18, kLaneState = 24 };
#ifndef PARADL_REFRESH_WARM
#define PARADL_REFRESH_WARM 8
#endif
constexpr int kRefreshWarm = PARADL_REFRESH_WARM;   // partitions per tile with a bound re-read each
static_assert(kLaneStateBytes == kLaneState * 8u * kThreads, "lane state layout");

template <int FAM>
__device__ void tile_body_comb(const LaunchArgs &a, const WorkItem &w, uint64_t tile, uint8_t *smem,
                               uint16_t *cuts, WarpTopK &tk, unsigned long long &cnt, const double *memo,
                               int64_t *lstate) {
    BlkCtx C = make_blk(w, smem, memo);
    const View &v = C.v;
    const SubHdr *S = v.S;
    const ImgHdr *H = v.H;
    const ModelHdr *M = v.M;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int G = M->G;
    const int64_t *PF = at<int64_t>(v.mb, M->off_pf);
    const int64_t *PB = at<int64_t>(v.mb, M->off_pb);
    const int64_t *PU = at<int64_t>(v.mb, M->off_pu);
    const int64_t *PW = at<int64_t>(v.mb, M->off_pw);
    const int64_t *PX = at<int64_t>(v.mb, M->off_pxy);
    const int64_t *PI = at<int64_t>(v.mb, M->off_pbi);
    const int64_t *Y = at<int64_t>(v.mb, M->off_y);
    const int64_t *bv = at<int64_t>(v.img, S->off_b);
    const int64_t delta = H->delta;
    const double INF = CUDART_INF;
    const uint32_t ns1 = (uint32_t)S->s_max + 1, nS = C.nS, nD = C.nD;
    const uint8_t *cb = reinterpret_cast<const uint8_t *>(memo) + w.cmb_off;
    const CmbN *tabN = reinterpret_cast<const CmbN *>(cb);
    const CmbS *tabS = reinterpret_cast<const CmbS *>(cb + ns1 * sizeof(CmbN));
    const uint32_t nSp = (nS + kSB - 1) / kSB * kSB;   // CmbS rows padded to whole passes (sok = 0)
    const CmbD *tabD =
        reinterpret_cast<const CmbD *>(cb + ns1 * sizeof(CmbN) + (size_t)S->radix[D_B] * ns1 * nSp * sizeof(CmbS));
    // per flops value tau = 1/R, per cap value the integer memory threshold (after CmbD)
    const double *tauT = reinterpret_cast<const double *>(reinterpret_cast<const uint8_t *>(tabD) +
                                                          (size_t)S->radix[D_B] * ns1 * nD * sizeof(CmbD));
    const int64_t *memT = reinterpret_cast<const int64_t *>(tauT + S->radix[D_FLOPS]);
    int64_t *ls = lstate + threadIdx.x;
    const uint64_t nblk = (w.hi - w.lo) / C.Q;
    const uint64_t c = w.steps;
    const uint64_t blk0 = (tile * 32 + lane) * c;
    const uint64_t nmine = blk0 < nblk ? min(c, nblk - blk0) : 0;
    const uint32_t iters = __reduce_max_sync(full, (uint32_t)nmine);
    Lane L;
    int clast = 0, ns = 1;
    int upd = 2;   // stage state to rebuild before the next partition: 0 none, 1 mid, 2 all
    // the partition's StageT from the lane state: formed once for the keys and again, only
    // when the screen passes, for the re-evaluation (so it is not live across the key block)
    auto form_st = [&](StageT &st, int64_t twob) {
        if (ns == 1) {
            st.maxF = PF[G] - PF[0];
            st.maxB = PB[G] - PB[0];
            st.maxU = PU[G] - PU[0];
            st.maxW = PW[G] - PW[0];
            st.memI = twob * (PX[G] - PX[0]) + 2 * (PW[G] - PW[0]) + (PI[G] - PI[0]);
        } else {
            // stage s-2 = rows (a, c], stage s-1 = rows (c, G]
            const int64_t cF = PF[clast], cB = PB[clast], cU = PU[clast], cW = PW[clast], cX = PX[clast],
                          cI = PI[clast], y = Y[clast - 1];
            const int64_t W1 = cW - ls[(LS_APRE + 3) * kThreads], W2 = PW[G] - cW;
            st.maxF = max(ls[(LS_PRE + 0) * kThreads], max(cF - ls[(LS_APRE + 0) * kThreads], PF[G] - cF));
            st.maxB = max(ls[(LS_PRE + 1) * kThreads], max(cB - ls[(LS_APRE + 1) * kThreads], PB[G] - cB));
            st.maxU = max(ls[(LS_PRE + 2) * kThreads], max(cU - ls[(LS_APRE + 2) * kThreads], PU[G] - cU));
            st.maxW = max(ls[(LS_PRE + 3) * kThreads], max(W1, W2));
            st.memI = max(ls[(LS_PRE + 4) * kThreads],
                          max(twob * (cX - ls[(LS_APRE + 4) * kThreads]) + 2 * W1 + (cI - ls[(LS_APRE + 5) * kThreads]),
                              twob * (PX[G] - cX) + 2 * W2 + (PI[G] - cI)));
            st.maxY = max(ls[(LS_PRE + 5) * kThreads], y);
        }
    };
    uint32_t tcnt = 0;   // feasible count of this tile (flushed into cnt before it could wrap)
    if (nmine) decode(v, w.lo + blk0 * C.Q, L, cuts, kThreads);
    for (uint32_t it = 0; it < iters; it++) {
        const bool act = it < nmine;
        StageT st;
        st.maxF = st.maxB = st.maxU = st.maxW = st.maxY = st.sumY = st.memI = 0;
        int64_t b = 1;
        if (act) {
            PCHECK(L.d[D_B] < S->radix[D_B] && L.ns >= 1 && L.ns <= S->s_max && L.part < S->part_n);
            b = bv[L.d[D_B]];
            const int64_t twob = 2 * b;
            if (upd) {
                ns = L.ns;
                if (ns >= 2) {
                    // a = c_{s-2} (row 0 if s = 2), b2 = c_{s-3} (row 0 if s <= 3)
                    const int a0 = ns >= 3 ? cuts[(ns - 3) * kThreads] : 0;
                    const int b2 = ns >= 4 ? cuts[(ns - 4) * kThreads] : 0;
                    StageT p2;
                    if (upd == 2) {   // maxima over stages 0..s-4 and the prefix values at b2
                        p2.maxF = p2.maxB = p2.maxU = p2.maxW = p2.maxY = p2.sumY = p2.memI = 0;
                        if (ns >= 4) stage_span(v, cuts, kThreads, twob, ns, 0, ns - 3, 0, p2);
                        ls[(LS_PRE2 + 0) * kThreads] = p2.maxF;
                        ls[(LS_PRE2 + 1) * kThreads] = p2.maxB;
                        ls[(LS_PRE2 + 2) * kThreads] = p2.maxU;
                        ls[(LS_PRE2 + 3) * kThreads] = p2.maxW;
                        ls[(LS_PRE2 + 4) * kThreads] = p2.memI;
                        ls[(LS_PRE2 + 5) * kThreads] = p2.maxY;
                        ls[(LS_BPRE + 0) * kThreads] = PF[b2];
                        ls[(LS_BPRE + 1) * kThreads] = PB[b2];
                        ls[(LS_BPRE + 2) * kThreads] = PU[b2];
                        ls[(LS_BPRE + 3) * kThreads] = PW[b2];
                        ls[(LS_BPRE + 4) * kThreads] = PX[b2];
                        ls[(LS_BPRE + 5) * kThreads] = PI[b2];
                    } else {
                        p2.maxF = ls[(LS_PRE2 + 0) * kThreads];
                        p2.maxB = ls[(LS_PRE2 + 1) * kThreads];
                        p2.maxU = ls[(LS_PRE2 + 2) * kThreads];
                        p2.maxW = ls[(LS_PRE2 + 3) * kThreads];
                        p2.memI = ls[(LS_PRE2 + 4) * kThreads];
                        p2.maxY = ls[(LS_PRE2 + 5) * kThreads];
                    }
                    // stage s-3 = rows (b2, a] (exists when s >= 3), folded into pre
                    const int64_t eF = PF[a0], eB = PB[a0], eU = PU[a0], eW = PW[a0], eX = PX[a0], eI = PI[a0];
                    if (ns >= 3) {
                        const int64_t W3 = eW - ls[(LS_BPRE + 3) * kThreads];
                        p2.maxF = max(p2.maxF, eF - ls[(LS_BPRE + 0) * kThreads]);
                        p2.maxB = max(p2.maxB, eB - ls[(LS_BPRE + 1) * kThreads]);
                        p2.maxU = max(p2.maxU, eU - ls[(LS_BPRE + 2) * kThreads]);
                        p2.maxW = max(p2.maxW, W3);
                        p2.memI = max(p2.memI, twob * (eX - ls[(LS_BPRE + 4) * kThreads]) + 2 * W3 +
                                                   (eI - ls[(LS_BPRE + 5) * kThreads]));
                        p2.maxY = max(p2.maxY, Y[a0 - 1]);
                    }
                    ls[(LS_PRE + 0) * kThreads] = p2.maxF;
                    ls[(LS_PRE + 1) * kThreads] = p2.maxB;
                    ls[(LS_PRE + 2) * kThreads] = p2.maxU;
                    ls[(LS_PRE + 3) * kThreads] = p2.maxW;
                    ls[(LS_PRE + 4) * kThreads] = p2.memI;
                    ls[(LS_PRE + 5) * kThreads] = p2.maxY;
                    ls[(LS_APRE + 0) * kThreads] = eF;
                    ls[(LS_APRE + 1) * kThreads] = eB;
                    ls[(LS_APRE + 2) * kThreads] = eU;
                    ls[(LS_APRE + 3) * kThreads] = eW;
                    ls[(LS_APRE + 4) * kThreads] = eX;
                    ls[(LS_APRE + 5) * kThreads] = eI;
                    clast = cuts[(ns - 2) * kThreads];
                }
                upd = 0;
            }
            PCHECK(ns == 1 || (clast >= 1 && clast <= G - 1 && clast > (ns >= 3 ? cuts[(ns - 3) * kThreads] : 0)));
            form_st(st, twob);
        }
        // ---- keys of the partition's S x dims x Ls x alpha x beta block
        double FBs = 0.0, Utau = 0.0, dmaxY = 0.0, mW = 0.0, part_inf = INF;
        double at0 = 0.0, at1 = 0.0, bt0 = 0.0, bt1 = 0.0;
        uint32_t ndok = 0, bi = 0;
        double tau = 0.0;
        if (act) {
            tau = tauT[L.d[D_FLOPS]];
            bi = L.d[D_B];
            const CmbN tn = tabN[ns];
            at0 = tn.a0, at1 = tn.a1, bt0 = tn.b0, bt1 = tn.b1;
            ndok = (uint32_t)tn.ndok;
            part_inf = (tn.ok && st.memI <= memT[L.d[D_CAP]]) ? 0.0 : INF;
            FBs = i2d(st.maxF + st.maxB);
            Utau = dmul(i2d(st.maxU), tau);
            dmaxY = i2d(delta * st.maxY);
            if (FAM == PARADL_PD) mW = i2d(delta * st.maxW);
        }
        const CmbS *srow = tabS + ((size_t)bi * ns1 + ns) * nSp;
        const CmbD *drow = tabD + ((size_t)bi * ns1 + ns) * nD;
        int hmin = 0x7fffffff;
        uint32_t nSok = 0;
        for (uint32_t iS0 = 0; iS0 < nSp; iS0 += kSB) {
            double comp[kSB], P[kSB][4];
#pragma unroll
            for (int u = 0; u < kSB; u++) {
                const CmbS q = srow[iS0 + u];
                const bool sok = act && q.sok;
                nSok += sok ? 1u : 0u;
                comp[u] = dadd(dadd(dmul(dmul(q.cseg, FBs), tau), Utau), sok ? part_inf : INF);
                const double pps = dmul(q.bS, dmaxY);
                const double x0 = dmul(pps, bt0), x1 = dmul(pps, bt1);
                P[u][0] = dmul(q.ppc, dadd(at0, x0));
                P[u][1] = dmul(q.ppc, dadd(at0, x1));
                P[u][2] = dmul(q.ppc, dadd(at1, x0));
                P[u][3] = dmul(q.ppc, dadd(at1, x1));
            }
            // per p_d value: the GE terms G = ge_c (alpha + ge_s beta) of the 2 x 2 rows, then the
            // 16 keys t = comp + G, t = t + P, key = t I and their smallest high word
            auto dims_keys = [&](const CmbD &d, double gs) {
                double Gq[4] = {0.0, 0.0, 0.0, 0.0};
                if (FAM == PARADL_PD) {
                    const double g0 = dmul(gs, d.b0), g1 = dmul(gs, d.b1);
                    Gq[0] = dmul(d.gc, dadd(d.a0, g0));
                    Gq[1] = dmul(d.gc, dadd(d.a0, g1));
                    Gq[2] = dmul(d.gc, dadd(d.a1, g0));
                    Gq[3] = dmul(d.gc, dadd(d.a1, g1));
                }
                int th = 0x7fffffff;
#pragma unroll
                for (int u = 0; u < kSB; u++) {
                    int h[4];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const double t = FAM == PARADL_PD ? dadd(dadd(comp[u], Gq[q]), P[u][q]) : dadd(comp[u], P[u][q]);
                        h[q] = __double2hiint(t);
                    }
                    th = min(th, min(h[0], h[1]));   // two 3-input minima per S value
                    th = min(th, min(h[2], h[3]));
                }
                // key = t I is monotone in t (I > 0): the smallest key of these 16 is at least
                // D(t_lo I), t_lo = the smallest t with its low word cleared
                hmin = min(hmin, __double2hiint(dmul(__hiloint2double(th, 0), d.I)));
            };
            if (w.flags & kWorkPow2) {   // every p_d a power of two: ge_s = mW 2^-k, no branch
#pragma unroll kCombUnroll
                for (uint32_t iD = 0; iD < nD; iD++) {
                    const CmbD d = drow[iD];
                    dims_keys(d, dmul(mW, d.scale));
                }
            } else {
#pragma unroll 1
                for (uint32_t iD = 0; iD < nD; iD++) {
                    const CmbD d = drow[iD];
                    dims_keys(d, d.div ? ddiv_rare(mW, i2d(d.pd)) : dmul(mW, d.scale));
                }
            }
        }
        if (act && part_inf == 0.0) {
            tcnt += nSok * ndok * C.nLAB;   // <= Q < 2^31 per partition (host check)
            if (tcnt & 0x80000000u) {
                cnt += tcnt;
                tcnt = 0;
            }
        }
        const bool maybe = act && hmin <= __double2hiint(tk.adm);
        if (__any_sync(full, maybe)) {
            const uint64_t gblk = S->offset + w.lo + (blk0 + it) * C.Q;
            StageT sr;
            sr.maxF = sr.maxB = sr.maxU = sr.maxW = sr.maxY = sr.sumY = sr.memI = 0;
            if (maybe) form_st(sr, 2 * bv[L.d[D_B]]);
            eval_partition<FAM, false>(C, maybe, L, sr, ns, gblk, tk, cnt);
        }
        // the shared bound only tightens the screen: every partition while the lists fill
        // (the first ones pass the screen until the bound converges), then every 8th
        // (`ab_refresh_period_s16.log`: every 2nd / 4th / 8th / 16th / 32nd)
        if ((int)it < kRefreshWarm || (it & 7) == 7) tk.refresh();   // (warm-up: N = 256 shards 0.93 -> 0.63 ms)
        if (it + 1 < nmine) {
            if (ns >= 2 && clast < G - 1) {   // lexicographic successor moves only the last cut
                clast++;
                L.part++;
            } else if (ns >= 3 && L.part + 1 < S->part_n) {
                // an earlier cut moves (same stage count: the last cut is at its maximum, so
                // the successor is inside this stage-count block unless every cut is)
                cuts[(ns - 2) * kThreads] = (uint16_t)clast;
                const int c3 = ns >= 4 ? cuts[(ns - 4) * kThreads] : 0;
                succ_comb(v, L, cuts, kThreads);
                L.part++;
                upd = (L.ns == ns && (ns < 4 || cuts[(ns - 4) * kThreads] == c3)) ? 1 : 2;
            } else {
                // a successor that moves c_{s-2} (same s, same slower digits, c_{s-3} kept)
                // rebuilds pre from pre2 and one stage; anything else rebuilds both
                if (ns >= 2) cuts[(ns - 2) * kThreads] = (uint16_t)clast;
                const int c3 = ns >= 4 ? cuts[(ns - 4) * kThreads] : 0;
                const uint32_t d0 = L.d[D_B], d1 = L.d[D_FLOPS], d2 = L.d[D_CAP];
                advance(w, v, L, cuts, kThreads);
                const bool mid = ns >= 3 && L.ns == ns && L.d[D_B] == d0 && L.d[D_FLOPS] == d1 && L.d[D_CAP] == d2 &&
                                 (ns < 4 || cuts[(ns - 4) * kThreads] == c3);
                upd = mid ? 1 : 2;
            }
        }
    }
    cnt += tcnt;
}

// Per-CTA prologue: memo tables of the lane-blocked work items (b/S and D/(b*dims0)),
// with the same fp64 operations compute_mid uses, and the low-bit stage tables of mode 2.
__device__ void build_memo(const LaunchArgs &a, uint8_t *smem, double *memo_base, LowE *low_base) {
    {
        SmemExtra *ex = reinterpret_cast<SmemExtra *>(smem + a.img_bytes);
        const ImgHdr *H = at<ImgHdr>(smem, 0);
        for (int n = threadIdx.x; n < PARADL_MAX_STAGES + 8; n += blockDim.x)
            ex->tier_by_n[n] = (int8_t)(n >= 1 ? tier_of(H, n) : 0);
    }
    for (int wi = 0; wi < a.n_work; wi++) {
        const WorkItem &w = a.work[wi];
        if (w.family == PARADL_DATA_LW && w.memo_n) {
            // per dims value and weighted layer l (row order): the Allreduce of delta |w_l|
            // over p PEs as c (alpha + s beta) -- make_ar's ring / tree choice per message
            const View v = make_view(smem, w.sub);
            const ModelHdr *M = v.M;
            const int64_t *PW = at<int64_t>(v.mb, M->off_pw);
            const int32_t *dmv = at<int32_t>(v.img, v.S->off_dims);
            const uint32_t nD = v.S->radix[D_DIMS], G = (uint32_t)M->G, lwn = w.memo_n / (2u * nD);
            double *tab = memo_base + w.memo_off / sizeof(double);
            for (uint32_t e = threadIdx.x; e < nD * G; e += blockDim.x) {
                const uint32_t iD = e / G, l = e - iD * G;
                const int64_t wl = PW[l + 1] - PW[l];
                if (wl <= 0) continue;
                uint32_t j = 0;   // rank among the weighted rows
                for (uint32_t q = 0; q < l; q++) j += PW[q + 1] > PW[q];
                const int64_t p = dmv[4 * iD];
                const ARt r = make_ar(v.H, p, i2d(v.H->delta * wl), div_i(v.H->delta * wl, p), 0);
                double *o = tab + ((size_t)iD * lwn + j) * 2;
                o[0] = r.on ? r.c : 0.0;
                o[1] = r.on ? r.s : 0.0;
            }
            continue;
        }
        if (w.mode == 0) continue;
        const View v = make_view(smem, w.sub);
        const SubHdr *S = v.S;
        const uint32_t nS = S->radix[D_S], nD = S->radix[D_DIMS];
        double *tab = memo_base + w.memo_off / sizeof(double);
        const int64_t *bv = at<int64_t>(v.img, S->off_b);
        const int32_t *Sv = at<int32_t>(v.img, S->off_S);
        const int32_t *dmv = at<int32_t>(v.img, S->off_dims);
        const uint32_t nrow = S->radix[D_B] * (nS + nD);
        if (w.family == PARADL_PD && (w.mode == 1 || w.mode == 3)) {
            // ring GE coefficient and tier per (stage count s, dims value): make_ar's ring
            // branch, ge_c = 2 (p_d - 1) (0 when p_d = 1), +inf when s p_d exceeds every tier
            const uint32_t nDp = nD + 1;
            const uint32_t n_stage = (S->part_mode == PARADL_PART_COMB ? S->s_max : S->G) + 1;
            double *gc = tab + nrow;
            int32_t *gt = reinterpret_cast<int32_t *>(gc + n_stage * nDp);
            // row s = 0 (no such stage count) holds the exact scale 2^-k of power-of-two p_d
            // (0: divide); column n_dims of gt holds the number of dims values in a tier
            for (uint32_t e = threadIdx.x; e < n_stage * nDp; e += blockDim.x) {
                const uint32_t sv = e / nDp, iD = e - sv * nDp;
                const int64_t pd = iD < nD ? dmv[4 * iD] : 1;
                if (sv == 0) {
                    gc[e] = (pd > 0 && (pd & (pd - 1)) == 0)
                                ? __longlong_as_double((long long)(1023 - (63 - __clzll(pd))) << 52)
                                : 0.0;
                    gt[e] = 0;
                } else if (iD == nD) {
                    int ok = 0;
                    for (uint32_t j = 0; j < nD; j++) ok += tier_of(v.H, (int64_t)sv * dmv[4 * j]) >= 0;
                    gc[e] = 0.0;
                    gt[e] = ok;
                } else {
                    const int tp = tier_of(v.H, (int64_t)sv * pd);
                    gc[e] = tp < 0 ? CUDART_INF : (pd != 1 ? i2d(2 * (pd - 1)) : 0.0);
                    gt[e] = max(tp, 0);
                }
            }
        }
        if (w.mode == 3) {
            // mode-3 tables (tile_body_comb): per stage count n the P2P tier's alpha/beta rows,
            // per (b, n, S) and (b, n, dims) the constants of eval_partition's trees
            const uint32_t ns1 = (uint32_t)S->s_max + 1, nb = S->radix[D_B];
            const uint32_t nA = S->radix[D_ALPHA], nBt = S->radix[D_BETA];
            const int NT = v.H->n_tiers;
            const double *al = at<double>(v.img, S->off_alpha), *be = at<double>(v.img, S->off_beta);
            uint8_t *cb = reinterpret_cast<uint8_t *>(memo_base) + w.cmb_off;
            CmbN *tn = reinterpret_cast<CmbN *>(cb);
            CmbS *ts = reinterpret_cast<CmbS *>(cb + ns1 * sizeof(CmbN));
            const uint32_t nSp = (nS + kSB - 1) / kSB * kSB;   // whole passes; padding rows sok = 0
            CmbD *td = reinterpret_cast<CmbD *>(cb + ns1 * sizeof(CmbN) + (size_t)nb * ns1 * nSp * sizeof(CmbS));
            const uint32_t ia1 = nA > 1 ? 1 : 0, ib1 = nBt > 1 ? 1 : 0;
            for (uint32_t n = threadIdx.x; n < ns1; n += blockDim.x) {
                const int t = n >= 1 ? tier_of(v.H, n) : -1;
                const int tt = max(t, 0) + v.H->p2p_off;   // point-to-point column (Q40)
                CmbN q;
                q.a0 = al[tt];
                q.a1 = al[ia1 * NT + tt];
                q.b0 = be[tt];
                q.b1 = be[ib1 * NT + tt];
                int ok = 0;
                for (uint32_t j = 0; j < nD; j++)
                    ok += w.family == PARADL_PD ? tier_of(v.H, (int64_t)n * dmv[4 * j]) >= 0 : 1;
                q.ndok = ok;
                q.ok = t >= 0;
                q.pad0 = q.pad1 = 0;
                tn[n] = q;
            }
            for (uint32_t e = threadIdx.x; e < nb * ns1 * nSp; e += blockDim.x) {
                const uint32_t ib = e / (ns1 * nSp), n = (e / nSp) % ns1, j = e % nSp;
                CmbS q;
                if (j < nS) {
                    const int64_t b = bv[ib], Sg = Sv[j];
                    q.bS = ddiv(i2d(b), i2d(Sg));
                    q.cseg = dmul(i2d((int64_t)n + Sg - 1), q.bS);
                    q.ppc = n > 1 ? i2d(2 * ((int64_t)n + Sg - 2)) : 0.0;
                    q.sok = Sg >= 1 && Sg <= b;
                } else {   // padding: comp = +inf, never counted
                    q.bS = q.cseg = q.ppc = 0.0;
                    q.sok = 0;
                }
                q.pad = 0;
                ts[e] = q;
            }
            for (uint32_t e = threadIdx.x; e < nb * ns1 * nD; e += blockDim.x) {
                const uint32_t ib = e / (ns1 * nD), n = (e / nD) % ns1, j = e % nD;
                const int64_t b = bv[ib];
                const int64_t pd = w.family == PARADL_PD ? dmv[4 * j] : 1;
                const int tp = tier_of(v.H, (int64_t)n * pd);
                const int tt = max(tp, 0);
                CmbD q;
                q.I = ddiv(i2d(v.M->D), i2d(b * pd));
                q.gc = tp < 0 ? CUDART_INF : (pd != 1 ? i2d(2 * (pd - 1)) : 0.0);
                q.a0 = al[tt];
                q.a1 = al[ia1 * NT + tt];
                // beta x phi_pd when the n stage Allreduces run at once (Q40): the oracle's
                // beta * phi product, formed once here instead of per configuration
                const double phi = (w.family == PARADL_PD && n > 1) ? v.H->phi_pd : 1.0;
                q.b0 = dmul(be[tt], phi);
                q.b1 = dmul(be[ib1 * NT + tt], phi);
                const bool pow2 = pd > 0 && (pd & (pd - 1)) == 0;
                q.scale = pow2 ? __longlong_as_double((long long)(1023 - (63 - __clzll(pd))) << 52) : 0.0;
                q.pd = (int32_t)pd;
                q.div = !pow2;
                td[e] = q;
            }
            double *tt = reinterpret_cast<double *>(td + (size_t)nb * ns1 * nD);
            int64_t *mt = reinterpret_cast<int64_t *>(tt + S->radix[D_FLOPS]);
            for (uint32_t e = threadIdx.x; e < S->radix[D_FLOPS]; e += blockDim.x)
                tt[e] = ddiv(1.0, at<double>(v.img, S->off_flops)[e]);   // = eval_partition's tau
            for (uint32_t e = threadIdx.x; e < S->radix[D_CAP]; e += blockDim.x)
                mt[e] = mem_threshold(v.H, at<double>(v.img, S->off_cap)[e]);
        }
        if (w.mode == 2 && (w.flags & kWorkMaskD)) {
            // screened masks (n_S = 1, one alpha/beta row): per stage count n the same fp64
            // values eval_partition forms: cseg = (n + S - 1) (b / S), pp_c, and alpha/beta of
            // tier_of(n) (0 when no tier holds n stages; such masks are infeasible)
            const uint32_t nb = S->radix[D_B];
            NTab *nt = reinterpret_cast<NTab *>(tab + nrow);
            const int64_t Sg = Sv[0];
            const double *al = at<double>(v.img, S->off_alpha), *be = at<double>(v.img, S->off_beta);
            for (uint32_t e = threadIdx.x; e < nb * kMaskTabN; e += blockDim.x) {
                const uint32_t r = e / kMaskTabN, n = e - r * kMaskTabN;
                const int t = n >= 1 ? tier_of(v.H, n) : -1;
                NTab q;
                q.cseg = dmul(i2d((int64_t)n + Sg - 1), ddiv(i2d(bv[r]), i2d(Sg)));
                q.ppc = i2d(n > 1 ? 2 * ((int64_t)n + Sg - 2) : 0);
                q.aw = t >= 0 ? al[t + v.H->p2p_off] : 0.0;   // point-to-point column (Q40)
                q.bw = t >= 0 ? be[t + v.H->p2p_off] : 0.0;
                nt[e] = q;
            }
        }
        for (uint32_t e = threadIdx.x; e < nrow; e += blockDim.x) {
            const uint32_t ib = e / (nS + nD), j = e - ib * (nS + nD);
            const int64_t b = bv[ib];
            if (j < nS) tab[e] = ddiv(i2d(b), i2d(Sv[j]));
            else {
                const int64_t pd = w.family == PARADL_PD ? dmv[4 * (j - nS)] : 1;
                tab[e] = ddiv(i2d(v.M->D), i2d(b * pd));
            }
        }
        if (w.mode == 2 && (w.flags & kWorkMaskS)) {
            // the (e, pop)-sorted table of 2^kLowBitsS low masks per b, tau / P2P betas folded in
            const ModelHdr *M = v.M;
            const int64_t *PF = at<int64_t>(v.mb, M->off_pf);
            const int64_t *PB = at<int64_t>(v.mb, M->off_pb);
            const int64_t *PU = at<int64_t>(v.mb, M->off_pu);
            const int64_t *PW = at<int64_t>(v.mb, M->off_pw);
            const int64_t *PX = at<int64_t>(v.mb, M->off_pxy);
            const int64_t *PI = at<int64_t>(v.mb, M->off_pbi);
            const int64_t *Y = at<int64_t>(v.mb, M->off_y);
            const double tau = ddiv(1.0, at<double>(v.img, S->off_flops)[0]);
            const double *be = at<double>(v.img, S->off_beta);
            const double mem_max_d = i2d(mem_threshold(v.H, at<double>(v.img, S->off_cap)[0]));
            LowS *ls = reinterpret_cast<LowS *>(low_base + w.low_off);
            const uint32_t n = S->radix[D_B] << kLowBitsS;
            for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) {
                const uint32_t ib = e >> kLowBitsS, x = e & ((1u << kLowBitsS) - 1);
                const int64_t b = bv[ib];
                int64_t F = 0, B = 0, U = 0, Mm = 0, Yy = 0;
                int beg = 0;
                uint32_t m = x;
                while (m) {   // stages [beg, end) closed by low cuts
                    const int end = __ffs(m);
                    m &= m - 1;
                    F = max(F, PF[end] - PF[beg]);
                    B = max(B, PB[end] - PB[beg]);
                    U = max(U, PU[end] - PU[beg]);
                    Mm = max(Mm, 2 * b * (PX[end] - PX[beg]) + 2 * (PW[end] - PW[beg]) + (PI[end] - PI[beg]));
                    Yy = max(Yy, Y[end - 1]);
                    beg = end;
                }
                const double Ypp = dmul(ddiv(i2d(b), i2d(Sv[0])), dmul(i2d(v.H->delta), i2d(Yy)));
                LowS q;
                q.F = i2d(F);
                q.B = i2d(B);
                q.Ut = dmul(i2d(U), tau);
                q.M = i2d(Mm);
                for (int t = 0; t < 4; t++) q.Yb[t] = t < v.H->n_ctiers ? dmul(Ypp, be[t + v.H->p2p_off]) : 0.0;
                // one capacity (host-checked): a low part over it makes every mask of the entry
                // infeasible -- its key becomes +inf through maxF and it is not counted
                if (!(i2d(Mm) <= mem_max_d)) q.F = CUDART_INF;
                ls[((size_t)ib << kLowBitsS) + lows_pos(x)] = q;
            }
            __syncthreads();
            // memory-feasible entries per (b, e, pop) subgroup (one thread per subgroup)
            uint32_t *fc = reinterpret_cast<uint32_t *>(ls + ((size_t)S->radix[D_B] << kLowBitsS));
            constexpr int kE = kLowBitsS + 1, kP = kLowBitsS + 2;
            for (uint32_t g = threadIdx.x; g < S->radix[D_B] * kE * kP; g += blockDim.x) {
                const uint32_t ib = g / (kE * kP), e = (g / kP) % kE, pop = g % kP;
                const int j0 = kSub.start[e][pop], j1 = j0 + kSub.cnt[e][pop];
                uint32_t k = 0;
                for (int j = j0; j < j1; j++) k += ls[((size_t)ib << kLowBitsS) + j].F != CUDART_INF;
                fc[g] = k;
            }
        } else if (w.mode == 2) {
            const ModelHdr *M = v.M;
            const int64_t *PF = at<int64_t>(v.mb, M->off_pf);
            const int64_t *PB = at<int64_t>(v.mb, M->off_pb);
            const int64_t *PU = at<int64_t>(v.mb, M->off_pu);
            const int64_t *PW = at<int64_t>(v.mb, M->off_pw);
            const int64_t *PX = at<int64_t>(v.mb, M->off_pxy);
            const int64_t *PI = at<int64_t>(v.mb, M->off_pbi);
            const int64_t *Y = at<int64_t>(v.mb, M->off_y);
            const uint32_t n = S->radix[D_B] << kLowBits;
            for (uint32_t e = threadIdx.x; e < n; e += blockDim.x) {
                const uint32_t ib = e >> kLowBits, x = e & ((1u << kLowBits) - 1);
                const int64_t b = bv[ib];
                LowE L{};
                int beg = 0;
                uint32_t m = x;
                while (m) {   // stages [beg, end) closed by low cuts
                    const int end = __ffs(m);
                    m &= m - 1;
                    const int64_t Wt = PW[end] - PW[beg], XY = PX[end] - PX[beg], BI = PI[end] - PI[beg];
                    L.F = max(L.F, PF[end] - PF[beg]);
                    L.B = max(L.B, PB[end] - PB[beg]);
                    L.U = max(L.U, PU[end] - PU[beg]);
                    L.W = max(L.W, Wt);
                    L.memI = max(L.memI, 2 * b * XY + 2 * Wt + BI);
                    L.maxY = max(L.maxY, Y[end - 1]);
                    L.sumY += Y[end - 1];
                    beg = end;
                }
                L.e_last = beg;
                L.pop = __popc(x);
                if (w.flags & kWorkMaskD) {
                    LowD d;
                    d.F = i2d(L.F);
                    d.B = i2d(L.B);
                    d.U = i2d(L.U);
                    d.M = i2d(L.memI);
                    d.Y = i2d(L.maxY);
                    d.pop = L.pop;
                    d.e_last = L.e_last;
                    d.Ypp = dmul(ddiv(i2d(b), i2d(Sv[0])), dmul(i2d(v.H->delta), d.Y));
                    d.pad_ = 0.0;
                    reinterpret_cast<LowD *>(low_base + w.low_off)[e] = d;

                } else {
                    (low_base + w.low_off)[e] = L;
                }
            }
        }
    }
    __syncthreads();
}

template <int FAM, int DENSE, int BLK>
__global__ void __launch_bounds__(kThreads, BLK == 3 ? PARADL_COMB_MINB : BLK == 2 ? PARADL_MINB + 1
                                            : (FAM == PARADL_PIPELINE && !DENSE && BLK == 0) ? PARADL_PIPE_MINB
                                                                                             : PARADL_MINB)
    sweep_kernel(const __grid_constant__ LaunchArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t mbar;
    __shared__ unsigned long long s_count;
    if (threadIdx.x == 0) s_count = 0;
    stage_image(smem, a.img, a.img_bytes, &mbar);
    SmemExtra *ex = reinterpret_cast<SmemExtra *>(smem + a.img_bytes);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint16_t *cuts = &ex->cuts[0][threadIdx.x];
    const unsigned full = 0xffffffffu;
    WarpTopK tk;
    tk.init(a.k, &ex->lists[warp][0], DENSE ? nullptr : a.gbound);
    unsigned long long cnt = 0;
    double *memo = reinterpret_cast<double *>(smem + a.img_bytes + sizeof(SmemExtra));
    LowE *lowtab = reinterpret_cast<LowE *>(smem + a.img_bytes + sizeof(SmemExtra) + a.memo_bytes);
    double *dtab = a.dtab_bytes ? reinterpret_cast<double *>(smem + a.img_bytes + sizeof(SmemExtra) + a.memo_bytes +
                                                             a.low_bytes)
                                : nullptr;
    if (BLK || FAM == PARADL_DATA_LW) build_memo(a, smem, memo, lowtab);

    for (;;) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(a.tile_counter, 1ull);
        t = __shfl_sync(full, t, 0);
        const uint64_t T = t * (uint64_t)a.n_shards + (uint64_t)a.shard;
        if (T >= a.total_tiles) break;
        int wi = 0;
        while (wi + 1 < a.n_work && T >= a.work[wi + 1].tile_base) wi++;
        const WorkItem &w = a.work[wi];
        if (BLK == 1)
            tile_body_blocked<FAM>(a, w, T - w.tile_base, smem, cuts, tk, cnt, memo, dtab);
        else if (BLK == 3) {
            if (FAM == PARADL_PIPELINE || FAM == PARADL_PD)
                tile_body_comb<FAM>(a, w, T - w.tile_base, smem, cuts, tk, cnt, memo,
                                    reinterpret_cast<int64_t *>(dtab));
        }
        else if (BLK == 2) {
            if (FAM == PARADL_PIPELINE && (w.flags & kWorkMaskS))
                tile_body_mask_s<FAM>(a, w, T - w.tile_base, smem, cuts, tk, cnt, memo,
                                      reinterpret_cast<const LowS *>(lowtab + w.low_off), ex->tier_by_n);
            else if (FAM == PARADL_PIPELINE && (w.flags & kWorkMaskD))
                tile_body_mask_d<FAM>(a, w, T - w.tile_base, smem, cuts, tk, cnt, memo,
                                      reinterpret_cast<const LowD *>(lowtab + w.low_off), ex->tier_by_n);
            else
                tile_body_mask<FAM>(a, w, T - w.tile_base, smem, cuts, tk, cnt, memo, lowtab + w.low_off);
        }
        else
            tile_body<FAM, DENSE>(a, w, T - w.tile_base, smem, cuts, tk, cnt, dtab, memo);
    }

    if (!DENSE) {
        // CTA merge: the 8 warp lists (512 entries) are bitonic-sorted in shared memory and
        // the first k written out.
        paradl_hit *lst = &ex->lists[0][0];   // the warp lists are already in place
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(full, cnt, o);
        if (lane == 0) atomicAdd(&s_count, cnt);
        __syncthreads();
        bitonic_sort_smem(lst, kWarps * PARADL_MAX_TOPK);
        // entries above the shared admission bound (some warp's k-th key) can never reach
        // the global top k: only the sorted prefix at or below it is written and counted
        double gk = CUDART_INF;
        if (a.gbound) {
            const unsigned long long g = *(volatile unsigned long long *)a.gbound;
            if (g != ~0ull) gk = __longlong_as_double((long long)g);
        }
        const int nv = __syncthreads_count(threadIdx.x < (unsigned)a.k && lst[threadIdx.x].idx != ~0ull &&
                                           lst[threadIdx.x].key_epoch_s <= gk);
        paradl_hit *out = a.cta_lists + (size_t)blockIdx.x * a.k;
        for (int i = threadIdx.x; i < nv; i += blockDim.x) out[i] = lst[i];
        if (threadIdx.x == 0) {
            a.cta_nvalid[blockIdx.x] = (uint32_t)nv;
            atomicAdd(a.count, s_count);
        }
    }
}

// ------------------------------------------------------------------ merge kernel
// Merges n_lists ascending lists of k hits (as produced by the sweep kernels and by
// paradl_topk_async) and sums n_counts counts.  The k-th entry of any full list bounds
// the k-th global entry, so only entries <= the smallest such bound can survive: one
// thread per list collects them (early exit, lists are sorted), then one warp selects.
constexpr int kMergeCand = 1536;
constexpr int kMergeLists = 4096;   // lists whose valid-prefix offsets fit the shared scan
constexpr int kLevelLists = 16;     // lists per block of the first merge level

__device__ __forceinline__ void hit_min(double &k, uint64_t &i, double k2, uint64_t i2) {
    if (hit_less(k2, i2, k, i)) {
        k = k2;
        i = i2;
    }
}

__global__ void __launch_bounds__(1024) merge_kernel(const paradl_hit *lists, int64_t n_lists, int32_t k,
                                                      const unsigned long long *counts, int32_t n_counts,
                                                      paradl_hit *out, unsigned long long *count_out,
                                                      const unsigned long long *gbound, int32_t lstride,
                                                      int32_t cstride, unsigned long long *bound_out,
                                                      const uint32_t *nvalid, paradl_hit *lv_out,
                                                      uint32_t *lv_nvalid, unsigned int *lv_done) {
    __shared__ paradl_hit cand[kMergeCand];
    __shared__ uint32_t s_pre[kMergeLists + 1];
    __shared__ unsigned long long s_cnt;
    __shared__ double s_wk[32];
    __shared__ uint64_t s_wi[32];
    __shared__ int s_nc;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lv_out) {
        // fused first level (gridDim.x blocks, 16 lists each, rank selection of at most 1024
        // entries in shared memory: exact ties cannot overflow), then the last block to
        // finish merges the gridDim.x level lists below (threadfence + ticket)
        if (threadIdx.x == 0) s_nc = 0;
        __syncthreads();
        double gk = CUDART_INF;
        if (gbound) {
            const unsigned long long g = *gbound;
            if (g != ~0ull) gk = __longlong_as_double((long long)g);
        }
        {
            const int li = threadIdx.x / PARADL_MAX_TOPK, j = threadIdx.x % PARADL_MAX_TOPK;
            const int64_t l = (int64_t)blockIdx.x * kLevelLists + li;
            if (li < kLevelLists && l < n_lists && j < (int)nvalid[l]) {
                const paradl_hit h = lists[l * lstride + j];
                if (h.key_epoch_s <= gk) cand[atomicAdd(&s_nc, 1)] = h;
            }
        }
        __syncthreads();
        const int n = s_nc;
        if (threadIdx.x < n) {
            const paradl_hit h = cand[threadIdx.x];
            int r = 0;
            for (int j = 0; j < n; j++) r += hit_less(cand[j].key_epoch_s, cand[j].idx, h.key_epoch_s, h.idx);
            if (r < k) lv_out[(int64_t)blockIdx.x * k + r] = h;
        }
        if (threadIdx.x == 0) lv_nvalid[blockIdx.x] = (uint32_t)min(n, k);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_nc = atomicAdd(lv_done, 1u) == gridDim.x - 1;
        __syncthreads();
        if (!s_nc) return;
        __threadfence();
        if (threadIdx.x == 0) *lv_done = 0u;   // ready for the next call
        lists = lv_out;
        nvalid = lv_nvalid;
        n_lists = gridDim.x;
        lstride = k;
        __syncthreads();
    }
    const unsigned full = 0xffffffffu;
    if (threadIdx.x == 0) {
        s_cnt = 0;
        s_nc = 0;
    }
    __syncthreads();
    unsigned long long c = 0;
    for (int i = threadIdx.x; i < n_counts; i += blockDim.x) c += counts[(int64_t)i * cstride];
    atomicAdd(&s_cnt, c);
    // 1. bound: smallest k-th entry over the lists
    double bk = CUDART_INF;
    uint64_t bi = ~0ull;
    // (nvalid: list l holds only its first nvalid[l] entries -- the sweep kernel dropped
    // the rest as above its admission bound)
    for (int64_t l = threadIdx.x; l < n_lists; l += blockDim.x)
        if (!nvalid || nvalid[l] == (uint32_t)k)
            hit_min(bk, bi, lists[l * lstride + (k - 1)].key_epoch_s, lists[l * lstride + (k - 1)].idx);
    for (int o = 16; o; o >>= 1) hit_min(bk, bi, __shfl_xor_sync(full, bk, o), __shfl_xor_sync(full, bi, o));
    if (lane == 0) {
        s_wk[warp] = bk;
        s_wi[warp] = bi;
    }
    __syncthreads();
    if (warp == 0) {
        bk = lane < (int)(blockDim.x >> 5) ? s_wk[lane] : CUDART_INF;
        bi = lane < (int)(blockDim.x >> 5) ? s_wi[lane] : ~0ull;
        for (int o = 16; o; o >>= 1) hit_min(bk, bi, __shfl_xor_sync(full, bk, o), __shfl_xor_sync(full, bi, o));
        if (lane == 0) {
            s_wk[0] = bk;
            s_wi[0] = bi;
        }
    }
    __syncthreads();
    bk = s_wk[0];
    bi = s_wi[0];
    // the sweep's shared admission bound (any warp's k-th key) is also valid: keys above it
    // cannot be in the top k (key-only bound: ties at it stay candidates)
    if (gbound) {
        const unsigned long long g = *gbound;
        if (g != ~0ull) hit_min(bk, bi, __longlong_as_double((long long)g), ~0ull);
    }
    // 2. candidates <= bound: one thread per entry (independent, coalesced loads).  Massive
    //    ties at the bound can overflow the candidate buffer: then the k-th smallest of the
    //    buffered candidates (real entries, so still a valid bound, now with an index that
    //    splits the ties) replaces the bound and the collection is repeated.
    for (int round = 0;; round++) {
        const int64_t n_ent = n_lists * (int64_t)k;
        if (nvalid && n_lists <= kMergeLists) {
            // pruned lists: exclusive prefix of the valid counts (warp 0, lane-chunked scan),
            // then one thread per valid entry (independent loads, one memory latency)
            for (int64_t l = threadIdx.x; l < n_lists; l += blockDim.x) s_pre[l + 1] = nvalid[l];
            __syncthreads();
            if (warp == 0) {
                const int nl = (int)n_lists, per = (nl + 31) / 32, b0 = min(nl, lane * per), b1 = min(nl, b0 + per);
                uint32_t sum = 0;
                for (int l = b0; l < b1; l++) sum += s_pre[l + 1];
                uint32_t inc = sum;
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(full, inc, o);
                    if (lane >= o) inc += v;
                }
                uint32_t run = inc - sum;
                for (int l = b0; l < b1; l++) {
                    const uint32_t v = s_pre[l + 1];
                    s_pre[l] = run;
                    run += v;
                }
                if (lane == 31) s_pre[nl] = inc;
            }
            __syncthreads();
            const uint32_t V = s_pre[n_lists];
            for (uint32_t e = threadIdx.x; e < V; e += blockDim.x) {
                int lo = 0, hi = (int)n_lists;   // last list with s_pre[l] <= e
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_pre[mid] <= e) lo = mid;
                    else hi = mid;
                }
                const paradl_hit h = lists[(int64_t)lo * lstride + (e - s_pre[lo])];
                if (hit_less(bk, bi, h.key_epoch_s, h.idx)) continue;
                const int pos = atomicAdd(&s_nc, 1);
                if (pos < kMergeCand) cand[pos] = h;
            }
        } else if (nvalid) {
            for (int64_t l = threadIdx.x; l < n_lists; l += blockDim.x) {
                const int nv = (int)nvalid[l];
                for (int j = 0; j < nv; j++) {
                    const paradl_hit h = lists[l * lstride + j];
                    if (hit_less(bk, bi, h.key_epoch_s, h.idx)) break;   // sorted: the rest is larger
                    const int pos = atomicAdd(&s_nc, 1);
                    if (pos < kMergeCand) cand[pos] = h;
                }
            }
        } else {
            for (int64_t e = threadIdx.x; e < n_ent; e += blockDim.x) {
                const int64_t l = e / k, j = e - l * k;
                const paradl_hit h = lists[l * lstride + j];
                if (h.idx == ~0ull || hit_less(bk, bi, h.key_epoch_s, h.idx)) continue;
                const int pos = atomicAdd(&s_nc, 1);
                if (pos < kMergeCand) cand[pos] = h;
            }
        }
        __syncthreads();
        if (s_nc <= kMergeCand || round == 8) break;
        // tighter bound: the candidate of rank k-1 among the buffered ones
        for (int i = threadIdx.x; i < kMergeCand; i += blockDim.x) {
            const paradl_hit h = cand[i];
            int r = 0;
            for (int j = 0; j < kMergeCand; j++) r += hit_less(cand[j].key_epoch_s, cand[j].idx, h.key_epoch_s, h.idx);
            if (r == k - 1) {
                s_wk[0] = h.key_epoch_s;
                s_wi[0] = h.idx;
            }
        }
        __syncthreads();
        bk = s_wk[0];
        bi = s_wi[0];
        if (threadIdx.x == 0) s_nc = 0;
        __syncthreads();
    }
    const int nc = s_nc;
    if (nc <= kMergeCand) {
        // rank selection: (key, idx) pairs are distinct, so a candidate's rank is the number
        // of candidates before it; ranks < k go straight to their output slot (one pass,
        // broadcast shared-memory reads, no sorting network)
        for (int i = threadIdx.x; i < nc; i += blockDim.x) {
            const paradl_hit h = cand[i];
            int r = 0;
            for (int j = 0; j < nc; j++) r += hit_less(cand[j].key_epoch_s, cand[j].idx, h.key_epoch_s, h.idx);
            if (r < k) {
                if (out) out[r] = h;
                if (r == k - 1 && bound_out)
                    atomicMin(bound_out, (unsigned long long)__double_as_longlong(h.key_epoch_s));
            }
        }
        if (out)
            for (int i = nc + threadIdx.x; i < k; i += blockDim.x) {
                out[i].idx = ~0ull;
                out[i].key_epoch_s = CUDART_INF;
            }
        if (threadIdx.x == 0 && count_out) *count_out = s_cnt;
        return;
    }
    if (warp != 0) return;
    // pathological ties: one warp scans everything
    __shared__ paradl_hit s_list[PARADL_MAX_TOPK];
    WarpTopK tk;
    tk.init(k, s_list);
    {
        const int64_t n = n_lists * (int64_t)k;
        for (int64_t e = 0; e < n; e += 32) {
            const int64_t j = e + lane;
            const int64_t jj = (j / k) * lstride + (j % k);
            const bool ok = j < n && (!nvalid || (j % k) < (int64_t)nvalid[j / k]) && lists[jj].idx != ~0ull;
            tk.offer(ok, ok ? lists[jj].key_epoch_s : CUDART_INF, ok ? lists[jj].idx : ~0ull);
        }
    }
    if (out && lane < k) out[lane] = s_list[lane];
    if (out && lane + 32 < k) out[lane + 32] = s_list[lane + 32];
    if (lane == 0 && count_out) *count_out = s_cnt;
    if (bound_out && tk.thi != ~0ull && lane == 0)
        atomicMin(bound_out, (unsigned long long)__double_as_longlong(tk.thk));
}

// ------------------------------------------------------------------ explain / decode
template <int FAM>
__device__ void explain_one(const View &v, const Lane &L, const uint16_t *cuts, paradl_config *cfg,
                            paradl_prediction *pr) {
    StageT st = {};
    const int64_t b = at<int64_t>(v.img, v.S->off_b)[L.d[D_B]];
    constexpr bool PIPE = FAM == PARADL_PIPELINE || FAM == PARADL_LAYERPURE || FAM == PARADL_PD || FAM == PARADL_GPIPE;
    if (PIPE) stage_terms(v, L, cuts, 1, b, st);
    Mid m;
    m.reset_memo();
    double gtab[4 * kGpMax];
    m.gp = gtab;
    m.gps = 1;
    m.lwt = nullptr;
    m.lwn = 0;
    compute_mid<FAM>(v, L, st, m);
    if (FAM == PARADL_GPIPE) gpipe_fill(v, L, cuts, 1, m);
    const int NT = v.H->n_tiers;
    const double *arow = at<double>(v.img, v.S->off_alpha) + (size_t)L.d[D_ALPHA] * NT;
    const double *brow = at<double>(v.img, v.S->off_beta) + (size_t)L.d[D_BETA] * NT;
    Phases ph;
    double t;
    if constexpr (FAM == PARADL_DATA_LW) {
        // the per-layer Allreduce fold of lw_ge, row by row (no shared table here)
        const int64_t *PW = at<int64_t>(v.mb, v.M->off_pw);
        const int64_t p = m.p;
        double ge = 0.0;
        if (m.pp_t < 0) ge = CUDART_INF;
        else
            for (int l = 0; l < v.M->G; l++) {
                const int64_t wl = PW[l + 1] - PW[l];
                if (wl <= 0) continue;
                const ARt r = make_ar(v.H, p, i2d(v.H->delta * wl), div_i(v.H->delta * wl, p), 0);
                ge = dadd(ge, dmul(r.on ? r.c : 0.0, dadd(arow[m.pp_t], dmul(r.on ? r.s : 0.0, brow[m.pp_t]))));
            }
        ph = Phases{m.comp, ge, 0.0, 0.0, 0.0, 0.0};
        t = dadd(m.comp, ge);
    } else {
        t = inner<FAM, true>(m, arow, brow, &ph);
    }
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
    if (S->family == PARADL_LAYERWISE) L.ns = 1;   // the mask is a strategy assignment, not stages
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
    for (int t = 0; t < PARADL_MAX_TIERS; t++) {   // the collective tiers
        const bool in = t < v.H->n_ctiers;
        cfg->alpha[t] = in ? at<double>(img, S->off_alpha)[(size_t)L.d[D_ALPHA] * NT + t] : 0.0;
        cfg->beta[t] = in ? at<double>(img, S->off_beta)[(size_t)L.d[D_BETA] * NT + t] : 0.0;
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
    case PARADL_SPATIAL_AG: explain_one<PARADL_SPATIAL_AG>(v, L, cuts, cfg, pr); break;
    case PARADL_GPIPE: explain_one<PARADL_GPIPE>(v, L, cuts, cfg, pr); break;
    case PARADL_DATA_LW: explain_one<PARADL_DATA_LW>(v, L, cuts, cfg, pr); break;
    case PARADL_LAYERWISE: explain_one<PARADL_LAYERWISE>(v, L, cuts, cfg, pr); break;
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

// ------------------------------------------------------------------ a5: halo table
// One warp per (dims, Ls) entry of each spatial / ds sub-sweep of the launch: lanes split
// the rows, then the integer halo volume / row count are summed and the split-limit bits
// OR-ed across the warp -- the same quantities spatial_terms computes row by row.
__global__ void halo_table_kernel(const __grid_constant__ HaloJobs J) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= J.total_entries) return;
    int jb = 0;
    while (jb + 1 < J.n_jobs && gw >= J.job[jb + 1].entry_base) jb++;
    const HaloJob &job = J.job[jb];
    const int e = gw - job.entry_base;
    const View v = make_view(J.img, job.sub);
    const uint32_t nL = v.S->radix[D_LS];
    const uint32_t id = e / nL, il = e - id * nL;
    const int32_t *dm = at<int32_t>(J.img, v.S->off_dims) + 4 * id;
    const int32_t split[3] = {dm[1], dm[2], dm[3]};
    const int32_t Ls = at<int32_t>(J.img, v.S->off_Ls)[il];
    const RowGeo *geo = at<RowGeo>(v.mb, v.M->off_geo);
    const int G = v.M->G;
    const int lim = Ls < G ? Ls : G;
    int64_t NS = 0, HV = 0;
    uint32_t reason = 0;
    for (int l = lane; l < lim; l += 32) {
        const RowGeo &r = geo[l];
        if (r.kind != PARADL_CONV && r.kind != PARADL_POOL) continue;
        NS++;
        for (int ax = 0; ax < 3; ax++) {
            if (split[ax] <= 1) continue;
            const int64_t h = r.K[ax] / 2;
            if (split[ax] > r.X[ax]) reason |= PARADL_R_SCALING;
            if (ceil_div64(r.X[ax], split[ax]) < h || ceil_div64(r.Y[ax], split[ax]) < h) reason |= PARADL_R_SPLIT;
            if (h == 0) continue;
            const int64_t nnb = split[ax] > 2 ? 2 : 1;
            int64_t cx = 1, cy = 1;
            for (int o = 0; o < 3; o++) {
                if (o == ax) continue;
                cx *= ceil_div64(r.X[o], split[o]);
                cy *= ceil_div64(r.Y[o], split[o]);
            }
            HV += (int64_t)r.C * h * cx * nnb + (int64_t)r.F * h * cy * nnb;
        }
    }
    for (int o = 16; o; o >>= 1) {
        NS += __shfl_xor_sync(0xffffffffu, NS, o);
        HV += __shfl_xor_sync(0xffffffffu, HV, o);
        reason |= __shfl_xor_sync(0xffffffffu, reason, o);
    }
    if (lane == 0) {
        HaloEntry hh;
        hh.NS = NS;
        hh.HV = HV;
        hh.reason = reason;
        hh.pad0 = 0;
        hh.pad1 = 0;
        job.tab[e] = hh;
    }
}

cudaError_t launch_halo_tables(const HaloJobs &jobs, cudaStream_t st) {
    const int threads = 256;
    const long long warps = jobs.total_entries;
    const int blocks = (int)((warps * 32 + threads - 1) / threads);
    void *args[] = {const_cast<HaloJobs *>(&jobs)};
    return cudaLaunchKernel((void *)halo_table_kernel, dim3(blocks), dim3(threads), args, 0, st);
}

// ------------------------------------------------------------------ pipeline structure table
// One thread per structure (cap, R, b, partition, S, dims, Ls) of a pipeline sub-sweep: the
// structure terms the mode-0 tiles would otherwise recompute once per warp and structure
// (decode, stage sums, compute_mid<PIPELINE>, fastify) -- the same device code, 32
// structures per warp instruction.  The image is read from global memory (L1/L2 cached).
__global__ void __launch_bounds__(256) struct_table_kernel(const uint8_t *img, uint32_t img_bytes, const StructJob job) {
    // one thread per (cap, R, b, partition) unit: the partition is unranked and its stage
    // sums formed once, then the unit's S x dims x Ls structures are emitted; the image is
    // staged into shared memory first (one TMA bulk copy, as in the sweep kernels)
    extern __shared__ __align__(128) uint8_t simg[];
    __shared__ uint64_t mbar;
    if (job.ctr && blockIdx.x == 0)   // replaces two memsets ahead of the sweep launches
        for (int i = threadIdx.x; i <= job.n_ctr + 1; i += blockDim.x) job.ctr[i] = i == job.n_ctr ? ~0ull : 0ull;
    stage_image(simg, img, img_bytes, &mbar);
    const View v = make_view(simg, job.sub);
    const SubHdr *S = v.S;
    const uint32_t nL = S->radix[D_LS], nD = S->radix[D_DIMS], nS = S->radix[D_S];
    const uint64_t K = (uint64_t)nS * nD * nL;
    const uint64_t unit = job.s_lo / K + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t s_hi = job.s_lo + job.n;
    if (unit * K >= s_hi) return;
    const uint64_t nAB = (uint64_t)S->radix[D_ALPHA] * S->radix[D_BETA];
    if (job.n_shards > 1) {   // skip units no tile of this shard touches
        const uint64_t c0 = max(unit * K * nAB, job.w_lo), c1 = min((unit + 1) * K * nAB, job.w_hi);
        if (c0 >= c1) return;
        const uint64_t ta = job.tile_base + (c0 - job.w_lo) / job.ts, tb = job.tile_base + (c1 - 1 - job.w_lo) / job.ts;
        bool need = tb - ta + 1 >= (uint64_t)job.n_shards;
        for (uint64_t t = ta; !need && t <= tb; t++) need = t % (uint64_t)job.n_shards == (uint64_t)job.shard;
        if (!need) return;
    }
    uint16_t cuts[kMaxCuts + 1];
    Lane L;
    decode(v, unit * K * nAB, L, cuts, 1);
    StageT st;
    stage_terms(v, L, cuts, 1, at<int64_t>(v.img, S->off_b)[L.d[D_B]], st);
    Mid m;
    m.reset_memo();
    for (uint64_t k = 0; k < K; k++) {
        const uint64_t s = unit * K + k;
        if (s < job.s_lo || s >= s_hi) continue;
        L.d[D_LS] = (uint32_t)(k % nL);
        L.d[D_DIMS] = (uint32_t)((k / nL) % nD);
        L.d[D_S] = (uint32_t)(k / ((uint64_t)nL * nD));
        compute_mid<PARADL_PIPELINE>(v, L, st, m);
        fastify(m);
        PipeRec r;
        r.comp = m.comp;
        r.pp_c = m.pp_c;
        r.pp_s = m.pp_s;
        r.I = m.I;
        r.reason = m.reason;
        r.pp_t = m.pp_t;
        r.pad[0] = r.pad[1] = 0;
        job.out[s - job.s_lo] = r;
    }
}

static cudaError_t ensure_smem_attr(void *fn, size_t smem);
cudaError_t launch_struct_table(const uint8_t *img, uint32_t img_bytes, const StructJob &job, uint64_t unit_len,
                                cudaStream_t st) {
    const int threads = 256;
    const uint64_t units = (job.s_lo + job.n + unit_len - 1) / unit_len - job.s_lo / unit_len;
    const unsigned blocks = (unsigned)((units + threads - 1) / threads);
    cudaError_t e = ensure_smem_attr((void *)struct_table_kernel, img_bytes);
    if (e != cudaSuccess) return e;
    struct_table_kernel<<<blocks, threads, img_bytes, st>>>(img, img_bytes, job);
    return cudaGetLastError();
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

// ------------------------------------------------------------------ compact mode: tile offsets
// Exclusive scan of the per-tile feasible counts in ascending index order (segments of the
// launches' tile spaces), one block: off[slot] = feasible configurations before the tile.
__global__ void __launch_bounds__(1024) compact_scan_kernel(const uint32_t *cnt, uint64_t *off,
                                                            const __grid_constant__ CompactSegs segs,
                                                            unsigned long long *total) {
    __shared__ unsigned long long wsum[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long run = 0;
    for (int g = 0; g < segs.n; g++) {
        for (uint64_t i0 = 0; i0 < segs.cnt[g]; i0 += blockDim.x) {
            const uint64_t i = i0 + threadIdx.x;
            const unsigned long long v = i < segs.cnt[g] ? cnt[segs.slot[g] + i] : 0ull;
            unsigned long long x = v;   // inclusive warp scan
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) wsum[warp] = x;
            __syncthreads();
            if (warp == 0) {
                unsigned long long z = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0ull;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned long long y = __shfl_up_sync(0xffffffffu, z, o);
                    if (lane >= o) z += y;
                }
                wsum[lane] = z;   // inclusive prefix over warps
            }
            __syncthreads();
            const unsigned long long before = (warp ? wsum[warp - 1] : 0ull) + x - v;
            if (i < segs.cnt[g]) off[segs.slot[g] + i] = run + before;
            run += wsum[(blockDim.x >> 5) - 1];
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) *total = run;
}

cudaError_t launch_compact_scan(const uint32_t *cnt, uint64_t *off, const CompactSegs &segs,
                                unsigned long long *total, cudaStream_t st) {
    compact_scan_kernel<<<1, 1024, 0, st>>>(cnt, off, segs, total);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ launchers
size_t sweep_smem_extra() { return sizeof(SmemExtra); }

static void *sweep_fn(int family, int dense, int blk) {
    if (blk) {
        if (dense) return nullptr;
        switch (family) {
        case PARADL_PIPELINE:
            return blk == 1   ? (void *)sweep_kernel<PARADL_PIPELINE, 0, 1>
                   : blk == 3 ? (void *)sweep_kernel<PARADL_PIPELINE, 0, 3>
                              : (void *)sweep_kernel<PARADL_PIPELINE, 0, 2>;
        case PARADL_LAYERPURE:
            return blk == 1 ? (void *)sweep_kernel<PARADL_LAYERPURE, 0, 1> : (void *)sweep_kernel<PARADL_LAYERPURE, 0, 2>;
        case PARADL_PD:
            return blk == 1   ? (void *)sweep_kernel<PARADL_PD, 0, 1>
                   : blk == 3 ? (void *)sweep_kernel<PARADL_PD, 0, 3>
                              : (void *)sweep_kernel<PARADL_PD, 0, 2>;
        default: return nullptr;
        }
    }
#define PARADL_CASE(F)                                                                     \
    case F:                                                                                \
        return dense == 2 ? (void *)sweep_kernel<F, 2, 0>                                  \
                          : dense ? (void *)sweep_kernel<F, 1, 0> : (void *)sweep_kernel<F, 0, 0>;
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
        PARADL_CASE(PARADL_SPATIAL_AG)
        PARADL_CASE(PARADL_GPIPE)
        PARADL_CASE(PARADL_DATA_LW)
        PARADL_CASE(PARADL_LAYERWISE)
    default: return nullptr;
    }
#undef PARADL_CASE
}

// The max-dynamic-smem attribute is per function and process-wide: only ever raise it, so a
// query for a small launch cannot invalidate a later launch that needs more.
static cudaError_t ensure_smem_attr(void *fn, size_t smem) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    static struct {
        void *fn;
        size_t smem;
    } cache[64];
    static int n = 0;
    int slot = -1;
    for (int i = 0; i < n; i++)
        if (cache[i].fn == fn) slot = i;
    if (slot >= 0 && cache[slot].smem >= smem) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (slot < 0 && n < 64) slot = n++;
    if (slot >= 0) cache[slot] = {fn, smem};
    return cudaSuccess;
}

int max_blocks_per_sm(int family, int dense, int blk, size_t smem) {
    void *fn = sweep_fn(family, dense, blk);
    if (!fn) return 0;
    if (ensure_smem_attr(fn, smem) != cudaSuccess) return 0;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kThreads, smem) != cudaSuccess) return 0;
    return nb;
}

cudaError_t launch_sweep(int family, int dense, int blk, const LaunchArgs &a, int grid, size_t smem,
                         cudaStream_t st) {
    void *fn = sweep_fn(family, dense, blk);
    if (!fn) return cudaErrorInvalidValue;
    cudaError_t e = ensure_smem_attr(fn, smem);
    if (e != cudaSuccess) return e;
    void *args[] = {const_cast<LaunchArgs *>(&a)};
    return cudaLaunchKernel(fn, dim3(grid), dim3(kThreads), args, smem, st);
}

cudaError_t launch_merge(const paradl_hit *lists, int64_t n_lists, int32_t k, const unsigned long long *counts,
                         int32_t n_counts, paradl_hit *out, unsigned long long *count_out, cudaStream_t st,
                         const unsigned long long *gbound, int32_t lstride, int32_t cstride,
                         unsigned long long *bound_out, const uint32_t *nvalid, paradl_hit *lv_out,
                         uint32_t *lv_nvalid, unsigned int *lv_done) {
    const unsigned grid = lv_out ? (unsigned)((n_lists + kLevelLists - 1) / kLevelLists) : 1u;
    merge_kernel<<<grid, 1024, 0, st>>>(lists, n_lists, k, counts, n_counts, out, count_out, gbound,
                                        lstride > 0 ? lstride : k, cstride > 0 ? cstride : 1, bound_out, nvalid,
                                        lv_out, lv_nvalid, lv_done);
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
