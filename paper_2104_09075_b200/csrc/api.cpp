// api.cpp -- host side of libparadl: the C ABI of include/paradl.h.
//
// Responsibilities: input validation and overflow proofs, the canonical
// index space of a sweep (mixed radices, partition counts), packing the device image that
// the kernels stage into shared memory, launch configuration (persistent grid sized from
// the occupancy API and the SM count), and result transfer.  No cost-model arithmetic is
// done here: every Table 2 term is evaluated by the kernels in kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "paradl_internal.h"

using namespace paradl;

// NVTX ranges around every evaluating entry point (header-only NVTX v3: a no-op unless a
// profiler such as nsys / ncu --nvtx injects itself)
namespace {
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
}  // namespace

namespace {

struct HostModel {
    std::vector<paradl_layer> rows;
    int64_t D = 0;
    ModelHdr layout{};
    uint8_t *d_block = nullptr;
    // host-side bounds for overflow proofs only
    __int128 FB = 0, XY = 0, W = 0, BI = 0, Ysum = 0, Ymax = 0, Hmax = 0, WU = 0;
};

struct DevBuf {
    void *p = nullptr;
    size_t n = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= n) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) n = bytes;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// One pass of paradl_sweep_compact through run_sweep (see there)
struct CompactCall {
    int pass;                        // 1: count per tile + scan; 2: write
    const paradl_compact_out *out;
};

}  // namespace

struct paradl_ctx {
    int device = -1;
    int n_sm = 0;
    size_t smem_optin = 0;
    std::string err;
    bool have_system = false;
    paradl_system sys{};
    std::vector<HostModel> models;
    // device scratch
    DevBuf img, lists, counters, results, one, halo, stab, nvalid, lists2, nvalid2, ccnt, coff;
    std::vector<uint8_t> last_img;     // host copy of the image currently on the device
    uint64_t stat_h2d = 0, stat_d2h = 0, stat_launches = 0;
    std::vector<cudaStream_t> streams;     // internal fork streams (one per family launch)
    std::vector<cudaEvent_t> events;
    cudaEvent_t fork_ev = nullptr;
    unsigned long long *last_count_ptr = nullptr;
    uint64_t sys_epoch = 0;
    // plan cache: serialized spec of the last planned sweep and its plan (host-side only)
    std::vector<uint8_t> plan_key;
    uint64_t plan_sys_epoch = ~0ull, plan_models_epoch = ~0ull;
    void *plan_cached = nullptr;   // Plan*
    // occupancy / smem-attribute cache: (family, dense, blk, smem) -> blocks per SM
    std::vector<std::pair<uint64_t, int>> occ_cache;
    uint64_t models_epoch = 0, img_epoch = ~0ull;
};

static paradl_status fail(paradl_ctx *c, paradl_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return st;
}

#define CUDA_TRY(ctx, expr)                                                                          \
    do {                                                                                             \
        cudaError_t e_ = (expr);                                                                     \
        if (e_ != cudaSuccess) return fail(ctx, PARADL_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)

static const __int128 kLimit = (__int128)1 << 62;

// ------------------------------------------------------------------ lifecycle
extern "C" paradl_status paradl_create(int32_t cuda_device, paradl_ctx **out) {
    if (!out) return PARADL_EINVAL;
    *out = nullptr;
    paradl_ctx *c = new (std::nothrow) paradl_ctx();
    if (!c) return PARADL_ENOMEM;
    c->device = cuda_device;
    if (cuda_device >= 0) {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || cuda_device >= n) {
            delete c;
            return PARADL_ECUDA;
        }
        if (cudaSetDevice(cuda_device) != cudaSuccess) {
            delete c;
            return PARADL_ECUDA;
        }
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, cuda_device);
        c->n_sm = v;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, cuda_device);
        c->smem_optin = (size_t)v;
    }
    *out = c;
    return PARADL_OK;
}

static void free_plan(void *p);

extern "C" void paradl_destroy(paradl_ctx *c) {
    if (!c) return;
    if (c->device >= 0) {
        cudaSetDevice(c->device);
        for (auto &m : c->models)
            if (m.d_block) cudaFree(m.d_block);
        c->img.release();
        c->lists.release();
        c->counters.release();
        c->results.release();
        c->one.release();
        c->halo.release();
        c->stab.release();
        c->ccnt.release();
        c->coff.release();
        c->nvalid.release();
        c->lists2.release();
        c->nvalid2.release();
        for (auto s2 : c->streams) cudaStreamDestroy(s2);
        for (auto e2 : c->events) cudaEventDestroy(e2);
        if (c->fork_ev) cudaEventDestroy(c->fork_ev);
    }
    free_plan(c->plan_cached);
    delete c;
}

extern "C" const char *paradl_last_error(const paradl_ctx *c) { return c ? c->err.c_str() : "null ctx"; }
extern "C" const char *paradl_version(void) { return "paradl-b200 1.1 (sm_100a)"; }

extern "C" int32_t paradl_struct_size(int32_t which) {
    switch (which) {
    case 0: return (int32_t)sizeof(paradl_layer);
    case 1: return (int32_t)sizeof(paradl_system);
    case 2: return (int32_t)sizeof(paradl_subsweep);
    case 3: return (int32_t)sizeof(paradl_config);
    case 4: return (int32_t)sizeof(paradl_prediction);
    case 5: return (int32_t)sizeof(paradl_hit);
    default: return -1;
    }
}

// ------------------------------------------------------------------ model
static paradl_status validate_row(paradl_ctx *c, const paradl_layer &r, int l) {
    if (r.kind < PARADL_CONV || r.kind > PARADL_NORM) return fail(c, PARADL_EINVAL, "row %d: bad kind %d", l, r.kind);
    if (r.ndim < 1 || r.ndim > 3) return fail(c, PARADL_EINVAL, "row %d: ndim must be 1..3", l);
    if (r.C < 1 || r.F < 1 || r.C > INT32_MAX || r.F > INT32_MAX)
        return fail(c, PARADL_EINVAL, "row %d: C, F must be in [1, 2^31)", l);
    __int128 px = 1, py = 1, pk = 1;
    for (int a = 0; a < 3; a++) {
        if (r.X[a] < 1 || r.Y[a] < 1 || r.X[a] > INT32_MAX || r.Y[a] > INT32_MAX)
            return fail(c, PARADL_EINVAL, "row %d: non-positive or huge extent on axis %d", l, a);
        if (r.K[a] < 0 || r.K[a] > INT32_MAX) return fail(c, PARADL_EINVAL, "row %d: bad kernel extent", l);
        if (a >= r.ndim && (r.X[a] != 1 || r.Y[a] != 1))
            return fail(c, PARADL_EINVAL, "row %d: unused axis %d must have extent 1", l, a);
        px *= r.X[a];
        py *= r.Y[a];
        pk *= r.K[a];
    }
    if (r.x != (__int128)r.C * px) return fail(c, PARADL_EINVAL, "row %d: x != C*prod(X)", l);
    if (r.y != (__int128)r.F * py) return fail(c, PARADL_EINVAL, "row %d: y != F*prod(Y)", l);
    if (r.w < 0 || r.bi < 0 || r.fw < 0 || r.bw < 0 || r.wu < 0)
        return fail(c, PARADL_EINVAL, "row %d: negative count", l);
    const bool weighted = r.kind == PARADL_CONV || r.kind == PARADL_FC;
    if (weighted && !(r.flags & PARADL_FLAG_FOLDED) && r.w != (__int128)r.C * r.F * pk)
        return fail(c, PARADL_EINVAL, "row %d: w != C*F*prod(K) (set PARADL_FLAG_FOLDED for folded rows)", l);
    if (!weighted && r.w != 0) return fail(c, PARADL_EINVAL, "row %d: weightless kind with w != 0 (P:181)", l);
    return PARADL_OK;
}

extern "C" paradl_status paradl_load_model(paradl_ctx *c, const paradl_layer *rows, int32_t G, int64_t D,
                                           int32_t *model_id) {
    NvtxRange nvtx_("paradl_load_model");
    if (!c) return PARADL_EINVAL;
    if (!rows || G < 1 || !model_id) return fail(c, PARADL_EINVAL, "need rows, G >= 1 and model_id");
    if (G > 4096) return fail(c, PARADL_EINVAL, "G > 4096 rows is not supported");
    if (D < 1) return fail(c, PARADL_EINVAL, "dataset size D must be >= 1");
    HostModel m;
    m.rows.assign(rows, rows + G);
    m.D = D;
    for (int l = 0; l < G; l++) {
        paradl_status st = validate_row(c, rows[l], l);
        if (st) return st;
        const paradl_layer &r = rows[l];
        m.FB += (__int128)r.fw + r.bw;
        m.WU += r.wu;
        m.XY += (__int128)r.x + r.y;
        m.W += r.w;
        m.BI += r.bi;
        m.Ysum += r.y;
        m.Ymax = std::max<__int128>(m.Ymax, r.y);
        for (int a = 0; a < 3; a++) m.Hmax = std::max<__int128>(m.Hmax, r.K[a] / 2);
    }
    if (m.FB > kLimit || m.XY > kLimit || m.W > kLimit)
        return fail(c, PARADL_EOVERFLOW, "model sums exceed 2^62");
    // block layout
    ModelHdr L{};
    size_t off = sizeof(ModelHdr);
    L.off_geo = (uint32_t)off;
    off = align16(off + sizeof(RowGeo) * G);
    const size_t arr = align16(sizeof(int64_t) * (G + 1));
    L.off_pf = (uint32_t)off; off += arr;
    L.off_pb = (uint32_t)off; off += arr;
    L.off_pu = (uint32_t)off; off += arr;
    L.off_pw = (uint32_t)off; off += arr;
    L.off_pxy = (uint32_t)off; off += arr;
    L.off_pbi = (uint32_t)off; off += arr;
    L.off_y = (uint32_t)off; off += align16(sizeof(int64_t) * G);
    L.bytes = (uint32_t)off;
    L.G = G;
    L.D = D;
    m.layout = L;
    if (c->device >= 0) {
        CUDA_TRY(c, cudaSetDevice(c->device));
        paradl_layer *d_rows = nullptr;
        CUDA_TRY(c, cudaMalloc(&d_rows, sizeof(paradl_layer) * G));
        cudaError_t e = cudaMalloc(&m.d_block, L.bytes);
        if (e == cudaSuccess) e = cudaMemcpy(d_rows, rows, sizeof(paradl_layer) * G, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = launch_prep_model(d_rows, G, D, m.d_block, L, 0);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        cudaFree(d_rows);
        if (e != cudaSuccess) {
            if (m.d_block) cudaFree(m.d_block);
            return fail(c, PARADL_ECUDA, "model prep: %s", cudaGetErrorString(e));
        }
    }
    c->models.push_back(std::move(m));
    c->models_epoch++;
    *model_id = (int32_t)c->models.size() - 1;
    return PARADL_OK;
}

// ------------------------------------------------------------------ system
static bool finite_pos(double x) { return std::isfinite(x) && x > 0.0; }

extern "C" paradl_status paradl_set_system(paradl_ctx *c, const paradl_system *s) {
    if (!c) return PARADL_EINVAL;
    if (!s) return fail(c, PARADL_EINVAL, "null system");
    if (s->n_tiers < 1 || s->n_tiers > PARADL_MAX_TIERS) return fail(c, PARADL_EINVAL, "n_tiers must be 1..%d", PARADL_MAX_TIERS);
    for (int t = 0; t < s->n_tiers; t++) {
        if (s->tiers[t].max_pes < 1 || (t > 0 && s->tiers[t].max_pes <= s->tiers[t - 1].max_pes))
            return fail(c, PARADL_EINVAL, "tier max_pes must be >= 1 and strictly increasing");
        if (!(std::isfinite(s->tiers[t].alpha_s) && s->tiers[t].alpha_s >= 0.0) || !finite_pos(s->tiers[t].beta_s_per_B))
            return fail(c, PARADL_EINVAL, "tier %d: need alpha >= 0 and beta > 0", t);
    }
    if (s->delta != 2 && s->delta != 4 && s->delta != 8) return fail(c, PARADL_EINVAL, "delta must be 2, 4 or 8");
    if (!finite_pos(s->flops_per_s) || !finite_pos(s->hbm_bytes)) return fail(c, PARADL_EINVAL, "R and capacity must be > 0");
    if (!(s->gamma > 0.0 && s->gamma <= 1.0)) return fail(c, PARADL_EINVAL, "gamma must be in (0,1]");
    if (!(std::isfinite(s->phi_df) && s->phi_df >= 1.0)) return fail(c, PARADL_EINVAL, "phi_df must be >= 1");
    if (!(std::isfinite(s->tree_threshold_B) && s->tree_threshold_B >= 0.0) || s->tree_chunks < 1)
        return fail(c, PARADL_EINVAL, "tree_threshold >= 0 and tree_chunks >= 1 required");
    if (s->filter_rs != 0 && s->filter_rs != 1) return fail(c, PARADL_EINVAL, "filter_rs must be 0 or 1");
    if (!finite_pos(s->p2p_alpha_scale) || !finite_pos(s->p2p_beta_scale))
        return fail(c, PARADL_EINVAL, "p2p scales must be > 0");
    if (!(std::isfinite(s->phi_pd) && s->phi_pd >= 1.0) || !(std::isfinite(s->phi_ds) && s->phi_ds >= 1.0))
        return fail(c, PARADL_EINVAL, "phi_pd and phi_ds must be >= 1");
    c->sys = *s;
    c->have_system = true;
    c->img_epoch = ~0ull;
    c->sys_epoch++;
    return PARADL_OK;
}

// ------------------------------------------------------------------ sweep planning
namespace {

struct SubPlan {
    SubHdr hdr{};
    int family = 0, model = 0;   // model = ctx model id
    int64_t bmax = 0;            // largest batch value
    bool dims0_pow2 = true;      // every dims[0] value a power of two
};

struct Plan {
    std::vector<SubPlan> subs;
    std::vector<int> model_ids;   // image model index -> ctx model id
    uint64_t total = 0;
    std::vector<uint8_t> image;   // host image without model blocks (blocks appended on device)
    uint32_t bytes = 0;           // total image bytes incl. model blocks
};

uint64_t binom_u64(int64_t n, int64_t k) {
    if (k < 0 || k > n) return 0;
    if (k > n - k) k = n - k;
    unsigned __int128 r = 1;
    for (int64_t i = 1; i <= k; i++) r = r * (unsigned __int128)(n - k + i) / (unsigned __int128)i;
    return (uint64_t)r;
}

}  // namespace

// A/B switch for experiments: PARADL_NO_MERGE_LEVEL=1 merges all CTA lists in one block
static bool merge_level_off() {
    static const bool off = [] {
        const char *e = getenv("PARADL_NO_MERGE_LEVEL");
        return e && e[0] == '1';
    }();
    return off;
}

// A/B switch for experiments: PARADL_NO_COMB=1 keeps COMB pipeline / pd sweeps on mode 1
// (tile_body_blocked) instead of mode 3 (tile_body_comb); same results
static bool comb_off() {
    static const bool off = getenv("PARADL_NO_COMB") != nullptr;
    return off;
}
// A/B switch for experiments: PARADL_NO_MASKS=1 keeps screened mask blocks on the unsorted table
static bool masks_off() {
    static const bool off = getenv("PARADL_NO_MASKS") != nullptr;
    return off;
}
// A/B switch for experiments: PARADL_NO_STRUCT_TABLE=1 recomputes pipeline structure terms
// inside the sweep kernel instead of reading the structure table (same results)
static bool struct_table_off() {
    static const bool off = [] {
        const char *e = getenv("PARADL_NO_STRUCT_TABLE");
        return e && e[0] == '1';
    }();
    return off;
}

static paradl_status plan_sweep_build(paradl_ctx *c, const paradl_sweep_spec *spec, Plan &P) {
    if (!spec || spec->n_sub < 1 || !spec->sub) return fail(c, PARADL_EINVAL, "empty sweep spec");
    if (spec->n_sub > kMaxSub) return fail(c, PARADL_EINVAL, "at most %d sub-sweeps", kMaxSub);
    if (!c->have_system) return fail(c, PARADL_ESTATE, "paradl_set_system not called");
    const paradl_system &sy = c->sys;
    const int NT = sy.n_tiers;
    // image tiers: the collective tiers, plus their point-to-point copies when the p2p
    // scales are not 1 (Q40; one IEEE product per value, the oracle forms the same product)
    const int NTI = (sy.p2p_alpha_scale != 1.0 || sy.p2p_beta_scale != 1.0) ? 2 * NT : NT;
    // value tables are appended after the headers
    std::vector<uint8_t> tab;
    auto put = [&](const void *src, size_t bytes) -> uint32_t {
        size_t off = align16(tab.size());
        tab.resize(off + align16(bytes ? bytes : 8), 0);
        if (bytes) memcpy(tab.data() + off, src, bytes);
        return (uint32_t)off;
    };
    unsigned __int128 total = 0;
    for (int i = 0; i < spec->n_sub; i++) {
        const paradl_subsweep &s = spec->sub[i];
        SubPlan sp;
        SubHdr &h = sp.hdr;
        if (s.family < 0 || s.family >= PARADL_N_FAMILIES) return fail(c, PARADL_EINVAL, "sub %d: bad family", i);
        if (s.model_id < 0 || s.model_id >= (int)c->models.size())
            return fail(c, PARADL_ESTATE, "sub %d: unknown model id %d", i, s.model_id);
        const HostModel &m = c->models[s.model_id];
        const int G = (int)m.rows.size();
        const int fam = s.family;
        const bool pipe = fam == PARADL_PIPELINE || fam == PARADL_LAYERPURE || fam == PARADL_PD || fam == PARADL_GPIPE;
        const bool spatial = fam == PARADL_SPATIAL || fam == PARADL_DS || fam == PARADL_SPATIAL_AG;
        if (s.n_cap < 0 || s.n_flops < 0 || s.n_b < 1 || s.n_S < 0 || s.n_dims < 0 || s.n_Ls < 0 || s.n_alpha < 0 ||
            s.n_beta < 0)
            return fail(c, PARADL_EINVAL, "sub %d: negative list length or empty b list", i);
        if ((s.n_cap && !s.cap) || (s.n_flops && !s.flops) || !s.b || (s.n_S && !s.S) || (s.n_dims && !s.dims) ||
            (s.n_Ls && !s.Ls) || (s.n_alpha && !s.alpha) || (s.n_beta && !s.beta))
            return fail(c, PARADL_EINVAL, "sub %d: null list pointer", i);
        if (spatial && s.n_Ls < 1) return fail(c, PARADL_EINVAL, "sub %d: spatial families need an Ls list", i);
        // materialise every list (defaults for empty ones)
        std::vector<double> cap(s.cap, s.cap + s.n_cap), fl(s.flops, s.flops + s.n_flops);
        if (cap.empty()) cap.push_back(sy.hbm_bytes);
        if (fl.empty()) fl.push_back(sy.flops_per_s);
        for (double v : cap) if (!finite_pos(v)) return fail(c, PARADL_EINVAL, "sub %d: capacity must be > 0", i);
        for (double v : fl) if (!finite_pos(v)) return fail(c, PARADL_EINVAL, "sub %d: flops must be > 0", i);
        std::vector<int64_t> bl(s.b, s.b + s.n_b);
        int64_t bmax = 0;
        for (int64_t v : bl) {
            if (v < 1 || v > ((int64_t)1 << 40)) return fail(c, PARADL_EINVAL, "sub %d: batch out of range", i);
            bmax = std::max(bmax, v);
        }
        std::vector<int32_t> Sl(s.S, s.S + s.n_S);
        if (Sl.empty()) Sl.push_back(1);
        for (int32_t v : Sl) if (v < 1) return fail(c, PARADL_EINVAL, "sub %d: S must be >= 1", i);
        std::vector<int32_t> dl(s.dims, s.dims + 4 * (size_t)s.n_dims);
        if (dl.empty()) dl = {1, 1, 1, 1};
        int64_t degmax = 1, pmax = 1;
        for (size_t j = 0; j < dl.size(); j += 4) {
            const int32_t *d = &dl[j];
            for (int a = 0; a < 4; a++)
                if (d[a] < 1 || d[a] > (1 << 24)) return fail(c, PARADL_EINVAL, "sub %d: dims must be in [1, 2^24]", i);
            bool ok = true;
            switch (fam) {
            case PARADL_SERIAL: case PARADL_PIPELINE: case PARADL_LAYERPURE: case PARADL_GPIPE:
                ok = d[0] == 1 && d[1] == 1 && d[2] == 1 && d[3] == 1; break;
            case PARADL_DATA: case PARADL_FILTER: case PARADL_CHANNEL: case PARADL_PD: case PARADL_DATA_LW:
            case PARADL_LAYERWISE:
                ok = d[1] == 1 && d[2] == 1 && d[3] == 1; break;
            case PARADL_DF: ok = d[2] == 1 && d[3] == 1; break;
            case PARADL_SPATIAL: case PARADL_SPATIAL_AG: ok = d[0] == 1; break;
            default: break;
            }
            if (!ok) return fail(c, PARADL_EINVAL, "sub %d: dims tuple does not fit the family", i);
            const int64_t deg = (fam == PARADL_DATA || fam == PARADL_DF || fam == PARADL_DS || fam == PARADL_PD ||
                                 fam == PARADL_DATA_LW || fam == PARADL_LAYERWISE)
                                    ? d[0]
                                    : 1;
            degmax = std::max(degmax, deg);
            sp.dims0_pow2 = sp.dims0_pow2 && (d[0] & (d[0] - 1)) == 0;
            pmax = std::max<int64_t>(pmax, (int64_t)d[0] * d[1] * d[2] * d[3]);
        }
        std::vector<int32_t> Ll(s.Ls, s.Ls + s.n_Ls);
        if (Ll.empty()) Ll.push_back(0);
        for (int32_t v : Ll) if (v < 0) return fail(c, PARADL_EINVAL, "sub %d: Ls must be >= 0", i);
        if (fam == PARADL_SPATIAL_AG)
            for (int32_t v : Ll) if (v < 1) return fail(c, PARADL_EINVAL, "sub %d: spatial_ag needs Ls >= 1", i);
        std::vector<double> al, be;
        if (s.n_alpha) al.assign(s.alpha, s.alpha + (size_t)s.n_alpha * NT);
        else for (int t = 0; t < NT; t++) al.push_back(sy.tiers[t].alpha_s);
        if (s.n_beta) be.assign(s.beta, s.beta + (size_t)s.n_beta * NT);
        else for (int t = 0; t < NT; t++) be.push_back(sy.tiers[t].beta_s_per_B);
        for (double v : al) if (!(std::isfinite(v) && v >= 0.0)) return fail(c, PARADL_EINVAL, "sub %d: alpha must be >= 0", i);
        for (double v : be) if (!finite_pos(v)) return fail(c, PARADL_EINVAL, "sub %d: beta must be > 0", i);
        if (NTI != NT) {
            // point-to-point copies of every row (Q40): [the NT tier values | each x its p2p scale]
            std::vector<double> al2, be2;
            for (size_t r = 0; r < al.size() / NT; r++) {
                for (int t = 0; t < NT; t++) al2.push_back(al[r * NT + t]);
                for (int t = 0; t < NT; t++) al2.push_back(al[r * NT + t] * sy.p2p_alpha_scale);
            }
            for (size_t r = 0; r < be.size() / NT; r++) {
                for (int t = 0; t < NT; t++) be2.push_back(be[r * NT + t]);
                for (int t = 0; t < NT; t++) be2.push_back(be[r * NT + t] * sy.p2p_beta_scale);
            }
            al.swap(al2);
            be.swap(be2);
        }
        // partition radix
        uint64_t part_n = 1;
        h.part_mode = s.part_mode;
        h.s_min = h.s_max = 1;
        std::vector<uint64_t> sblk, binom;
        if (fam == PARADL_LAYERWISE) {
            // one strategy bit per COMM row (Q39)
            if (s.part_mode != PARADL_PART_MASK) return fail(c, PARADL_EINVAL, "sub %d: layerwise needs the mask partition mode", i);
            int nc = 0;
            for (const auto &r : m.rows) nc += (r.flags & PARADL_FLAG_COMM) != 0;
            if (nc > 62) return fail(c, PARADL_EINVAL, "sub %d: layerwise needs at most 62 COMM rows", i);
            part_n = (uint64_t)1 << nc;
        } else if (!pipe) {
            if (s.part_mode != PARADL_PART_NONE) return fail(c, PARADL_EINVAL, "sub %d: partition mode on a non-pipeline family", i);
        } else if (s.part_mode == PARADL_PART_MASK) {
            if (G > 64) return fail(c, PARADL_EINVAL, "sub %d: mask mode needs G <= 64", i);
            if (fam == PARADL_GPIPE && G > PARADL_GPIPE_MAX_STAGES)
                return fail(c, PARADL_EINVAL, "sub %d: gpipe mask mode needs G <= %d", i, PARADL_GPIPE_MAX_STAGES);
            part_n = (uint64_t)1 << (G - 1);
            h.s_min = 1;
            h.s_max = G;
        } else if (s.part_mode == PARADL_PART_COMB) {
            if (s.s_min < 1 || s.s_max < s.s_min || s.s_max > G) return fail(c, PARADL_EINVAL, "sub %d: need 1 <= s_min <= s_max <= G", i);
            if (s.s_max - 1 > kMaxCuts) return fail(c, PARADL_EINVAL, "sub %d: combination mode supports s_max <= %d", i, kMaxCuts + 1);
            if (fam == PARADL_GPIPE && s.s_max > PARADL_GPIPE_MAX_STAGES)
                return fail(c, PARADL_EINVAL, "sub %d: gpipe supports s_max <= %d", i, PARADL_GPIPE_MAX_STAGES);
            h.s_min = s.s_min;
            h.s_max = s.s_max;
            h.kmax = s.s_max - 1;
            unsigned __int128 acc = 0;
            sblk.push_back(0);
            for (int st = s.s_min; st <= s.s_max; st++) {
                acc += binom_u64(G - 1, st - 1);
                if (acc >> 63) return fail(c, PARADL_EOVERFLOW, "sub %d: too many partitions", i);
                sblk.push_back((uint64_t)acc);
            }
            part_n = (uint64_t)acc;
            h.binom_stride = h.kmax + 1;
            binom.resize((size_t)G * h.binom_stride);
            for (int n = 0; n < G; n++)
                for (int j = 0; j <= h.kmax; j++) binom[(size_t)n * h.binom_stride + j] = binom_u64(n, j);
        } else {
            return fail(c, PARADL_EINVAL, "sub %d: pipeline families need a partition mode", i);
        }
        // overflow proofs for every int64 intermediate of the kernels
        {
            const __int128 B = (__int128)bmax * degmax, dl_ = sy.delta;
            const __int128 hv = 6 * m.Hmax * m.XY;
            const __int128 terms[] = {B * m.FB, 2 * B * m.XY, B * dl_ * m.Ysum, (__int128)bmax * dl_ * hv,
                                      dl_ * m.W, 2 * (__int128)bmax * m.XY + 2 * m.W + m.BI,
                                      2 * dl_ * (__int128)bmax * m.Ysum, (__int128)m.D};
            for (__int128 t : terms)
                if (t < 0 || t >= kLimit) return fail(c, PARADL_EOVERFLOW, "sub %d: an int64 intermediate may exceed 2^62", i);
            if (pmax > ((int64_t)1 << 40)) return fail(c, PARADL_EOVERFLOW, "sub %d: PE count too large", i);
        }
        // image model index
        int mi = -1;
        for (size_t q = 0; q < P.model_ids.size(); q++)
            if (P.model_ids[q] == s.model_id) mi = (int)q;
        if (mi < 0) {
            if ((int)P.model_ids.size() >= kMaxModelsPerSweep) return fail(c, PARADL_EINVAL, "at most %d models per sweep", kMaxModelsPerSweep);
            P.model_ids.push_back(s.model_id);
            mi = (int)P.model_ids.size() - 1;
        }
        h.family = fam;
        h.model = mi;
        h.G = G;
        h.radix[D_BETA] = (uint32_t)(be.size() / NTI);
        h.radix[D_ALPHA] = (uint32_t)(al.size() / NTI);
        h.radix[D_LS] = (uint32_t)Ll.size();
        h.radix[D_DIMS] = (uint32_t)(dl.size() / 4);
        h.radix[D_S] = (uint32_t)Sl.size();
        h.radix[D_PART] = 0;
        h.radix[D_B] = (uint32_t)bl.size();
        h.radix[D_FLOPS] = (uint32_t)fl.size();
        h.radix[D_CAP] = (uint32_t)cap.size();
        h.part_n = part_n;
        if (spatial && (uint64_t)h.radix[D_DIMS] * h.radix[D_LS] >= (1ull << 24))
            return fail(c, PARADL_EINVAL, "sub %d: n_dims * n_Ls must be < 2^24 for spatial families", i);
        if ((uint64_t)h.radix[D_ALPHA] * h.radix[D_BETA] >= (1ull << 31))
            return fail(c, PARADL_EINVAL, "sub %d: n_alpha * n_beta must be < 2^31", i);
        unsigned __int128 cnt = part_n;
        for (int d = 0; d < kDigits; d++)
            if (d != D_PART) cnt *= h.radix[d];
        if (cnt >> 63) return fail(c, PARADL_EOVERFLOW, "sub %d: more than 2^63 configurations", i);
        h.count = (uint64_t)cnt;
        h.offset = (uint64_t)total;
        total += cnt;
        if (total >> 63) return fail(c, PARADL_EOVERFLOW, "sweep larger than 2^63 configurations");
        h.off_cap = put(cap.data(), cap.size() * 8);
        h.off_flops = put(fl.data(), fl.size() * 8);
        h.off_b = put(bl.data(), bl.size() * 8);
        h.off_S = put(Sl.data(), Sl.size() * 4);
        h.off_dims = put(dl.data(), dl.size() * 4);
        h.off_Ls = put(Ll.data(), Ll.size() * 4);
        h.off_alpha = put(al.data(), al.size() * 8);
        h.off_beta = put(be.data(), be.size() * 8);
        h.off_binom = put(binom.data(), binom.size() * 8);
        h.off_sblk = put(sblk.data(), sblk.size() * 8);
        sp.family = fam;
        sp.model = s.model_id;
        sp.bmax = bmax;
        P.subs.push_back(sp);
    }
    P.total = (uint64_t)total;
    // assemble: [ImgHdr][SubHdr...][tables][model blocks]
    const size_t hdr_bytes = sizeof(ImgHdr) + sizeof(SubHdr) * P.subs.size();
    ImgHdr H{};
    H.n_sub = (int32_t)P.subs.size();
    H.n_models = (int32_t)P.model_ids.size();
    H.n_tiers = NTI;
    H.n_ctiers = NT;
    H.p2p_off = NTI == NT ? 0 : NT;
    H.phi_pd = sy.phi_pd;
    H.phi_ds = sy.phi_ds;
    H.delta = sy.delta;
    H.tree_chunks = sy.tree_chunks;
    H.ar_mult = sy.filter_rs ? 1.0 : 2.0;
    H.gamma = sy.gamma;
    H.phi_df = sy.phi_df;
    H.tree_thr = sy.tree_threshold_B;
    for (int t = 0; t < PARADL_MAX_TIERS; t++) H.max_pes[t] = t < NT ? sy.tiers[t].max_pes : 0;
    size_t off = align16(hdr_bytes + tab.size());
    for (size_t q = 0; q < P.model_ids.size(); q++) {
        H.model_off[q] = (uint32_t)off;
        off += align16(c->models[P.model_ids[q]].layout.bytes);
    }
    if (off > 0xffffffffu) return fail(c, PARADL_ENOMEM, "image too large");
    P.bytes = (uint32_t)off;
    H.bytes = P.bytes;
    for (size_t q = 0; q < P.subs.size(); q++) {
        H.sub_off[q] = (uint32_t)(sizeof(ImgHdr) + sizeof(SubHdr) * q);
        SubHdr &h = P.subs[q].hdr;
        for (uint32_t *o : {&h.off_cap, &h.off_flops, &h.off_b, &h.off_S, &h.off_dims, &h.off_Ls, &h.off_alpha,
                            &h.off_beta, &h.off_binom, &h.off_sblk})
            *o += (uint32_t)hdr_bytes;
    }
    P.image.assign(align16(hdr_bytes + tab.size()), 0);
    memcpy(P.image.data(), &H, sizeof H);
    for (size_t q = 0; q < P.subs.size(); q++)
        memcpy(P.image.data() + sizeof(ImgHdr) + sizeof(SubHdr) * q, &P.subs[q].hdr, sizeof(SubHdr));
    memcpy(P.image.data() + hdr_bytes, tab.data(), tab.size());
    return PARADL_OK;
}

static void free_plan(void *p) { delete (Plan *)p; }

// Serialises every input a plan depends on (spec fields and list contents).
static void spec_key(const paradl_sweep_spec *spec, int NT, std::vector<uint8_t> &k) {
    k.clear();
    auto app = [&](const void *p, size_t n) {
        const uint8_t *b = (const uint8_t *)p;
        k.insert(k.end(), b, b + n);
    };
    app(&spec->n_sub, sizeof spec->n_sub);
    for (int i = 0; i < spec->n_sub; i++) {
        const paradl_subsweep &x = spec->sub[i];
        app(&x.family, 14 * sizeof(int32_t));   // family .. reserved (scalar header)
        if (x.n_cap > 0 && x.cap) app(x.cap, 8ull * x.n_cap);
        if (x.n_flops > 0 && x.flops) app(x.flops, 8ull * x.n_flops);
        if (x.n_b > 0 && x.b) app(x.b, 8ull * x.n_b);
        if (x.n_S > 0 && x.S) app(x.S, 4ull * x.n_S);
        if (x.n_dims > 0 && x.dims) app(x.dims, 16ull * x.n_dims);
        if (x.n_Ls > 0 && x.Ls) app(x.Ls, 4ull * x.n_Ls);
        if (x.n_alpha > 0 && x.alpha) app(x.alpha, 8ull * x.n_alpha * NT);
        if (x.n_beta > 0 && x.beta) app(x.beta, 8ull * x.n_beta * NT);
    }
}

// Plans the sweep into the ctx-owned plan, reusing it when the spec, system and models are
// unchanged (the bench and multi-GPU steps call the same sweep repeatedly).  *out stays
// valid until the next planning call on this ctx.
static paradl_status plan_sweep(paradl_ctx *c, const paradl_sweep_spec *spec, const Plan **out) {
    Plan *cached = (Plan *)c->plan_cached;
    if (!cached) {
        cached = new (std::nothrow) Plan();
        if (!cached) return fail(c, PARADL_ENOMEM, "out of host memory");
        c->plan_cached = cached;
    }
    std::vector<uint8_t> key;
    const bool keyable = spec && spec->n_sub >= 1 && spec->sub && spec->n_sub <= kMaxSub && c->have_system;
    if (keyable) {
        spec_key(spec, c->sys.n_tiers, key);
        if (c->plan_sys_epoch == c->sys_epoch && c->plan_models_epoch == c->models_epoch && key == c->plan_key) {
            *out = cached;
            return PARADL_OK;
        }
    }
    c->plan_sys_epoch = ~0ull;   // invalid until rebuilt successfully
    *cached = Plan();
    paradl_status st = plan_sweep_build(c, spec, *cached);
    if (st) return st;
    if (keyable) {
        c->plan_key.swap(key);
        c->plan_sys_epoch = c->sys_epoch;
        c->plan_models_epoch = c->models_epoch;
    }
    *out = cached;
    return PARADL_OK;
}

static paradl_status need_device(paradl_ctx *c) {
    if (!c) return PARADL_EINVAL;
    c->stat_h2d = c->stat_d2h = c->stat_launches = 0;
    if (c->device < 0) return fail(c, PARADL_ESTATE, "host-only context: no CUDA device (no CPU fallback exists)");
    if (cudaSetDevice(c->device) != cudaSuccess) return fail(c, PARADL_ECUDA, "cudaSetDevice failed");
    return PARADL_OK;
}

// Uploads the image (skipped when identical to the one already on the device).
static paradl_status upload(paradl_ctx *c, const Plan &P, cudaStream_t st) {
    if (P.bytes + sweep_smem_extra() > c->smem_optin)
        return fail(c, PARADL_ENOMEM, "sweep image of %u bytes does not fit shared memory (%zu available)", P.bytes,
                    c->smem_optin - sweep_smem_extra());
    bool same = c->img_epoch == c->models_epoch && c->last_img == P.image && c->img.n >= P.bytes;
    if (same) return PARADL_OK;
    CUDA_TRY(c, c->img.ensure(P.bytes));
    uint8_t *d = (uint8_t *)c->img.p;
    CUDA_TRY(c, cudaMemcpyAsync(d, P.image.data(), P.image.size(), cudaMemcpyHostToDevice, st));
    c->stat_h2d += P.image.size();
    const ImgHdr *H = reinterpret_cast<const ImgHdr *>(P.image.data());
    for (size_t q = 0; q < P.model_ids.size(); q++) {
        const HostModel &m = c->models[P.model_ids[q]];
        CUDA_TRY(c, cudaMemcpyAsync(d + H->model_off[q], m.d_block, m.layout.bytes, cudaMemcpyDeviceToDevice, st));
    }
    c->last_img = P.image;
    c->img_epoch = c->models_epoch;
    return PARADL_OK;
}

extern "C" paradl_status paradl_sweep_size(paradl_ctx *c, const paradl_sweep_spec *spec, uint64_t *n) {
    if (!c || !n) return PARADL_EINVAL;
    const Plan *PP = nullptr;
    paradl_status st = plan_sweep(c, spec, &PP);
    if (st) return st;
    const Plan &P = *PP;
    *n = P.total;
    return PARADL_OK;
}

// mixed-radix digits of the lane stride 32 for one sub-sweep
static void stride_digits(const SubHdr &h, WorkItem &a) {
    uint64_t rem = 32;
    a.inc_top = -1;
    for (int d = 0; d < kDigits; d++) {
        if (d == D_PART) {
            a.inc_part = rem % h.part_n;
            rem /= h.part_n;
            if (a.inc_part) a.inc_top = d;
        } else {
            a.inc[d] = (uint32_t)(rem % h.radix[d]);
            rem /= h.radix[d];
            if (a.inc[d]) a.inc_top = d;
        }
    }
}

// Launches the sweep for every sub-sweep intersecting [first, first+count): one persistent
// launch per strategy family (its work items share a tile queue), all forked onto internal
// streams so that small latency-bound families overlap each other and the big ones; the
// caller's stream then waits for all of them.  Per-CTA top-k lists land contiguously in
// c->lists (reduce mode); *n_lists_out = total CTAs.
static paradl_status run_sweep(paradl_ctx *c, const Plan &P, uint64_t first, uint64_t count, int shard, int n_shards,
                               bool dense, int k, const paradl_dense_out *out, cudaStream_t st, int *n_lists_out,
                               const CompactCall *cmp = nullptr) {
    const size_t smem = P.bytes + sweep_smem_extra();
    std::vector<LaunchArgs> L;
    std::vector<int> fam_of;
    HaloJobs hj{};
    hj.img = (const uint8_t *)c->img.p;
    size_t halo_entries = 0;
    if (n_lists_out) *n_lists_out = 0;
    for (size_t q = 0; q < P.subs.size(); q++) {
        const SubHdr &h = P.subs[q].hdr;
        const uint64_t s0 = h.offset, s1 = h.offset + h.count;
        const uint64_t r0 = std::max(s0, first), r1 = std::min(s1, first + count);
        if (r0 >= r1) continue;
        const int fam = P.subs[q].family;
        size_t li = 0;
        while (li < fam_of.size() && (fam_of[li] != fam || L[li].n_work + 3 > kMaxWork)) li++;
        if (li == fam_of.size()) {
            fam_of.push_back(fam);
            L.emplace_back();
            memset(&L.back(), 0, sizeof(LaunchArgs));
        }
        LaunchArgs &a = L[li];
        // lane-blocked modes for pipeline families with a small alpha/beta block (reduce mode):
        // the block-aligned middle of the range is mode 1 (COMB, or MASK with G < 10) or mode 2
        // (MASK, 256-mask blocks with the low-bit table); ragged ends stay mode 0
        const bool pipe = fam == PARADL_PIPELINE || fam == PARADL_LAYERPURE || fam == PARADL_PD;
        const uint64_t nAB = (uint64_t)h.radix[D_ALPHA] * h.radix[D_BETA];
        const uint64_t Q = nAB * h.radix[D_LS] * h.radix[D_DIMS] * h.radix[D_S];
        // memo: [n_b][n_S + n_dims] doubles; pd adds the ring GE table by (s, dims):
        // [n_s][n_dims + 1] doubles (ge_c) + as many int32 (tier), n_s = max stage count + 1
        const uint64_t n_stage = (h.part_mode == PARADL_PART_COMB ? (uint64_t)h.s_max : (uint64_t)h.G) + 1;
        const uint64_t ctab_n = fam == PARADL_PD ? n_stage * (h.radix[D_DIMS] + 1) : 0;
        const bool mask2 = h.part_mode == PARADL_PART_MASK && h.G >= 10 && h.radix[D_B] <= 2;
        // screened pipeline masks: per (b, stage count n <= 64) {cseg, pp_c, alpha, beta} (NTab)
        const uint64_t maskd_n = (mask2 && fam == PARADL_PIPELINE && Q == 1) ? h.radix[D_B] * 4ull * kMaskTabN : 0;
        const uint64_t memo_n =
            (uint64_t)h.radix[D_B] * (h.radix[D_S] + h.radix[D_DIMS]) + ctab_n + (ctab_n + 1) / 2 + maskd_n;
        int mode = (!dense && pipe && nAB < 32 && memo_n <= 2048 && Q < (1ull << 22))
                       ? (mask2 ? 2 : 1)
                       : 0;
        // mode 3 (tile_body_comb): COMB pipeline / pd with ring collectives and <= 2 x 2
        // alpha/beta rows -- incremental stage terms, per-(b, s, S) / (b, s, dims) tables
        const uint64_t ns1 = (uint64_t)h.s_max + 1;
        // CmbS rows padded to whole passes of 4 S values (kSB in kernels.cu)
        const uint64_t cmb_bytes =
            ns1 * 48 + (uint64_t)h.radix[D_B] * ns1 * ((h.radix[D_S] + 3) / 4 * 4 * 32ull + h.radix[D_DIMS] * 64ull) +
            8ull * (h.radix[D_FLOPS] + h.radix[D_CAP]);   // + tau per flops value, memory threshold per cap
        if (mode == 1 && h.part_mode == PARADL_PART_COMB && (fam == PARADL_PIPELINE || fam == PARADL_PD) &&
            (fam == PARADL_PIPELINE || c->sys.tree_threshold_B <= 0.0) && h.radix[D_ALPHA] <= 2 &&
            h.radix[D_BETA] <= 2 && cmb_bytes <= (32u << 10) && !comb_off() &&
            (uint64_t)h.radix[D_S] * h.radix[D_DIMS] * h.radix[D_LS] * h.radix[D_ALPHA] * h.radix[D_BETA] < (1ull << 31) &&
            smem + kLaneStateBytes + cmb_bytes + memo_n * sizeof(double) + 1024 <= c->smem_optin)
            mode = 3;
        // screened masks hold every stage quantity as an exact double: the model totals bound
        // each stage term, so they must stay below 2^53 (kWorkMaskD)
        bool maskd_ok = false;
        if (mode == 2 && maskd_n) {
            const HostModel &hm = c->models[P.subs[q].model];
            const __int128 lim = (__int128)1 << 53;
            const __int128 memb = 2 * (__int128)P.subs[q].bmax * hm.XY + 2 * hm.W + hm.BI;
            maskd_ok = hm.FB < lim && hm.WU < lim && memb < lim && (__int128)c->sys.delta * hm.Ymax < lim;
        }
        // sorted 512-mask blocks (kWorkMaskS, tile_body_mask_s): one flops value, <= 4 tiers
        const bool masks_ok =
            maskd_ok && h.radix[D_FLOPS] == 1 && h.radix[D_CAP] == 1 && c->sys.n_tiers <= 4 && !masks_off();
        const int low_bits = masks_ok ? kLowBitsSorted : 8;
        const uint64_t unit = mode == 2 ? Q << low_bits : Q;
        const uint64_t lo = r0 - s0, hi = r1 - s0;
        uint64_t b0 = lo, b1 = lo;   // [b0, b1): blocked part
        if (mode) {
            b0 = (lo + unit - 1) / unit * unit;
            b1 = hi / unit * unit;
            if (b1 <= b0) b0 = b1 = lo;
        }
        const uint64_t parts[3][2] = {{lo, b0}, {b0, b1}, {b1, hi}};
        for (int pi = 0; pi < 3; pi++) {
            if (pi == 0 && b1 == b0) {   // whole range in mode 0
                WorkItem &w = a.work[a.n_work++];
                w.sub = (int32_t)q;
                w.family = fam;
                w.lo = lo;
                w.hi = hi;
                stride_digits(h, w);
                break;
            }
            if (parts[pi][0] >= parts[pi][1]) continue;
            WorkItem &w = a.work[a.n_work++];
            w.sub = (int32_t)q;
            w.family = fam;
            w.lo = parts[pi][0];
            w.hi = parts[pi][1];
            if (pi == 1) {
                w.mode = mode;
                memset(w.inc, 0, sizeof w.inc);
                w.inc_part = mode == 2 ? (1ull << low_bits) : 1;
                w.inc_top = D_PART;
                w.memo_n = (uint32_t)memo_n;
                w.memo_off = a.memo_bytes;
                a.memo_bytes += (uint32_t)align16(memo_n * sizeof(double));
                if (mode == 3) {
                    w.cmb_off = a.memo_bytes;
                    a.memo_bytes += (uint32_t)align16(cmb_bytes);
                    if (fam != PARADL_PD || P.subs[q].dims0_pow2) w.flags |= kWorkPow2;
                }
                if (mode == 1 && (fam == PARADL_PIPELINE || fam == PARADL_PD)) {
                    // screened path: per-lane dims table (ge_c, ge_s fp64 + ge_t u8) per thread
                    const uint32_t nD = h.radix[D_DIMS];
                    const uint32_t tb = (uint32_t)align16((size_t)nD * 8u * kThreads);
                    if (tb <= kMaxDtabBytes) a.dtab_bytes = std::max(a.dtab_bytes, tb);
                }
                if (maskd_ok) w.flags |= kWorkMaskD;
                if (masks_ok) w.flags |= kWorkMaskS;
                if (mode == 2) {
                    w.low_off = a.low_bytes / 64;
                    // 64-byte entries per b: LowE / LowD over 256 low masks, or (kWorkMaskS) the
                    // sorted LowS table over 512 followed by its per-(b, e, pop) feasible counts
                    a.low_bytes += h.radix[D_B] * (1u << low_bits) * 64u +
                                   // (whole 64-byte units: low_off counts them)
                                   (masks_ok ? (h.radix[D_B] * (kLowBitsSorted + 1) * (kLowBitsSorted + 2) * 4u + 63u) & ~63u : 0u);
                }
            } else {
                stride_digits(h, w);
            }
        }
        if (fam == PARADL_DATA_LW) {
            // per-layer Allreduce coefficients (c_l, s_l) per dims value, built in shared memory
            // by every CTA (build_memo): [n_dims][weighted rows][2] doubles
            const HostModel &hm = c->models[P.subs[q].model];
            uint32_t lw = 0;
            for (const auto &r : hm.rows) lw += r.w > 0;
            const uint64_t n = (uint64_t)h.radix[D_DIMS] * lw * 2;
            if (n * sizeof(double) > (64u << 10)) return fail(c, PARADL_EINVAL, "sub %d: data_lw table (dims x weighted layers) exceeds 64 KB", (int)q);
            for (int i = 0; i < a.n_work; i++) {
                WorkItem &w = a.work[i];
                if (w.sub != (int32_t)q || w.memo_n) continue;
                w.memo_n = (uint32_t)n;
                w.memo_off = a.memo_bytes;
                a.memo_bytes += (uint32_t)align16(n * sizeof(double));
            }
        }
        if (fam == PARADL_GPIPE) {
            // per-lane stage table (f, g, m, u per stage) of the GPipe schedule evaluation
            a.dtab_bytes = std::max<uint32_t>(a.dtab_bytes, kGpipeTabBytes);
        }
        if (fam == PARADL_SPATIAL || fam == PARADL_DS || fam == PARADL_SPATIAL_AG) {
            HaloJob &j = hj.job[hj.n_jobs++];
            j.sub = (int32_t)q;
            j.n_entries = (int32_t)(h.radix[D_DIMS] * h.radix[D_LS]);
            j.entry_base = (int32_t)halo_entries;
            halo_entries += j.n_entries;
        }
    }
    // lane-blocked work items go to their own launches (kernel template BLK = 1 or 2)
    std::vector<int> blk_of(L.size(), 0);
    {
        const size_t n0 = L.size();
        for (size_t li = 0; li < n0; li++) {
            LaunchArgs by_mode[4];
            for (auto &x : by_mode) memset(&x, 0, sizeof x);
            for (int i = 0; i < L[li].n_work; i++) {
                const WorkItem &w = L[li].work[i];
                by_mode[w.mode].work[by_mode[w.mode].n_work++] = w;
            }
            bool first = true;
            const uint32_t memo_bytes = L[li].memo_bytes, low_bytes = L[li].low_bytes, dtab_bytes = L[li].dtab_bytes;
            for (int md = 0; md < 4; md++) {
                LaunchArgs &x = by_mode[md];
                if (x.n_work == 0) continue;
                if (md) {
                    x.memo_bytes = memo_bytes;
                    x.low_bytes = low_bytes;
                    x.dtab_bytes = md == 1 ? dtab_bytes : md == 3 ? kLaneStateBytes : 0;
                } else if (fam_of[li] == PARADL_GPIPE) {
                    x.dtab_bytes = dtab_bytes;   // per-lane stage table
                } else if (fam_of[li] == PARADL_DATA_LW) {
                    x.memo_bytes = memo_bytes;   // per-layer Allreduce tables
                }
                if (first) {
                    L[li] = x;
                    blk_of[li] = md;
                    first = false;
                } else {
                    L.push_back(x);
                    fam_of.push_back(fam_of[li]);
                    blk_of.push_back(md);
                }
            }
        }
    }
    const size_t nl = L.size();
    if (nl == 0) return PARADL_OK;
    if (halo_entries > (size_t)INT32_MAX) return fail(c, PARADL_EINVAL, "halo tables too large");
    hj.total_entries = (int32_t)halo_entries;
    if (halo_entries) {
        CUDA_TRY(c, c->halo.ensure(sizeof(HaloEntry) * halo_entries));
        for (int j = 0; j < hj.n_jobs; j++) hj.job[j].tab = (HaloEntry *)c->halo.p + hj.job[j].entry_base;
        for (auto &a : L)
            for (int i = 0; i < a.n_work; i++)
                for (int j = 0; j < hj.n_jobs; j++)
                    if (hj.job[j].sub == a.work[i].sub) a.work[i].halo = hj.job[j].tab;
    }
    // pipeline structure tables (reduce mode, lane-strided work items of >= 2^22 configs):
    // one record per structure, computed by a thread-per-structure kernel before the sweep
    std::vector<StructJob> sjobs;
    if (!dense && !struct_table_off()) {
        uint64_t n_rec = 0;
        for (auto &a : L)
            for (int i = 0; i < a.n_work; i++) {
                WorkItem &w = a.work[i];
                if (w.mode != 0 || w.family != PARADL_PIPELINE || w.hi - w.lo < (1ull << 22)) continue;
                const SubHdr &h = P.subs[w.sub].hdr;
                const uint64_t nAB = (uint64_t)h.radix[D_ALPHA] * h.radix[D_BETA];
                StructJob j{};
                j.sub = w.sub;
                j.w_lo = w.lo;
                j.w_hi = w.hi;
                j.shard = 0;
                j.n_shards = 1;   // tile fields set once the tiles are planned
                j.s_lo = w.lo / nAB;
                j.n = (w.hi + nAB - 1) / nAB - j.s_lo;
                w.stab_lo = j.s_lo;
                w.stab = reinterpret_cast<const PipeRec *>((uintptr_t)n_rec);   // offset until allocated
                n_rec += j.n;
                sjobs.push_back(j);
            }
        if (n_rec) {
            CUDA_TRY(c, c->stab.ensure(sizeof(PipeRec) * n_rec));
            PipeRec *base = (PipeRec *)c->stab.p;
            size_t q = 0;
            for (auto &a : L)
                for (int i = 0; i < a.n_work; i++) {
                    WorkItem &w = a.work[i];
                    if (w.mode != 0 || w.family != PARADL_PIPELINE || w.hi - w.lo < (1ull << 22)) continue;
                    const uint64_t off = (uint64_t)(uintptr_t)w.stab;
                    w.stab = base + off;
                    sjobs[q++].out = base + off;
                }
        }
    }
    // tiles and grids
    std::vector<int> grids(nl);
    std::vector<size_t> smems(nl);
    size_t total_ctas = 0;
    for (size_t li = 0; li < nl; li++) {
        LaunchArgs &a = L[li];
        if (smem + a.memo_bytes + a.low_bytes + a.dtab_bytes > c->smem_optin) {
            if (fam_of[li] == PARADL_GPIPE || blk_of[li] == 3)
                return fail(c, PARADL_ENOMEM, "image + per-lane tables exceed shared memory");
            a.dtab_bytes = 0;   // unscreened path
        }
        smems[li] = smem + a.memo_bytes + a.low_bytes + a.dtab_bytes;
        const uint64_t okey = ((uint64_t)fam_of[li] << 40) | ((uint64_t)(dense ? (cmp ? 2 : 1) : 0) << 38) |
                              ((uint64_t)blk_of[li] << 35) |
                              (uint64_t)smems[li];
        int nb = -1;
        for (auto &kv : c->occ_cache)
            if (kv.first == okey) nb = kv.second;
        if (nb < 0) {
            nb = max_blocks_per_sm(fam_of[li], dense ? (cmp ? 2 : 1) : 0, blk_of[li], smems[li]);
            c->occ_cache.push_back({okey, nb});
        }
        if (nb < 1) return fail(c, PARADL_ECUDA, "sweep kernel cannot be resident with %zu bytes of shared memory", smems[li]);
        // A/B knob: PARADL_MAX_BPS=n caps the resident CTAs per SM (occupancy experiments)
        static const int max_bps = getenv("PARADL_MAX_BPS") ? atoi(getenv("PARADL_MAX_BPS")) : 0;
        if (max_bps > 0) nb = std::min(nb, max_bps);
        const int grid_max = c->n_sm * nb;
        const uint64_t warps = (uint64_t)grid_max * kWarps;
        uint64_t tiles = 0;
        for (int i = 0; i < a.n_work; i++) {
            WorkItem &w = a.work[i];
            const uint64_t range = w.hi - w.lo;
            if (w.mode != 0) {
                const SubHdr &h = P.subs[w.sub].hdr;
                const uint64_t Q = (uint64_t)h.radix[D_ALPHA] * h.radix[D_BETA] * h.radix[D_LS] * h.radix[D_DIMS] *
                                   h.radix[D_S];
                const uint64_t nblk = range / (w.mode == 2 ? Q << ((w.flags & kWorkMaskS) ? kLowBitsSorted : 8) : Q);
                // Tiles per warp of this rank's shard: the last wave of a dynamic tile queue leaves
                // at most one tile per warp unbalanced, and each tile pays a decode (unranking) and
                // a stage-state rebuild; 1..256 partitions per lane per tile.
                // 64 tiles per warp while a tile still holds >= 64 partitions (blocks) per lane,
                // else 16 (COMB partitions: cfg5, session 16, 1 shard 28.5 -> 28.1 ms, 2 shards
                // 14.86 -> 14.58 ms, 4 shards best at 16 per warp, 7.74 vs 7.94 ms at 32) or, for
                // 512-mask blocks (cheap tiles), tiles of 64 blocks per lane (cfg3 196.7 -> 191.9
                // ms); `ab_tiles_unrank_s16.log`.
                // A/B knob: PARADL_TPW = a fixed number of tiles per warp instead
                static const uint64_t tpw = getenv("PARADL_TPW") ? std::max(1, atoi(getenv("PARADL_TPW"))) : 0;
                const uint64_t per = nblk / n_shards / (32ull * warps);
                uint64_t cper = tpw ? per / tpw
                                : per / 64 >= 64 ? per / 64
                                : w.mode == 2 ? std::min<uint64_t>(64, per / 16)
                                              : per / 16;
                cper = std::max<uint64_t>(1, std::min<uint64_t>(cper, 256));
                w.steps = (uint32_t)cper;
                w.n_tiles = (nblk + 32ull * cper - 1) / (32ull * cper);
            } else {
                // >= ~8 tiles per warp for balance, but at least one whole alpha/beta block per
                // tile (structure terms are computed once per block), 32..131072 configs per tile
                const SubHdr &h = P.subs[w.sub].hdr;
                const uint64_t nAB = (uint64_t)h.radix[D_ALPHA] * h.radix[D_BETA];
                // families whose per-configuration work dwarfs the structure terms (a schedule,
                // a per-layer fold) split alpha/beta blocks across warps instead
                const bool heavy = w.family == PARADL_GPIPE || w.family == PARADL_DATA_LW;
                uint64_t steps = std::max<uint64_t>(range / n_shards / (32ull * warps * 8ull), heavy ? 4 : (nAB + 31) / 32);
                steps = std::max<uint64_t>(1, std::min<uint64_t>(steps, 4096));
                w.steps = (uint32_t)steps;
                w.n_tiles = (range + 32ull * steps - 1) / (32ull * steps);
            }
            w.tile_base = tiles;
            tiles += w.n_tiles;
        }
        a.total_tiles = tiles;
        for (int i = 0; i < a.n_work; i++)   // structure tables of this launch: shard's tiles only
            for (StructJob &j : sjobs)
                if (j.sub == a.work[i].sub && j.w_lo == a.work[i].lo && a.work[i].stab) {
                    j.ts = 32ull * a.work[i].steps;
                    j.tile_base = a.work[i].tile_base;
                    j.shard = shard;
                    j.n_shards = n_shards;
                }
        const uint64_t my_tiles = tiles > (uint64_t)shard ? (tiles - shard + n_shards - 1) / n_shards : 0;
        const uint64_t need_ctas = (my_tiles + kWarps - 1) / kWarps;   // small launches: one tile per warp
        grids[li] = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)grid_max, need_ctas));
        total_ctas += grids[li];
    }
    // counters: [nl] tile queues, [nl] count, [nl + 1] admission bound, [nl + 2] merge ticket
    // compact mode: the launches' tile spaces concatenated (slot_base[li] + T), and the tile
    // segments of every work item in ascending index order for the scan
    std::vector<uint64_t> slot_base(nl, 0);
    uint64_t n_slots = 0;
    CompactSegs segs{};
    if (cmp) {
        for (size_t li = 0; li < nl; li++) {
            slot_base[li] = n_slots;
            n_slots += L[li].total_tiles;
        }
        std::vector<std::pair<uint64_t, std::pair<uint64_t, uint64_t>>> order;
        for (size_t li = 0; li < nl; li++)
            for (int i = 0; i < L[li].n_work; i++) {
                const WorkItem &w = L[li].work[i];
                order.push_back({P.subs[w.sub].hdr.offset + w.lo, {slot_base[li] + w.tile_base, w.n_tiles}});
            }
        std::sort(order.begin(), order.end());
        if (order.size() > (size_t)kMaxSegs) return fail(c, PARADL_EINVAL, "compact sweep: too many work items");
        segs.n = (int32_t)order.size();
        for (size_t g = 0; g < order.size(); g++) {
            segs.slot[g] = order[g].second.first;
            segs.cnt[g] = order[g].second.second;
        }
        CUDA_TRY(c, c->ccnt.ensure(sizeof(uint32_t) * std::max<uint64_t>(1, n_slots)));
        CUDA_TRY(c, c->coff.ensure(sizeof(uint64_t) * std::max<uint64_t>(1, n_slots)));
    }
    CUDA_TRY(c, c->counters.ensure(sizeof(unsigned long long) * (nl + 3)));
    if (!dense) CUDA_TRY(c, c->lists.ensure(sizeof(paradl_hit) * total_ctas * k));
    if (!dense) CUDA_TRY(c, c->nvalid.ensure(sizeof(uint32_t) * total_ctas));
    unsigned long long *ctr = (unsigned long long *)c->counters.p;
    if (!sjobs.empty()) {   // the first structure-table launch zeroes them (it precedes every sweep)
        sjobs[0].ctr = ctr;
        sjobs[0].n_ctr = (int32_t)(nl + 1);
    } else {
        CUDA_TRY(c, cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * (nl + 3), st));
        CUDA_TRY(c, cudaMemsetAsync(ctr + nl + 1, 0xFF, sizeof(unsigned long long), st));   // no bound yet
    }

    if (halo_entries) {
        CUDA_TRY(c, launch_halo_tables(hj, st));
        c->stat_launches++;
    }
    for (const StructJob &j : sjobs) {
        const SubHdr &h = P.subs[j.sub].hdr;
        const uint64_t unit_len = (uint64_t)h.radix[D_S] * h.radix[D_DIMS] * h.radix[D_LS];
        CUDA_TRY(c, launch_struct_table((const uint8_t *)c->img.p, P.bytes, j, unit_len, st));
        c->stat_launches++;
    }
    // fork onto internal streams
    const bool fork = nl > 1;
    if (fork) {
        while (c->streams.size() < nl) {
            cudaStream_t s2;
            cudaEvent_t e2;
            CUDA_TRY(c, cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
            CUDA_TRY(c, cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
            c->streams.push_back(s2);
            c->events.push_back(e2);
        }
        if (!c->fork_ev) CUDA_TRY(c, cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventRecord(c->fork_ev, st));
    }
    size_t cta_off = 0;
    for (size_t li = 0; li < nl; li++) {
        LaunchArgs &a = L[li];
        a.img = (const uint8_t *)c->img.p;
        a.img_bytes = P.bytes;
        a.first = first;
        a.shard = shard;
        a.n_shards = n_shards;
        a.tile_counter = ctr + li;
        a.count = ctr + nl;
        a.gbound = ctr + nl + 1;
        a.k = k;
        a.cta_lists = dense ? nullptr : (paradl_hit *)c->lists.p + cta_off * k;
        a.cta_nvalid = dense ? nullptr : (uint32_t *)c->nvalid.p + cta_off;
        if (dense && cmp) {
            if (cmp->pass == 1) {
                a.c_cnt = (uint32_t *)c->ccnt.p + slot_base[li];
            } else {
                a.c_off = (const uint64_t *)c->coff.p + slot_base[li];
                a.c_idx = cmp->out->idx;
                a.c_cap = cmp->out->capacity;
                a.t_iter = cmp->out->t_iter;
                a.mem = cmp->out->mem;
            }
        } else if (dense) {
            a.t_iter = out->t_iter;
            a.mem = out->mem;
            a.bits = out->feasible_bits;
            a.reason = out->reason;
        }
        cudaStream_t ls = st;
        if (fork) {
            ls = c->streams[li];
            CUDA_TRY(c, cudaStreamWaitEvent(ls, c->fork_ev, 0));
        }
        CUDA_TRY(c, launch_sweep(fam_of[li], dense ? (cmp ? 2 : 1) : 0, blk_of[li], a, grids[li], smems[li], ls));
        c->stat_launches++;
        if (fork) CUDA_TRY(c, cudaEventRecord(c->events[li], ls));
        cta_off += grids[li];
    }
    if (fork)
        for (size_t li = 0; li < nl; li++) CUDA_TRY(c, cudaStreamWaitEvent(st, c->events[li], 0));
    if (cmp && cmp->pass == 1) {
        CUDA_TRY(c, launch_compact_scan((const uint32_t *)c->ccnt.p, (uint64_t *)c->coff.p, segs,
                                        (unsigned long long *)cmp->out->n_feasible, st));
        c->stat_launches++;
    }
    c->last_count_ptr = ctr + nl;
    if (n_lists_out) *n_lists_out = (int)total_ctas;
    return PARADL_OK;
}

extern "C" paradl_status paradl_sweep(paradl_ctx *c, const paradl_sweep_spec *spec, uint64_t first, uint64_t count,
                                      const paradl_dense_out *out, void *stream) {
    NvtxRange nvtx_("paradl_sweep");
    paradl_status s = need_device(c);
    if (s) return s;
    if (!out) return fail(c, PARADL_EINVAL, "null dense output");
    const Plan *PP = nullptr;
    s = plan_sweep(c, spec, &PP);
    if (s) return s;
    const Plan &P = *PP;
    if (first > P.total || count > P.total - first) return fail(c, PARADL_ERANGE, "range outside the sweep (%llu configs)", (unsigned long long)P.total);
    cudaStream_t st = (cudaStream_t)stream;
    s = upload(c, P, st);
    if (s) return s;
    if (count == 0) return PARADL_OK;
    if (out->feasible_bits) CUDA_TRY(c, cudaMemsetAsync(out->feasible_bits, 0, sizeof(uint32_t) * ((count + 31) / 32), st));
    return run_sweep(c, P, first, count, 0, 1, true, 0, out, st, nullptr);
}

extern "C" paradl_status paradl_sweep_compact(paradl_ctx *c, const paradl_sweep_spec *spec, uint64_t first,
                                              uint64_t count, const paradl_compact_out *out, void *stream) {
    NvtxRange nvtx_("paradl_sweep_compact");
    paradl_status s = need_device(c);
    if (s) return s;
    if (!out || !out->idx || !out->n_feasible) return fail(c, PARADL_EINVAL, "null compact output");
    const Plan *PP = nullptr;
    s = plan_sweep(c, spec, &PP);
    if (s) return s;
    const Plan &P = *PP;
    if (first > P.total || count > P.total - first) return fail(c, PARADL_ERANGE, "range outside the sweep (%llu configs)", (unsigned long long)P.total);
    cudaStream_t st = (cudaStream_t)stream;
    s = upload(c, P, st);
    if (s) return s;
    if (count == 0) {
        CUDA_TRY(c, cudaMemsetAsync(out->n_feasible, 0, sizeof(uint64_t), st));
        return PARADL_OK;
    }
    // pass 1: feasible count per tile, then the exclusive scan over the tiles in index order;
    // pass 2: the same tiles write their feasible configurations from the scanned offsets
    const CompactCall p1{1, out}, p2{2, out};
    s = run_sweep(c, P, first, count, 0, 1, true, 0, nullptr, st, nullptr, &p1);
    if (s) return s;
    return run_sweep(c, P, first, count, 0, 1, true, 0, nullptr, st, nullptr, &p2);
}

extern "C" paradl_status paradl_topk_async(paradl_ctx *c, const paradl_sweep_spec *spec, uint64_t first, uint64_t count,
                                           int32_t shard, int32_t n_shards, int32_t k, paradl_hit *d_hits,
                                           uint64_t *d_n_feasible, void *stream) {
    NvtxRange nvtx_("paradl_topk_async");
    paradl_status s = need_device(c);
    if (s) return s;
    if (k < 1 || k > PARADL_MAX_TOPK) return fail(c, PARADL_EINVAL, "k must be in 1..%d", PARADL_MAX_TOPK);
    if (n_shards < 1 || shard < 0 || shard >= n_shards) return fail(c, PARADL_EINVAL, "bad shard / n_shards");
    if (!d_hits || !d_n_feasible) return fail(c, PARADL_EINVAL, "null output");
    const Plan *PP = nullptr;
    s = plan_sweep(c, spec, &PP);
    if (s) return s;
    const Plan &P = *PP;
    if (first > P.total || count > P.total - first) return fail(c, PARADL_ERANGE, "range outside the sweep (%llu configs)", (unsigned long long)P.total);
    cudaStream_t st = (cudaStream_t)stream;
    s = upload(c, P, st);
    if (s) return s;
    int nlists = 0;
    c->last_count_ptr = nullptr;
    s = run_sweep(c, P, first, count, shard, n_shards, false, k, nullptr, st, &nlists);
    if (s) return s;
    CUDA_TRY(c, c->counters.ensure(sizeof(unsigned long long) * 2));
    unsigned long long *cnt = c->last_count_ptr;
    if (nlists == 0) {
        cnt = (unsigned long long *)c->counters.p;
        CUDA_TRY(c, cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
    }
    const uint32_t *mvalid = nlists ? (const uint32_t *)c->nvalid.p : nullptr;
    paradl_hit *lv_out = nullptr;
    uint32_t *lv_nv = nullptr;
    unsigned int *lv_done = nullptr;
    if (nlists > 64 && !merge_level_off()) {
        // many CTA lists: the merge launch first reduces groups of 16 lists per block (no
        // overflow on exact ties), its last block merges the group lists
        const int64_t nb = (nlists + 15) / 16;
        CUDA_TRY(c, c->lists2.ensure(sizeof(paradl_hit) * nb * k));
        CUDA_TRY(c, c->nvalid2.ensure(sizeof(uint32_t) * nb));
        lv_out = (paradl_hit *)c->lists2.p;
        lv_nv = (uint32_t *)c->nvalid2.p;
        // last-block ticket: the per-call counters block, zeroed before every sweep
        lv_done = (unsigned int *)(c->last_count_ptr + 2);
    }
    CUDA_TRY(c, launch_merge((const paradl_hit *)c->lists.p, nlists, k, cnt, 1, d_hits,
                             (unsigned long long *)d_n_feasible, st, nlists ? c->last_count_ptr + 1 : nullptr, 0, 0,
                             nullptr, mvalid, lv_out, lv_nv, lv_done));
    c->stat_launches++;
    return PARADL_OK;
}

extern "C" paradl_status paradl_merge_topk(paradl_ctx *c, const paradl_hit *d_lists, int32_t n_lists, int32_t k,
                                           const uint64_t *d_counts, paradl_hit *d_out, uint64_t *d_count_out,
                                           void *stream) {
    NvtxRange nvtx_("paradl_merge_topk");
    paradl_status s = need_device(c);
    if (s) return s;
    if (k < 1 || k > PARADL_MAX_TOPK || n_lists < 0 || (n_lists && (!d_lists || !d_counts)) || !d_out || !d_count_out)
        return fail(c, PARADL_EINVAL, "bad merge arguments");
    CUDA_TRY(c, launch_merge(d_lists, n_lists, k, (const unsigned long long *)d_counts, n_lists, d_out,
                             (unsigned long long *)d_count_out, (cudaStream_t)stream));
    c->stat_launches++;
    return PARADL_OK;
}

extern "C" paradl_status paradl_merge_records(paradl_ctx *c, const paradl_hit *d_records, int32_t n_records,
                                              int32_t k, paradl_hit *d_out, uint64_t *d_count_out, void *stream) {
    NvtxRange nvtx_("paradl_merge_records");
    paradl_status s = need_device(c);
    if (s) return s;
    if (k < 1 || k > PARADL_MAX_TOPK || n_records < 0 || (n_records && !d_records) || !d_out || !d_count_out)
        return fail(c, PARADL_EINVAL, "bad merge arguments");
    const unsigned long long *counts = n_records ? (const unsigned long long *)&d_records[k].idx : nullptr;
    CUDA_TRY(c, launch_merge(d_records, n_records, k, counts, n_records, d_out, (unsigned long long *)d_count_out,
                             (cudaStream_t)stream, nullptr, k + 1, (int32_t)((k + 1) * sizeof(paradl_hit) / 8)));
    c->stat_launches++;
    return PARADL_OK;
}

extern "C" paradl_status paradl_topk(paradl_ctx *c, const paradl_sweep_spec *spec, uint64_t first, uint64_t count,
                                     int32_t k, paradl_hit *hits, uint64_t *n_feasible, void *stream) {
    NvtxRange nvtx_("paradl_topk");
    paradl_status s = need_device(c);
    if (s) return s;
    if (!hits || !n_feasible) return fail(c, PARADL_EINVAL, "null output");
    if (k < 1 || k > PARADL_MAX_TOPK) return fail(c, PARADL_EINVAL, "k must be in 1..%d", PARADL_MAX_TOPK);
    CUDA_TRY(c, c->results.ensure(sizeof(paradl_hit) * PARADL_MAX_TOPK + 16));
    paradl_hit *dh = (paradl_hit *)c->results.p;
    uint64_t *dc = (uint64_t *)((uint8_t *)c->results.p + sizeof(paradl_hit) * PARADL_MAX_TOPK);
    s = paradl_topk_async(c, spec, first, count, 0, 1, k, dh, dc, stream);
    if (s) return s;
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(c, cudaMemcpyAsync(hits, dh, sizeof(paradl_hit) * k, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaMemcpyAsync(n_feasible, dc, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    c->stat_d2h += sizeof(paradl_hit) * k + sizeof(uint64_t);
    CUDA_TRY(c, cudaStreamSynchronize(st));
    return PARADL_OK;
}

extern "C" paradl_status paradl_argmin(paradl_ctx *c, const paradl_sweep_spec *spec, uint64_t first, uint64_t count,
                                       paradl_hit *best, uint64_t *n_feasible, void *stream) {
    NvtxRange nvtx_("paradl_argmin");
    return paradl_topk(c, spec, first, count, 1, best, n_feasible, stream);
}

static paradl_status explain_impl(paradl_ctx *c, const paradl_sweep_spec *spec, uint64_t idx, paradl_config *cfg,
                                  paradl_prediction *pred) {
    paradl_status s = need_device(c);
    if (s) return s;
    const Plan *PP = nullptr;
    s = plan_sweep(c, spec, &PP);
    if (s) return s;
    const Plan &P = *PP;
    if (idx >= P.total) return fail(c, PARADL_ERANGE, "index %llu outside the sweep", (unsigned long long)idx);
    s = upload(c, P, 0);
    if (s) return s;
    int sub = 0;
    while (idx >= P.subs[sub].hdr.offset + P.subs[sub].hdr.count) sub++;
    CUDA_TRY(c, c->one.ensure(sizeof(paradl_config) + sizeof(paradl_prediction)));
    paradl_config *dcfg = (paradl_config *)c->one.p;
    paradl_prediction *dpr = (paradl_prediction *)((uint8_t *)c->one.p + sizeof(paradl_config));
    CUDA_TRY(c, launch_explain((const uint8_t *)c->img.p, P.bytes, sub, idx - P.subs[sub].hdr.offset, dcfg, dpr, 0));
    paradl_config hc;
    paradl_prediction hp;
    CUDA_TRY(c, cudaMemcpy(&hc, dcfg, sizeof hc, cudaMemcpyDeviceToHost));
    CUDA_TRY(c, cudaMemcpy(&hp, dpr, sizeof hp, cudaMemcpyDeviceToHost));
    if (cfg) *cfg = hc;
    if (pred) *pred = hp;
    return PARADL_OK;
}

extern "C" paradl_status paradl_decode(paradl_ctx *c, const paradl_sweep_spec *spec, uint64_t idx, paradl_config *out) {
    if (!out) return fail(c, PARADL_EINVAL, "null output");
    return explain_impl(c, spec, idx, out, nullptr);
}

extern "C" paradl_status paradl_explain(paradl_ctx *c, const paradl_sweep_spec *spec, uint64_t idx,
                                        paradl_prediction *out) {
    NvtxRange nvtx_("paradl_explain");
    if (!out) return fail(c, PARADL_EINVAL, "null output");
    return explain_impl(c, spec, idx, nullptr, out);
}

extern "C" uint64_t paradl_stat(const paradl_ctx *c, int32_t which) {
    if (!c) return 0;
    switch (which) {
    case 0: return c->stat_h2d;
    case 1: return c->stat_d2h;
    case 2: return c->stat_launches;
    default: return 0;
    }
}

extern "C" paradl_status paradl_fp64_peak(paradl_ctx *c, double ms, double *inst_per_s) {
    paradl_status s = need_device(c);
    if (s) return s;
    if (!inst_per_s || !(ms > 0)) return fail(c, PARADL_EINVAL, "bad arguments");
    double *sink = nullptr;
    CUDA_TRY(c, cudaMalloc(&sink, 256 * sizeof(double)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int threads = 0;
    int iters = 64;
    float el = 0.f;
    cudaError_t e = cudaSuccess;
    for (int round = 0; round < 12; round++) {   // grow until the launch lasts ~ms
        e = launch_fp64_bench(c->n_sm, iters, sink, 0, &threads);
        if (e != cudaSuccess) break;
        cudaEventRecord(e0, 0);
        e = launch_fp64_bench(c->n_sm, iters, sink, 0, &threads);
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&el, e0, e1);
        if (e != cudaSuccess || el >= ms) break;
        iters *= 2;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (e != cudaSuccess) return fail(c, PARADL_ECUDA, "fp64 bench: %s", cudaGetErrorString(e));
    *inst_per_s = (double)threads * iters * 16.0 * 8.0 / (el * 1e-3);
    return PARADL_OK;
}
