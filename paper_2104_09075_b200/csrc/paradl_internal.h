// paradl_internal.h -- device image layout shared by the host library (api.cpp) and the
// CUDA kernels (kernels.cu).  Not part of the public ABI (include/paradl.h).
//
// A sweep is evaluated from one contiguous "image" in device global memory that every
// persistent CTA stages into shared memory with one TMA bulk copy (cp.async.bulk +
// mbarrier):
//
//   [ImgHdr][SubHdr x n_sub][value tables, binomials, stage-block offsets][model blocks]
//
// A model block is produced on the device by the prep kernel at paradl_load_model
// (prefix sums and totals) and copied device-to-device into the image.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "paradl.h"

namespace paradl {

constexpr int kMaxSub = 64;
constexpr int kMaxWork = 8;              // work items per sweep launch (kernel parameter size)
constexpr int kMaxModelsPerSweep = 8;
constexpr int kThreads = 256;            // threads per CTA of the sweep kernels
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kWorkMaskD = 1u;
constexpr uint32_t kWorkPow2 = 2u;       // mode 3: every dims p_d is a power of two (ge_s by an exact scale)
constexpr int kLowBitsSorted = 9;       // kWorkMaskS blocks: 2^9 masks (kernels.cu kLowBitsS)
constexpr uint32_t kWorkMaskS = 4u;      // mode 2 (kWorkMaskD, one configuration per mask, one flops value):
                                         // the screen reads the (e, pop)-sorted table with tau / beta folded in
constexpr uint32_t kMaskTabN = 72;              // per-stage-count tables of the screened mask path (n <= 64)
constexpr uint32_t kMaxDtabBytes = 48u << 10;   // cap of the mode-1 per-lane dims tables
constexpr int kMaxCuts = PARADL_MAX_COMB_CUTS;
constexpr int kGpMax = PARADL_GPIPE_MAX_STAGES;
// mode-3 (COMB, incremental stage terms) per-lane stage state: 24 int64 per thread, column layout
constexpr uint32_t kLaneStateBytes = 24u * 8u * kThreads;
// GPIPE per-lane stage table in shared memory: 4 doubles (f, g, m, u) per stage, column per thread
constexpr uint32_t kGpipeTabBytes = 4u * kGpMax * 8u * kThreads;

// digits of the canonical mixed radix, fast -> slow
enum { D_BETA = 0, D_ALPHA, D_LS, D_DIMS, D_S, D_PART, D_B, D_FLOPS, D_CAP, kDigits };

struct RowGeo {            // 48 B: geometry of one layer row (halo / limits)
    int32_t kind, flags;
    int32_t C, F;
    int32_t X[3], Y[3], K[3];
    int32_t pad;
};

struct ModelHdr {          // 128 B, start of a model block
    int32_t G, pad0;
    int64_t D;
    // per-model integer sums (Table 2 Sigma_l), computed by the prep kernel
    int64_t FB, WU, W, BI, XY, YC, NC, Fmin, Cmin2;
    // byte offsets from the start of the block
    uint32_t off_geo, off_pf, off_pb, off_pu, off_pw, off_pxy, off_pbi, off_y;
    uint32_t bytes, pad1;
};
static_assert(sizeof(ModelHdr) == 128, "ModelHdr layout");

struct ImgHdr {
    uint32_t bytes;
    int32_t n_sub, n_models, n_tiers;
    int32_t delta, tree_chunks;
    double gamma, phi_df, tree_thr;
    double ar_mult;                    // filter/channel/df FB-AR = ar_mult x FB-AG: 2 (Allreduce), 1 (Reduce-Scatter)
    double phi_pd, phi_ds;             // contention on the pd stage Allreduces (s > 1), ds reduce-to-leader (p1 > 1)
    // tiers: n_ctiers collective tiers (tier_of scans these); alpha/beta rows hold n_tiers values,
    // the point-to-point copies (x p2p scales) at p2p_off + t when the scales are not 1 (Q40)
    int32_t n_ctiers, p2p_off;
    int64_t max_pes[PARADL_MAX_TIERS];
    uint32_t model_off[kMaxModelsPerSweep];
    uint32_t sub_off[kMaxSub];
};
static_assert(sizeof(ImgHdr) % 16 == 0, "ImgHdr alignment");

struct SubHdr {
    int32_t family, model;                 // model = index into ImgHdr::model_off
    int32_t part_mode, s_min, s_max, kmax; // kmax = s_max - 1 (COMB)
    uint32_t radix[kDigits];               // radix[D_PART] unused (see part_n)
    int32_t G;
    uint64_t part_n;                       // partition radix
    uint64_t count, offset;                // configs in this sub-sweep, global index offset
    uint32_t off_cap, off_flops, off_b, off_S, off_dims, off_Ls, off_alpha, off_beta;
    uint32_t off_binom, off_sblk;          // uint64 C(n,j) [n*(kmax+1)+j], n < G; uint64 s-block offsets
    uint32_t binom_stride, pad0, pad1, pad2;
};
static_assert(sizeof(SubHdr) % 16 == 0, "SubHdr alignment");

// Halo-table entry per (dims index, Ls index) of a spatial / ds sub-sweep (row a5).
struct HaloEntry {
    int64_t NS, HV;
    uint32_t reason, pad0;
    uint64_t pad1;
};
static_assert(sizeof(HaloEntry) == 32, "HaloEntry layout");

// One contiguous local index range [lo, hi) of one sub-sweep inside a sweep launch.
// Tiles of 32*steps consecutive configurations; tile_base = index of its first tile in
// the launch's global tile space (all work items concatenated, spec order).
struct WorkItem {
    int32_t sub, family;
    uint32_t steps;                // mode 0: steps of 32 configs per tile; mode 1: partitions per lane per tile
    int32_t inc_top;               // highest digit with a non-zero stride increment
    uint64_t lo, hi, n_tiles, tile_base;
    uint32_t inc[kDigits];         // mixed-radix digits of the lane stride (32 configs, or 1 partition)
    int32_t mode;                  // 0: lane-strided (lanes = 32 consecutive configs); 1: lane-blocked
                                   // (pipeline families: each lane owns whole partitions, [lo,hi) aligned);
                                   // 2: 256-mask blocks (MASK); 3: lane-blocked COMB, incremental stage terms
    uint64_t inc_part;
    const HaloEntry *halo;         // spatial / ds: [n_dims][n_Ls] table (device global), else null
    uint32_t memo_off, memo_n;     // mode 1/2: smem table [n_b][n_S + n_dims] of b/S and D/(b*p_d)
    uint32_t low_off, flags;       // mode 2: index of its [n_b][256] low-bit stage table (LowE units);
                                   // flags: kWorkMaskD = screened pipeline masks, stage terms as exact doubles
    uint32_t cmb_off, pad_c;       // mode 3: byte offset (from the memo base) of its comb tables
                                   // [CmbN x (s_max+1)][CmbS x n_b(s_max+1)n_S][CmbD x n_b(s_max+1)n_dims]
    const struct PipeRec *stab;    // mode 0 pipeline, reduce: structure table (device global), else null
    uint64_t stab_lo;              // structure index of stab[0] within the sub-sweep
};

// Structure record of a pipeline sub-sweep (reduce mode): the alpha/beta-invariant terms of
// compute_mid<PIPELINE> + fastify for one structure (cap, R, b, partition, S, dims, Ls),
// written by the structure-table kernel, read by the sweep kernel's mode-0 tiles.
struct PipeRec {
    double comp, pp_c, pp_s, I;
    uint32_t reason;
    int32_t pp_t;
    uint32_t pad[2];
};
static_assert(sizeof(PipeRec) == 48, "PipeRec layout");

struct StructJob {
    int32_t sub, pad;
    uint64_t s_lo, n;              // structures [s_lo, s_lo + n) of sub-sweep `sub`
    PipeRec *out;
    unsigned long long *ctr;       // non-null: zero ctr[0, n_ctr), set ctr[n_ctr] = ~0 and zero
    int32_t n_ctr, pad2;           // ctr[n_ctr + 1] (tile counters, count, admission bound, merge ticket)
    // sharded calls: only structures overlapping this shard's tiles are computed (tile T
    // covers local configs [w_lo + (T - tile_base) ts, +ts); T % n_shards == shard)
    uint64_t w_lo, w_hi, ts, tile_base;
    int32_t shard, n_shards;
};

// Arguments of one persistent sweep launch (passed as a __grid_constant__ parameter).
struct LaunchArgs {
    const uint8_t *img;            // device image
    uint32_t img_bytes;            // multiple of 16
    int32_t n_work;
    uint32_t memo_bytes;           // lane-blocked memo tables after SmemExtra (multiple of 16)
    uint32_t low_bytes;            // mode-2 low-bit stage tables after the memo tables
    uint64_t first;                // global index of dense element 0
    uint64_t total_tiles;
    int32_t shard, n_shards;
    unsigned long long *tile_counter;
    int32_t k;
    uint32_t dtab_bytes;           // mode-1 screened path: per-lane dims tables after the low tables
    paradl_hit *cta_lists;         // [gridDim.x][k] (reduce mode)
    uint32_t *cta_nvalid;          // [gridDim.x] entries written per CTA list (reduce mode)
    unsigned long long *count;     // feasible count accumulator (reduce mode)
    unsigned long long *gbound;    // shared top-k admission bound (reduce mode; ~0 = none)
    double *t_iter;                // dense outputs (indexed by global idx - first)
    double *mem;
    uint32_t *bits;
    uint8_t *reason;
    // compact mode (paradl_sweep_compact): pass 1 writes the feasible count of every tile to
    // c_cnt[T]; pass 2 writes tile T's feasible configurations from offset c_off[T] on
    uint32_t *c_cnt;
    const uint64_t *c_off;
    uint64_t *c_idx;
    uint64_t c_cap;
    WorkItem work[kMaxWork];
};

// Tile segments of a compact sweep in ascending index order: slots [slot, slot + n) of the
// per-launch tile-count arrays (launch tile spaces concatenated)
constexpr int kMaxSegs = 256;
struct CompactSegs {
    int32_t n, pad;
    uint64_t slot[kMaxSegs];
    uint64_t cnt[kMaxSegs];
};

struct HaloJob {
    int32_t sub, n_entries;
    int32_t entry_base, pad;
    HaloEntry *tab;
};
struct HaloJobs {
    const uint8_t *img;
    int32_t n_jobs, total_entries;
    HaloJob job[kMaxSub];
};

// launchers implemented in kernels.cu
cudaError_t launch_prep_model(const paradl_layer *d_rows, int32_t G, int64_t D, uint8_t *d_block,
                              const ModelHdr &layout, cudaStream_t st);
// dense: 0 reduce, 1 dense writes, 2 compact writes
cudaError_t launch_sweep(int family, int dense, int blk, const LaunchArgs &a, int grid, size_t smem,
                         cudaStream_t st);
int max_blocks_per_sm(int family, int dense, int blk, size_t smem);
size_t sweep_smem_extra();
cudaError_t launch_merge(const paradl_hit *lists, int64_t n_lists, int32_t k,
                         const unsigned long long *counts, int32_t n_counts, paradl_hit *out,
                         unsigned long long *count_out, cudaStream_t st,
                         const unsigned long long *gbound = nullptr, int32_t lstride = 0, int32_t cstride = 0,
                         unsigned long long *bound_out = nullptr, const uint32_t *nvalid = nullptr,
                         paradl_hit *lv_out = nullptr, uint32_t *lv_nvalid = nullptr, unsigned int *lv_done = nullptr);
cudaError_t launch_halo_tables(const HaloJobs &jobs, cudaStream_t st);
cudaError_t launch_compact_scan(const uint32_t *cnt, uint64_t *off, const CompactSegs &segs,
                                unsigned long long *total, cudaStream_t st);
cudaError_t launch_struct_table(const uint8_t *img, uint32_t img_bytes, const StructJob &job, uint64_t unit_len,
                                cudaStream_t st);
cudaError_t launch_fp64_bench(int n_sm, int iters, double *d_sink, cudaStream_t st, int *threads_out);
cudaError_t launch_explain(const uint8_t *img, uint32_t img_bytes, int32_t sub, uint64_t local,
                           paradl_config *d_cfg, paradl_prediction *d_pred, cudaStream_t st);

}  // namespace paradl
