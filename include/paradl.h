/*
 * paradl.h -- C ABI of the B200-native ParaDL sweep library (libparadl.so).
 *
 * What it computes: ParaDL's per-iteration compute / communication / memory cost
 * model (arXiv 2104.09075, Table 2 "Computation, Communication, and Memory
 * Analysis Summary", and Appendix A.1) evaluated for every
 * configuration of a sweep (strategy x PE counts x batch x split x pipeline stage
 * partition x segments x system alpha/beta/FLOPS/capacity), checked for feasibility
 * (Table 2 "Number of PEs" column; memory capacity) and reduced to
 * the best configurations ("Suggesting the best strategy").  The exact fp64
 * expression trees and the readings of the paper are in DESIGN.md §2.
 *
 * Conventions for every call:
 *   - returns paradl_status: 0 = OK, < 0 = error; paradl_last_error(ctx) then holds a
 *     ctx-owned message valid until the next call on that ctx.  No exception and no
 *     abort crosses the ABI.
 *   - inputs are plain host pointers that are copied during the call: the caller keeps
 *     ownership and may free them on return.
 *   - pointers documented "DEVICE" are CUDA device pointers owned by the caller; the
 *     library never frees them.  Streams are cudaStream_t passed as void* (NULL = the
 *     legacy default stream).
 *   - a ctx is bound to one CUDA device and is not thread-safe; use one ctx per host
 *     thread.  All computation happens in CUDA kernels; there is no CPU fallback: a
 *     ctx created with cuda_device = -1 is "host-only" and supports validation calls
 *     (load_model, set_system, sweep_size) but returns PARADL_ESTATE for the rest.
 *   - infeasible configurations are results, not errors (feasibility bit + reason).
 */
#ifndef PARADL_H
#define PARADL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARADL_ABI_VERSION 2
#define PARADL_MAX_TIERS 4
#define PARADL_MAX_STAGES 64     /* stage_end[] capacity of paradl_config */
#define PARADL_MAX_COMB_CUTS 15  /* combination-mode partitions: s_max <= 16 */
#define PARADL_MAX_TOPK 64

typedef enum {
    PARADL_OK = 0,
    PARADL_EINVAL = -1,     /* malformed argument (message says which) */
    PARADL_ENOMEM = -2,     /* device/host allocation failed, or the staged image exceeds shared memory */
    PARADL_ECUDA = -3,      /* a CUDA runtime call failed */
    PARADL_EOVERFLOW = -4,  /* an int64 intermediate (e.g. B*sum FLOPs) could exceed 2^63 for this sweep */
    PARADL_ERANGE = -5,     /* idx or [first, first+count) outside the sweep */
    PARADL_ESTATE = -6      /* no system set / unknown model id / host-only ctx */
} paradl_status;

/* Row kinds (non-conv layers adapted to the conv notation). */
enum { PARADL_CONV = 0, PARADL_FC = 1, PARADL_POOL = 2, PARADL_ELEM = 3, PARADL_NORM = 4 };
/* Row flags. COMM: the row is a filter/channel communication point (Table 3).
 * FOLDED: w / fw include folded layers (e.g. a projection shortcut), so w != C*F*prod(K). */
enum { PARADL_FLAG_COMM = 1u, PARADL_FLAG_FOLDED = 4u };

/* Strategy families (Table 2 rows). dims[4] meaning per family:
 *   SERIAL, PIPELINE, LAYERPURE, GPIPE: (1,1,1,1)     DATA, FILTER, CHANNEL: (p,1,1,1)
 *   DF (data+filter): (p1,p2,1,1)              SPATIAL, SPATIAL_AG: (1,pw,ph,pd)
 *   DS (data+spatial): (p1,pw,ph,pd)           PD (pipeline+data): (p_d,1,1,1)
 * SPATIAL_AG: spatial on the first Ls rows, then an Allgather of y_Ls and the remaining
 *   rows replicated on every PE (the paper's implementation; Q35).
 *   Needs Ls >= 1.
 * GPIPE: a pipeline partition timed by the GPipe schedule itself (S segments, forward
 *   wave then backward wave, blocking boundary sends, per-stage WU, DESIGN.md
 *   Q36) instead of Table 2's max-stage form.  Needs s <= PARADL_GPIPE_MAX_STAGES
 *   (COMB: s_max, MASK: G) and S >= 1.
 * DATA_LW: dims (p,1,1,1); the Data row with the gradient exchanged as one Allreduce per
 *   weighted layer (message delta |w_l|, row order), each message ring or tree by its size
 *   against tree_threshold_B ("ring ... for large message sizes and a tree-based algorithm
 *   for small message sizes"; tree time P:559; Q37).
 * LAYERWISE: dims (p,1,1,1), partition mode MASK with one bit per COMM row (row order):
 *   1 = that weighted layer is filter-parallel, 0 = data-parallel, over the same p PEs
 *   ("applying different parallel strategies for different layers"); rows
 *   between COMM rows follow the COMM row before them.  Mini-batch B = b p.  Strategy
 *   changes exchange the b-sample boundary activation (Q39).  At most 62 COMM
 *   rows. */
enum { PARADL_SERIAL = 0, PARADL_DATA, PARADL_SPATIAL, PARADL_FILTER, PARADL_CHANNEL,
       PARADL_DF, PARADL_DS, PARADL_PIPELINE, PARADL_LAYERPURE, PARADL_PD,
       PARADL_SPATIAL_AG, PARADL_GPIPE, PARADL_DATA_LW, PARADL_LAYERWISE, PARADL_N_FAMILIES };
#define PARADL_GPIPE_MAX_STAGES 8

/* Partition radix of the pipeline families (groups g_i, P:519 footnote).
 * COMB: every contiguous partition into s in [s_min, s_max] stages; s ascending, cut
 *       tuples c_1<...<c_{s-1} (c_j = rows in stages 1..j) in lexicographic order.
 * MASK: all 2^(G-1) partitions (G <= 64); partition index = mask, bit j <=> cut after row j+1. */
enum { PARADL_PART_NONE = 0, PARADL_PART_COMB = 1, PARADL_PART_MASK = 2 };

/* Infeasibility reasons (bit set; 0 = feasible). */
enum { PARADL_R_SCALING = 1,   /* Table 2 "Number of PEs" limit violated */
       PARADL_R_MEMORY = 2,    /* mem > capacity (closed bound: mem == cap is feasible) */
       PARADL_R_SPLIT = 4,     /* spatial split too fine for the halo (local extent < floor(K/2)) */
       PARADL_R_TIER = 8,      /* a communicator spans more PEs than the largest tier; t_iter = +inf */
       PARADL_R_SEGMENTS = 16  /* pipeline segments S > per-replica batch */ };

typedef struct paradl_ctx paradl_ctx;

/* Create a context on CUDA device `cuda_device` (>= 0), or a host-only context (-1). */
paradl_status paradl_create(int32_t cuda_device, paradl_ctx **out);
/* Frees all device memory the ctx owns. NULL is a no-op. */
void paradl_destroy(paradl_ctx *ctx);
const char *paradl_last_error(const paradl_ctx *ctx);
const char *paradl_version(void);

/* One row of the layer table = one of the paper's G "layers" (Table 4 counts).
 * Tensors x[N,C,X], y[N,F,Y], w[C,F,K], bi[F].  Unused spatial axes are 1;
 * weightless rows have K = 0.  x, y are per-sample element counts; fw, bw are
 * per-sample FLOPs of FW_l, BW_l; wu is per-iteration FLOPs of WU_l.
 * Validated: kind/ndim range, C,F,X,Y >= 1, x == C*prod(X), y == F*prod(Y),
 * w == C*F*prod(K) for CONV/FC unless FLAG_FOLDED, w == 0 for weightless kinds, all
 * counts >= 0.  160 bytes. */
typedef struct {
    int32_t kind, ndim;
    int64_t C, F, X[3], Y[3], K[3];
    int64_t x, y, w, bi, fw, bw, wu;
    uint32_t flags, reserved;
} paradl_layer;

/* Copies G rows (G >= 1) and dataset size D (Table 1, >= 1) to the device and derives the
 * per-model sums / prefix arrays there (CUDA prep kernel).  Returns the model id (0, 1, ...). */
paradl_status paradl_load_model(paradl_ctx *ctx, const paradl_layer *rows, int32_t G,
                                int64_t dataset_D, int32_t *model_id);

/* Hockney alpha-beta link model per tier of a hierarchical system:
 * a collective over n PEs uses the smallest tier with max_pes >= n. */
typedef struct { int64_t max_pes; double alpha_s; double beta_s_per_B; } paradl_tier;

typedef struct {
    int32_t n_tiers;            /* 1..PARADL_MAX_TIERS, max_pes strictly increasing, >= 1 */
    int32_t delta;              /* bytes per element, delta in {2,4,8} (Table 1) */
    paradl_tier tiers[PARADL_MAX_TIERS];
    double flops_per_s;         /* R > 0: FW_l = fw_l / R (Q28) */
    double hbm_bytes;           /* per-PE memory capacity > 0 */
    double gamma;               /* memory reuse factor in (0,1] */
    double phi_df;              /* >= 1: contention on the df inter-group Allreduce */
    double tree_threshold_B;    /* >= 0: Allreduce messages below it use the tree form; 0 = ring only */
    int32_t tree_chunks;        /* k >= 1 of the tree form */
    int32_t filter_rs;          /* 0: filter/channel/df backward dL/dx exchange is an Allreduce (Table 2);
                                   1: a Reduce-Scatter, (p-1)(alpha + (m/p) beta) (P:355 footnote; Q38) */
    /* Point-to-point patterns (spatial / ds halo exchange, pipeline / layer-pure / GPipe
     * boundary sends) use alpha x p2p_alpha_scale and beta x p2p_beta_scale of their tier,
     * collectives the tier itself ("different network parameters ... for MPI and NCCL",
     * P:768-769; Q40).  > 0; 1 = Table 2 literal. */
    double p2p_alpha_scale, p2p_beta_scale;
    /* >= 1: contention on the pd stage Allreduces when s > 1 run at once, and on the ds
     * reduce-to-leader when p1 > 1 groups reduce at once (beta x phi; Q40). */
    double phi_pd, phi_ds;
} paradl_system;

/* Base system: default alpha/beta per tier, R, capacity (sweeps may override per radix). */
paradl_status paradl_set_system(paradl_ctx *ctx, const paradl_system *sys);

/* One sub-sweep: the Cartesian product of its value lists, in the canonical order
 * (slow -> fast): cap, flops, b, partition, S, dims, Ls, alpha, beta.
 * An empty list (n_* = 0) is one value: cap -> sys.hbm_bytes, flops -> sys.flops_per_s,
 * S -> 1, dims -> (1,1,1,1), Ls -> 0, alpha/beta -> the system tiers.  b must be
 * non-empty; SPATIAL/DS need a non-empty Ls list.  Ls = number of leading rows forming
 * the spatial prefix (the Conv/Pool rows among them carry halos).
 * alpha/beta rows have n_tiers values each (row-major). */
typedef struct {
    int32_t family, model_id;
    int32_t part_mode, s_min, s_max;
    int32_t n_cap, n_flops, n_b, n_S, n_dims, n_Ls, n_alpha, n_beta, reserved;
    const double *cap;        /* bytes */
    const double *flops;      /* FLOP/s */
    const int64_t *b;         /* samples per data-parallel replica (B = b * data degree, Q2) */
    const int32_t *S;         /* pipeline segments */
    const int32_t *dims;      /* n_dims x 4, see the family enum */
    const int32_t *Ls;        /* spatial prefix lengths */
    const double *alpha;      /* n_alpha x n_tiers, seconds */
    const double *beta;       /* n_beta x n_tiers, seconds per byte */
} paradl_subsweep;

typedef struct { int32_t n_sub, reserved; const paradl_subsweep *sub; } paradl_sweep_spec;

/* Dense outputs for configs [first, first+count): element i is config first+i.
 * All DEVICE pointers, caller-allocated; any may be NULL (not written).
 *   t_iter: count doubles, seconds per iteration (+inf if reason has PARADL_R_TIER)
 *   mem: count doubles, bytes per PE
 *   feasible_bits: ceil(count/32) words, bit i%32 of word i/32 = feasible(first+i)
 *   reason: count bytes, PARADL_R_* bits. */
typedef struct { double *t_iter; double *mem; uint32_t *feasible_bits; uint8_t *reason; } paradl_dense_out;

/* Ranking key = predicted epoch time t_iter * (D/B) (Table 1 I = D/B); ties -> lower idx.
 * Unused slots of a top-k result hold idx = UINT64_MAX, key = +inf. */
typedef struct { uint64_t idx; double key_epoch_s; } paradl_hit;

typedef struct {
    int32_t sub, family, model_id, n_stages;
    int64_t i_cap, i_flops, i_b, i_S, i_dims, i_Ls, i_alpha, i_beta;
    uint64_t i_part;
    double cap, flops;
    int64_t b, B, p;           /* per-replica batch, mini-batch B, total PEs */
    int32_t S, Ls, dims[4];
    double alpha[PARADL_MAX_TIERS], beta[PARADL_MAX_TIERS];
    int32_t stage_end[PARADL_MAX_STAGES];   /* rows in stages 1..i, last = G */
} paradl_config;

/* Phase breakdown of one configuration (phases of P:755), per iteration.  SPATIAL_AG
 * reports its boundary Allgather in t_fb_ag; GPIPE reports the whole schedule time
 * (compute, boundary sends, WU) in t_comp. */
typedef struct {
    double t_comp, t_ge, t_fb_ag, t_fb_ar, t_halo, t_p2p, t_iter, t_epoch, mem, I;
    uint32_t reason;
    int32_t feasible;
} paradl_prediction;

/* Compact outputs for the feasible configurations of [first, first+count), in ascending
 * index order (row a9 compact mode; the per-configuration breakdown of P:427-429 restricted
 * to what fits the PEs).  All DEVICE pointers, caller-allocated:
 *   idx: capacity uint64, global configuration indices, strictly ascending
 *   t_iter, mem: capacity doubles each (may be NULL: not written), as in paradl_dense_out
 *   n_feasible: one uint64, the number of feasible configurations in the range; entries past
 *     `capacity` are not written (the caller compares *n_feasible with capacity). */
typedef struct {
    uint64_t *idx;
    double *t_iter;
    double *mem;
    uint64_t capacity;
    uint64_t *n_feasible;
} paradl_compact_out;

/* Number of configurations of the sweep (host-only ctx allowed). */
paradl_status paradl_sweep_size(paradl_ctx *ctx, const paradl_sweep_spec *spec, uint64_t *n);

/* Dense evaluation, asynchronous on `stream`. */
paradl_status paradl_sweep(paradl_ctx *ctx, const paradl_sweep_spec *spec, uint64_t first,
                           uint64_t count, const paradl_dense_out *out, void *stream);

/* Compact evaluation, asynchronous on `stream`: two passes over the same tiles -- the first
 * counts the feasible configurations of every tile (warp ballots), an exclusive scan over the
 * tiles in index order gives each tile its output offset, the second re-evaluates the tiles
 * and writes (idx, t_iter, mem) at offset + popc(ballot & lanes below) (coalesced SoA stores).
 * The values equal paradl_sweep's for the same configurations.  Errors: as paradl_sweep;
 * PARADL_EINVAL for a NULL idx or n_feasible. */
paradl_status paradl_sweep_compact(paradl_ctx *ctx, const paradl_sweep_spec *spec, uint64_t first,
                                   uint64_t count, const paradl_compact_out *out, void *stream);

/* Top-k (1 <= k <= PARADL_MAX_TOPK) of the feasible configurations of [first, first+count)
 * by (key, idx), plus their count.  Host outputs; synchronises `stream`. */
paradl_status paradl_topk(paradl_ctx *ctx, const paradl_sweep_spec *spec, uint64_t first,
                          uint64_t count, int32_t k, paradl_hit *hits, uint64_t *n_feasible,
                          void *stream);
/* = paradl_topk with k = 1. */
paradl_status paradl_argmin(paradl_ctx *ctx, const paradl_sweep_spec *spec, uint64_t first,
                            uint64_t count, paradl_hit *best, uint64_t *n_feasible, void *stream);

/* Sharded, device-output, asynchronous top-k for multi-GPU runs: the range is cut into
 * tiles and only tiles t with t % n_shards == shard are evaluated.  d_hits: DEVICE, k
 * entries; d_n_feasible: DEVICE, one uint64.  Nothing is synchronised. */
paradl_status paradl_topk_async(paradl_ctx *ctx, const paradl_sweep_spec *spec, uint64_t first,
                                uint64_t count, int32_t shard, int32_t n_shards, int32_t k,
                                paradl_hit *d_hits, uint64_t *d_n_feasible, void *stream);
/* Merge n_lists device top-k lists (n_lists x k, e.g. gathered from all ranks) and their
 * counts into one list and one total (all DEVICE pointers), asynchronously. */
paradl_status paradl_merge_topk(paradl_ctx *ctx, const paradl_hit *d_lists, int32_t n_lists,
                                int32_t k, const uint64_t *d_counts, paradl_hit *d_out,
                                uint64_t *d_count_out, void *stream);

/* Multi-GPU record layout: a record is paradl_hit[k + 1] whose first k entries are a top-k
 * list (as written by paradl_topk_async to d_hits = record) and whose entry k holds the
 * feasible count in its idx field (d_n_feasible = &record[k].idx).  Merges n_records such
 * records (contiguous, DEVICE, e.g. one all_gather of every rank's record) asynchronously. */
paradl_status paradl_merge_records(paradl_ctx *ctx, const paradl_hit *d_records, int32_t n_records,
                                   int32_t k, paradl_hit *d_out, uint64_t *d_count_out, void *stream);

/* Decode / explain one index (evaluated by a CUDA kernel; host outputs; synchronous). */
paradl_status paradl_decode(paradl_ctx *ctx, const paradl_sweep_spec *spec, uint64_t idx,
                            paradl_config *out);
paradl_status paradl_explain(paradl_ctx *ctx, const paradl_sweep_spec *spec, uint64_t idx,
                             paradl_prediction *out);

/* Counters of the last call on this ctx: which = 0: host->device bytes copied (image
 * upload; 0 when the identical image was already resident), 1: device->host bytes,
 * 2: number of CUDA kernels launched.  Returns 0 for an unknown `which`. */
uint64_t paradl_stat(const paradl_ctx *ctx, int32_t which);

/* Roofline denominator: runs an FP64 FMA-chain microbenchmark on the ctx's device for
 * about `ms` milliseconds and returns the sustained FP64 pipe rate in DFMA instructions
 * per second (one DFMA = 2 FLOP).  Not part of the cost model. */
paradl_status paradl_fp64_peak(paradl_ctx *ctx, double ms, double *inst_per_s);

/* Sizes of the ABI structs, for binding self-checks. */
int32_t paradl_struct_size(int32_t which);   /* 0 layer, 1 system, 2 subsweep, 3 config, 4 prediction, 5 hit */

#ifdef __cplusplus
}
#endif
#endif /* PARADL_H */
