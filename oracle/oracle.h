/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU evaluation of ParaDL's cost model
 * (arXiv 2104.09075, Table 2 P:455-516 and Appendix A.1).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  It shares no code, header, table or helper
 * with the CUDA product (paper_2104_09075_b200/, include/paradl.h): every
 * struct below is the oracle's own.
 *
 * Readings of the paper used here are listed in DESIGN.md §2 (Q1..Q33).
 * Parity status: see the header of oracle.c.
 */
#ifndef PARADL_ORACLE_H
#define PARADL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_CONV = 0, OR_FC = 1, OR_POOL = 2, OR_ELEM = 3, OR_NORM = 4 };
enum { OR_FLAG_COMM = 1, OR_FLAG_FOLDED = 4 };
enum { OR_SERIAL = 0, OR_DATA, OR_SPATIAL, OR_FILTER, OR_CHANNEL, OR_DF, OR_DS,
       OR_PIPELINE, OR_LAYERPURE, OR_PD,
       OR_SPATIAL_AG,   /* spatial on the first Ls rows, Allgather, replicated rest (Q35) */
       OR_GPIPE,        /* pipeline timed by the GPipe schedule itself (Q36) */
       OR_DATA_LW,      /* data parallel, one gradient Allreduce per weighted layer, each message
                         * ring or tree by its size (Q37) */
       OR_LAYERWISE,    /* per-layer strategy: every COMM row data- or filter-parallel over the
                         * same p PEs, with activation exchanges at strategy changes (P:413,
                         * P:450; Q39).  MASK partition radix over the COMM rows. */
       OR_N_FAMILIES };
enum { OR_PART_NONE = 0, OR_PART_COMB = 1, OR_PART_MASK = 2 };
/* infeasibility reasons (bit set) */
enum { OR_R_SCALING = 1, OR_R_MEMORY = 2, OR_R_SPLIT = 4, OR_R_TIER = 8, OR_R_SEGMENTS = 16 };
enum { OR_MAX_TIERS = 4, OR_MAX_STAGES = 64 };

typedef struct {
    int32_t kind, ndim;
    int64_t C, F, X[3], Y[3], K[3];
    int64_t x, y, w, bi, fw, bw, wu;
    uint32_t flags, pad_;
} or_layer;

typedef struct {
    int32_t G, pad_;
    const or_layer *rows;
    int64_t D;                         /* dataset size (Table 1) */
} or_model;

typedef struct { int64_t max_pes; double alpha, beta; } or_tier;

typedef struct {
    int32_t n_tiers, delta;
    or_tier tiers[OR_MAX_TIERS];
    double flops_per_s, hbm_bytes, gamma, phi_df, tree_threshold;
    int32_t tree_chunks, filter_rs;   /* filter_rs: backward dL/dx exchange as Reduce-Scatter (P:355 fn) */
    /* f1 (Q40): point-to-point patterns (halo exchange, pipeline boundary
     * sends) use the tier's alpha x p2p_alpha_scale and beta x p2p_beta_scale (e.g. MPI vs
     * NCCL); phi_pd / phi_ds: contention on the pd stage Allreduces (s > 1 concurrent groups)
     * and on the ds reduce-to-leader (p1 > 1 concurrent groups).  All 1 = Table 2 literal. */
    double p2p_alpha_scale, p2p_beta_scale, phi_pd, phi_ds;
} or_system;

typedef struct {
    int32_t family, model;
    int32_t part_mode, s_min, s_max;
    int32_t n_cap, n_flops, n_b, n_S, n_dims, n_Ls, n_alpha, n_beta, pad_;
    const double *cap, *flops;
    const int64_t *b;
    const int32_t *S, *dims /* n_dims x 4 */, *Ls;
    const double *alpha /* n_alpha x n_tiers */, *beta /* n_beta x n_tiers */;
} or_sub;

typedef struct { int32_t n_sub, pad_; const or_sub *subs; } or_spec;

typedef struct {
    int32_t sub, family, model, pad_;
    int64_t i_cap, i_flops, i_b, i_S, i_dims, i_Ls, i_alpha, i_beta;
    uint64_t i_part;
    double cap, flops;
    int64_t b;
    int32_t S, Ls, dims[4];
    double alpha[OR_MAX_TIERS], beta[OR_MAX_TIERS];
    int32_t n_stages, pad2_;
    int32_t stage_end[OR_MAX_STAGES];   /* rows in stages 1..i (exclusive end, 0-based) */
} or_config;

typedef struct {
    double t_comp, t_ge, t_fb_ag, t_fb_ar, t_halo, t_p2p, t_iter, t_epoch, mem, I;
    int64_t B, p;
    uint32_t reason;
    int32_t feasible;
} or_pred;

typedef struct { uint64_t idx; double key; } or_hit;

/* 0 on success, <0 on a malformed input (message in or_last_error()). */
const char *or_last_error(void);
int or_sweep_size(const or_model *models, int n_models, const or_system *sys,
                  const or_spec *spec, uint64_t *n_out);
int or_decode(const or_model *models, int n_models, const or_system *sys,
              const or_spec *spec, uint64_t idx, or_config *out);
/* canonical evaluation (exact integer sums; one fixed fp64 tree per term) */
int or_eval(const or_model *models, const or_system *sys, const or_config *cfg, or_pred *out);
/* literal per-layer fp64 left fold of Table 2 as printed (checks the factoring) */
int or_eval_fold(const or_model *models, const or_system *sys, const or_config *cfg, or_pred *out);
/* halo volume of one row for a split (elements per sample), which=0: halo(x), 1: halo(dL/dy) */
int64_t or_halo_elements(const or_layer *row, const int32_t split[3], int which);

int or_eval_many(const or_model *models, int n_models, const or_system *sys,
                 const or_spec *spec, const uint64_t *idx, int64_t n,
                 double *t_iter, double *mem, uint32_t *reason, double *key, int nthreads);
int or_sweep_dense(const or_model *models, int n_models, const or_system *sys,
                   const or_spec *spec, uint64_t first, uint64_t count,
                   double *t_iter, double *mem, uint32_t *feasible_bits, uint8_t *reason,
                   int nthreads);
int or_topk(const or_model *models, int n_models, const or_system *sys,
            const or_spec *spec, uint64_t first, uint64_t count, int32_t k,
            or_hit *hits, uint64_t *n_feasible, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
