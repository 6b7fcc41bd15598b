/*
 * rplu_b200.h — C ABI of the B200-native Randomly Pivoted LU pivot loop.
 *
 * The reference (`rplu` 0.1.0, pure Python/numpy) has no FFI; this ABI is the
 * drop-in boundary its three hot entry points bind to through ctypes
 * (see INTEGRATION.md):
 *
 *   rplu_dense_run   replaces the loop of rplu.dense_pivots.eliminate
 *                    (pkg/src/rplu/dense_pivots.py:129-209, rank-1 rules
 *                    rplu / c2plu / cplu, _draw_rank1_pivot :103-126)
 *   rplu_cauchy_run  replaces rplu.cauchy.structured_eliminate with plan=None
 *                    (pkg/src/rplu/cauchy.py:177-256) and exact_row_norms
 *                    (cauchy.py:129-137)
 *   rplu_gauss_*, rplu_cur_downdate, rplu_sample_index
 *                    the device primitives of rplu.lowmem_cur.cur_build
 *                    (pkg/src/rplu/lowmem_cur.py:212-300) for the
 *                    Gaussian-kernel operator; the host driver sequences them
 *   rplu_mf_run      the whole loop of rplu.lowmem_cur.cur_build on the device
 *                    (Gaussian-kernel or dense real operator)
 *   rplu_lu_error    the fused L.U reconstruction error (K11, FP64 tensor cores)
 *   rplu_shard_*     row-block sharded eliminate across GPUs
 *
 * Conventions
 *   - extern "C", plain pointers and sizes, no exceptions cross the ABI.
 *   - Every call returns an int status: RPLU_OK (0) or a negative error class;
 *     rplu_last_error() returns a thread-local message for the last failure.
 *   - "device" pointers are CUDA device addresses on the context's GPU; the
 *     library never frees caller memory.  "host" pointers are CPU memory.
 *   - The caller's uniform stream is passed as a host array of doubles in
 *     [0,1) drawn in order from the reference's RngState; the call reports how
 *     many it consumed so the caller can advance its generator exactly.
 *   - Calls are synchronous with respect to the host: on return all results
 *     are in the caller's buffers.  One context per host thread.
 */
#ifndef RPLU_B200_H
#define RPLU_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RPLU_B200_ABI_VERSION 2

/* status codes (negative = error class; mapped to Python exceptions) */
#define RPLU_OK 0
#define RPLU_ERR_ARG (-1)        /* ValueError        (bad argument / range) */
#define RPLU_ERR_ZERO_PIVOT (-2) /* ZeroDivisionError (pivot zero after resample) */
#define RPLU_ERR_CAPABILITY (-3) /* CapabilityError   (unsupported operation) */
#define RPLU_ERR_CUDA (-4)       /* RuntimeError      (CUDA failure) */

/* element types of the residual / generators */
#define RPLU_F32 1
#define RPLU_F64 2
#define RPLU_C128 3

/* flags */
#define RPLU_FLAG_TIME_KERNELS 1 /* bracket K2/K3 launches with CUDA events */
#define RPLU_FLAG_NO_GRAPH 2     /* never capture the step loop into a CUDA graph */
#define RPLU_FLAG_LAZY 4         /* dense: force the delayed-update loop */
#define RPLU_FLAG_EAGER 8        /* dense: force the eager (update every step) loop;
                                    default: delayed updates when R exceeds L2 */
#define RPLU_FLAG_STEPWISE 16   /* dense / Cauchy-like: per-step launches even where the whole
                                    loop would run as one resident cooperative launch */
#define RPLU_FLAG_NO_GRAM 64    /* dense fp64 delayed-update loop: compute each step's
                                    masses by applying the pending terms (2q FP64 operations
                                    per element) instead of from the Gram form (one dot
                                    product per element, flush every 16 steps) */
#define RPLU_FLAG_EXACT 32      /* dense delayed-update loop: apply the pending rank-1 terms
                                    with the reference's rounding (multiply, then subtract:
                                    bit-identical to the eager loop and to the reference's
                                    arithmetic; the Python layer always sets it unless
                                    fused_updates=True); without it: one FMA per term (L/U
                                    agree to rounding, half the FP64 work) */

/* pivot rules: rplu (random, 2 uniforms/step), c2plu / cplu (greedy) */
#define RPLU_RULE_RPLU 0
#define RPLU_RULE_C2PLU 1
#define RPLU_RULE_CPLU 2

typedef struct rplu_ctx rplu_ctx;

int rplu_abi_version(void);
/* Kernels launched so far (process-wide) by the standalone primitives
 * (rplu_gauss_*, rplu_cur_downdate, rplu_sample_index, rplu_loewner_fill,
 * rplu_bary_eval, rplu_mgs_arnoldi); the loop drivers report their own
 * counts in their out structs. */
int64_t rplu_kernel_launch_count(void);
const char* rplu_last_error(void);

/* Create a context bound to CUDA device `device` (workspace is grown lazily). */
int rplu_ctx_create(int device, rplu_ctx** out);
int rplu_ctx_destroy(rplu_ctx* ctx);

/* ------------------------------------------------------------------------ */
/* Dense Alg 1 (eliminate).                                                  */

typedef struct rplu_dense_args {
  int32_t dtype;          /* RPLU_F32 | RPLU_F64 | RPLU_C128 */
  int32_t rule;           /* RPLU_RULE_* */
  int64_t n, m;           /* residual shape */
  int64_t ld;             /* row stride of R in elements (>= m) */
  int64_t steps;          /* pivots requested, 0 <= steps <= min(n, m) */
  double stop_tol;        /* >= 0; tol stop when ||R||_F <= stop_tol*||A||_F */
  void* R;                /* device: n x ld, row-major, overwritten by the residual */
  void* Lt;               /* device: steps x n; row t holds column t of L */
  void* U;                /* device: steps x ldu; row t of U */
  int64_t ldu;            /* row stride of U in elements (>= m) */
  const double* uniforms; /* host: uniform stream (rule rplu), may be NULL otherwise */
  int64_t n_uniforms;     /* length of `uniforms` (4*steps always suffices) */
  void* stream;           /* cudaStream_t to run on (NULL = legacy default) */
  int32_t flags;          /* RPLU_FLAG_* */
  int32_t reserved;
} rplu_dense_args;

typedef struct rplu_dense_out {
  int64_t* pivots;              /* host, caller-owned, >= 2*steps: i0,j0,i1,j1,... */
  double* resid_fro;            /* host, caller-owned, >= steps+1 */
  int64_t steps_done;           /* pivots taken */
  int64_t uniforms_consumed;    /* uniforms read from the stream */
  int64_t near_boundary_draws;  /* draws within 1e-12 relative of a CDF boundary */
  int32_t clean_early_stop;     /* residual exactly zero before `steps` */
  int32_t tol_stop;             /* stop_tol reached */
  int64_t zero_pivot_i;         /* set with RPLU_ERR_ZERO_PIVOT */
  int64_t zero_pivot_j;
  /* with RPLU_FLAG_TIME_KERNELS: CUDA-event time summed over the launches of
   * the fused Schur-update kernel (K3) and of the select kernel (K2), and the
   * number of library kernels launched by the call */
  double sweep_ms;
  double select_ms;
  int64_t sweep_launches;
  int64_t kernel_launches;
  /* algorithmic HBM bytes of the timed update launches (2*n*m*s for an eager
   * update or a lazy flush, n*m*s for a lazy read-only pass), and the
   * delayed-update flush interval used (0 = eager loop) */
  double sweep_bytes;
  int64_t lazy_block;
} rplu_dense_out;

int rplu_dense_run(rplu_ctx* ctx, const rplu_dense_args* args, rplu_dense_out* out);

/* ------------------------------------------------------------------------ */
/* Row-block sharded dense RPLU (one rank per GPU).  The host
 * driver (paper_2601_22344_b200.distributed) interleaves these calls with two
 * collectives per step on the same stream:
 *   begin -> allgather(local_total) ->
 *   for t: select(t) -> allreduce_sum(msg) -> update(t) -> allgather(local_total)
 *   select(steps) (final residual norm) -> finish.
 * With t = -1 the kernels read the step from a device counter, so one step
 * (kernels + collectives) can be captured in a CUDA graph and replayed.
 * Non-owning ranks contribute -0.0, so the sums reproduce the owner's bits.
 * With lazy_block != 0 the local rows take the delayed-update loop of
 * rplu_dense_run (one read of the row block per step, a write every block
 * steps; the owner rebuilds its pivot row on the fly) and finish applies the
 * pending steps after an early stop; the results are bit-identical. */

typedef struct rplu_shard_args {
  int32_t dtype;          /* RPLU_F32 | RPLU_F64 | RPLU_C128 */
  int32_t world, rank;    /* shard count and this shard's index */
  int32_t lazy_block;     /* 0: eager K3 update; > 0 (<= 16): delayed-update
                           * block (flush every lazy_block steps; 16-byte
                           * aligned rows of R and U); < 0: the default (fp64:
                           * Gram-form masses, flush every 16 steps; else
                           * 6 / 5).  rplu_shard_lazy_block resolves it. */
  int64_t n_local, m;     /* local row block shape */
  int64_t ld;             /* row stride of R (elements) */
  int64_t row_offset;     /* global index of local row 0 */
  int64_t steps;
  double stop_tol;
  void* R;                /* device: n_local x ld residual rows, updated in place */
  void* Lt;               /* device: steps x n_local (local rows of L, transposed) */
  void* U;                /* device: steps x ldu (replicated on every rank) */
  int64_t ldu;
  const double* uniforms; /* host uniform stream (uploaded by begin) */
  int64_t n_uniforms;
  void* stream;
} rplu_shard_args;

/* K1 masses of the local rows, state reset, uniforms upload; writes the local
 * mass total to local_total (device double). */
int rplu_shard_begin(rplu_ctx* ctx, const rplu_shard_args* a, double* local_total);
/* Global owner selection from totals[world] (device), owner's row/column draw;
 * writes the pivot message msg (device, 32 + m*sizeof(element) bytes):
 * [i_global, j, a_re, a_im] as fp64, then the pivot row (owner bits, or -0.0
 * on the other ranks).  t < 0: take the step from the device counter. */
int rplu_shard_select(rplu_ctx* ctx, const rplu_shard_args* a, int64_t t, const double* totals,
                      void* msg);
/* Post the reduced message (state + U[t,:]), K3 fused update of the local
 * rows, local total; advances the device step counter.  Delayed-update
 * shards with t < 0: -1 - t is the step's position inside its block of
 * lazy_block steps (the number of pending terms and the flush at the last
 * position are fixed at launch, the absolute step comes from the device
 * counter), so one whole block -- kernels and collectives -- is captured
 * once and replayed; a trailing partial block runs with explicit t. */
int rplu_shard_update(rplu_ctx* ctx, const rplu_shard_args* a, int64_t t, const void* msg,
                      double* local_total);
/* The flush interval the shard calls use for these arguments (0: eager). */
int rplu_shard_lazy_block(const rplu_shard_args* a);
/* 1 if the loop is still running (synchronizes the stream). */
int rplu_shard_active(rplu_ctx* ctx, const rplu_shard_args* a, int32_t* active);
/* Copy pivots / residual norms / flags to the host (out as for rplu_dense_run). */
int rplu_shard_finish(rplu_ctx* ctx, const rplu_shard_args* a, rplu_dense_out* out);

/* The same sharded elimination driven entirely from C across the GPUs of one
 * node: one host thread, NCCL communicators from ncclCommInitAll (libnccl is
 * loaded at run time), per step the shard select on every device, one grouped
 * ncclAllReduce(sum) of the pivot message, the shard update and one grouped
 * ncclAllGather of the shard totals (SURVEY §8(b) rplu_ctx_create(ngpus,
 * devs), §8(e)).  A group owns one context and one stream per device. */
typedef struct rplu_group rplu_group;
int rplu_group_create(int32_t ngpus, const int32_t* devs, rplu_group** out);
int rplu_group_destroy(rplu_group* g);

typedef struct rplu_group_shard {
  void* R;              /* device (on devs[d]): n_local x ld rows, updated in place */
  void* Lt;             /* device: steps x n_local */
  void* U;              /* device: (steps + 1) x ldu, replicated */
  int64_t n_local, ld, row_offset;
} rplu_group_shard;

typedef struct rplu_group_dense_args {
  int32_t dtype;
  int32_t lazy_block;   /* as rplu_shard_args.lazy_block (0: eager, < 0: default) */
  int64_t m, steps, ldu;
  double stop_tol;
  const double* uniforms;  /* host */
  int64_t n_uniforms;
  const rplu_group_shard* shards;  /* [ngpus], contiguous row blocks in device order */
} rplu_group_dense_args;

/* Replicated results (pivots, resid_fro, flags) in out, as rplu_dense_run;
 * each shard's L rows stay in its Lt, U is replicated in every shard's U. */
int rplu_group_dense_run(rplu_group* g, const rplu_group_dense_args* a, rplu_dense_out* out);

/* Squared row masses sum_j |R_ij|^2 of a device matrix (K1), written to the
 * device array `masses` (n doubles).  Used by the sharded driver for step 0
 * and by accessors' row_norms(). */
int rplu_row_masses(rplu_ctx* ctx, int32_t dtype, const void* R, int64_t n, int64_t m,
                    int64_t ld, double* masses, void* stream);

/* ------------------------------------------------------------------------ */
/* Cauchy-like structured elimination, exact row norms (structured_eliminate,
 * plan=None).  Entries A_ij = (G_i . B_:,j) / (x_i - y_j), complex128.      */

typedef struct rplu_cauchy_args {
  int32_t rule;           /* RPLU_RULE_RPLU | RPLU_RULE_C2PLU */
  int32_t p;              /* displacement rank, 1..8 */
  int64_t n, m;           /* shape */
  int64_t rank;           /* pivots requested, 0 <= rank <= min(n, m) */
  double stop_tol;        /* stop when max_i u_i <= stop_tol^2 * max_i u_i^(0) */
  const void* x;          /* device complex128[n] */
  const void* y;          /* device complex128[m] */
  void* G;                /* device complex128 n x p row-major; updated in place */
  void* Bt;               /* device complex128 m x p row-major (column j of B
                             contiguous = the reference's F-order B); updated */
  void* C;                /* device complex128 rank x n: column c of each step, or NULL */
  void* Rrow;             /* device complex128 rank x m: row r of each step, or NULL */
  void* a;                /* device complex128[rank]: pivot values, or NULL */
  const double* uniforms; /* host uniform stream (rule rplu; 3*rank suffices) */
  int64_t n_uniforms;
  void* stream;
  int32_t flags;          /* RPLU_FLAG_* */
  int32_t reserved;
} rplu_cauchy_args;

typedef struct rplu_cauchy_out {
  int64_t* rows;          /* host, caller-owned, >= rank: pivot rows */
  int64_t* cols;          /* host, caller-owned, >= rank: pivot columns */
  double* bound_maxes;    /* host, >= rank: max_i u_i at the start of each step */
  double* bound_sums;     /* host, >= rank: sum_i u_i at the start of each step */
  int64_t steps_done;
  int64_t bounds_recorded;
  int64_t uniforms_consumed;
  int64_t near_boundary_draws;
  int32_t tol_stop;
  int32_t degenerate_stop;
  int64_t zero_pivot_i, zero_pivot_j;
  double masses_ms;       /* RPLU_FLAG_TIME_KERNELS: CUDA-event time of K5 */
  int64_t masses_launches;
  int64_t kernel_launches;
} rplu_cauchy_out;

int rplu_cauchy_run(rplu_ctx* ctx, const rplu_cauchy_args* args, rplu_cauchy_out* out);

/* Row-block sharded Cauchy-like RPLU: x and G are sharded
 * by rows, y and B replicated (B updated redundantly on every rank).  Per step
 * the host driver runs
 *   select(t) -> allreduce_sum(msg) -> update(t) -> allgather(local_stats)
 * where local_stats = [sum_i u_i, max_i u_i] of the local rows (device
 * doubles) and totals = the allgathered [world][2] stats.  The owner shard
 * (CDF over shard sums with u1, or the first shard holding the global max
 * for c2plu) writes the pivot message msg (RPLU_CAUCHY_MSG_DOUBLES fp64):
 * [i_global, 0, x_i (re, im), G_i (p complex)]; the other ranks write -0.0.
 * update regenerates the pivot row r from the message on every rank
 * (identical bits), draws the column with u2 (same draw everywhere), and
 * updates the local G rows and all of B, then K5 masses of the local rows.
 * With C / Rrow / a set, the kept steps hold the LOCAL c rows (rank x
 * n_local).  Host step loop (t >= 0); no tree plan on this path. */
#define RPLU_CAUCHY_MSG_DOUBLES 20

typedef struct rplu_cauchy_shard_args {
  int32_t rule;           /* RPLU_RULE_RPLU | RPLU_RULE_C2PLU */
  int32_t p;              /* displacement rank, 1..8 */
  int32_t world, rank;    /* shard count and this shard's index */
  int64_t n_local, m;     /* local rows, all columns */
  int64_t row_offset;     /* global index of local row 0 */
  int64_t steps;          /* pivots requested (the global rank) */
  double stop_tol;
  const void* x;          /* device complex128[n_local] (local rows) */
  const void* y;          /* device complex128[m] (replicated) */
  void* G;                /* device complex128 n_local x p (local rows) */
  void* Bt;               /* device complex128 m x p (replicated) */
  void* C;                /* device complex128 steps x n_local, or NULL */
  void* Rrow;             /* device complex128 steps x m, or NULL */
  void* a;                /* device complex128[steps], or NULL */
  const double* uniforms; /* host uniform stream (uploaded by begin) */
  int64_t n_uniforms;
  void* stream;
} rplu_cauchy_shard_args;

int rplu_cauchy_shard_begin(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, double* local_stats);
int rplu_cauchy_shard_select(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, int64_t t,
                             const double* totals, void* msg);
int rplu_cauchy_shard_update(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, int64_t t,
                             const void* msg, double* local_stats);
int rplu_cauchy_shard_active(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, int32_t* active);
int rplu_cauchy_shard_finish(rplu_ctx* ctx, const rplu_cauchy_shard_args* a,
                             rplu_cauchy_out* out);

/* Certified row-norm upper bounds from a quadtree interaction plan
 * (treebounds.py:213-242, Alg C.2): exact <= u_i <= nu*exact.  The plan is
 * built on the host (Alg C.1, paper_2601_22344_b200.treebounds.build_plan)
 * and flattened into device CSR arrays (int64 / fp64). */
typedef struct rplu_tree_plan {
  int64_t n, m;            /* target / source point counts */
  int32_t p;               /* displacement rank */
  int32_t n_levels;        /* internal-node levels (ABI 2) */
  int64_t n_tleaves;       /* target leaves */
  const int64_t* tperm;    /* [n] target points grouped by leaf */
  const int64_t* tstart;   /* [n_tleaves+1] */
  const int64_t* agg_start;  /* [n_tleaves+1] aggregated list per leaf */
  const int64_t* agg_node;   /* source node of each aggregated entry */
  const double* agg_alpha;   /* 1 / d_min^2(node, leaf) */
  const int64_t* ex_start;   /* [n_tleaves+1] exact list per leaf */
  const int64_t* ex_leaf;    /* source leaf index of each exact entry */
  int64_t n_snodes, n_sleaves;
  const int64_t* spts;     /* [m] source points grouped by source leaf */
  const int64_t* sstart;   /* [n_sleaves+1] */
  const int64_t* cstart;   /* [n_snodes+1] children of each source node (CSR) */
  const int64_t* cidx;
  const int64_t* leaf_node;  /* [n_sleaves] node id of each source leaf */
  const int64_t* lvl_nodes;  /* internal nodes grouped by level, deepest first */
  const int64_t* lvl_start;  /* HOST array [n_levels+1]: level slices of lvl_nodes */
} rplu_tree_plan;

int rplu_tree_bounds(rplu_ctx* ctx, const rplu_tree_plan* plan, const void* x, const void* y,
                     const void* G, const void* Bt, double* u, void* stream);

/* Plan-path step primitives (structured_eliminate with a plan,
 * cauchy.py:207-277), driven by the host rejection loop:
 *   rplu_cauchy_plan_row: pivot row r = (G_i . B)/(x_i - y) into rbuf[m]
 *     (complex128) and |r|^2 into wbuf[m] (numpy-exact arithmetic); out3 =
 *     {sum_j |r_j|^2, max_j |r_j|, bounds[i] (0 if bounds is NULL)} on the
 *     host (synchronous);
 *   rplu_cauchy_plan_update: with a = rbuf[j], G -= (c/a) G_i and
 *     B_:,l -= B_:,j (r_l/a) in place (c = column j); optional Cout[n] = c
 *     and Rout[m] = r (kept steps).  Asynchronous on `stream`. */
int rplu_cauchy_plan_row(rplu_ctx* ctx, int32_t p, int64_t n, int64_t m, const void* x,
                         const void* y, void* G, void* Bt, int64_t i, void* rbuf, double* wbuf,
                         const double* bounds, double* out3, void* stream);
int rplu_cauchy_plan_update(rplu_ctx* ctx, int32_t p, int64_t n, int64_t m, const void* x,
                            const void* y, void* G, void* Bt, int64_t i, int64_t j,
                            const void* rbuf, void* Cout, void* Rout, void* stream);
/* One proposal of the rejection loop (cauchy.py:236-250) in a single host
 * synchronisation: i = sample_index(bounds, u), then rplu_cauchy_plan_row for
 * that i.  out5 = {i, near-boundary flag of the draw, sum_j |r_j|^2,
 * max_j |r_j|, bounds[i]}. */
int rplu_cauchy_plan_propose(rplu_ctx* ctx, int32_t p, int64_t n, int64_t m, const void* x,
                             const void* y, void* G, void* Bt, const double* bounds, double u,
                             void* rbuf, double* wbuf, double* out5, void* stream);

/* Host-native interaction-plan build (no GPU needed), replacing the Python
 * quadtrees and dual traversal of rplu.treebounds.build_plan
 * (treebounds.py:47-104, :141-180) with identical results.  x: n complex
 * points (re, im pairs), y: m.  On coincident target / source points returns
 * RPLU_ERR_ARG with coincident[0] = target index, coincident[1] = source
 * index (CoincidentPointsError in the Python layer). */
typedef struct rplu_plan_host rplu_plan_host;
int rplu_plan_build(const double* x, int64_t n, const double* y, int64_t m, double nu,
                    int64_t leaf_size, int64_t* coincident, rplu_plan_host** out);
/* counts[8]: target nodes, target leaves, target child links, source nodes,
 * source leaves, source child links, aggregated entries, exact entries */
int rplu_plan_counts(const rplu_plan_host* h, int64_t* counts);
/* which = 0 target tree, 1 source tree: node boxes (x0, y0, size), parent,
 * children CSR (cstart[nodes+1], cidx), leaves in traversal order and their
 * points (lpstart[leaves+1], lpidx) */
int rplu_plan_tree(const rplu_plan_host* h, int32_t which, double* x0, double* y0, double* size,
                   int64_t* parent, int64_t* cstart, int64_t* cidx, int64_t* leaves,
                   int64_t* lpstart, int64_t* lpidx);
/* per target leaf (target-leaf order): aggregated (source node, alpha) and
 * exact (source node) lists as CSR */
int rplu_plan_lists(const rplu_plan_host* h, int64_t* agg_start, int64_t* agg_node,
                    double* agg_alpha, int64_t* ex_start, int64_t* ex_node);
int rplu_plan_free(rplu_plan_host* h);

/* exact_row_norms (cauchy.py:129-137): u_i = sum_j |G_i.B_:,j / (x_i-y_j)|^2
 * into the device array `out` (n doubles). */
int rplu_cauchy_row_norms(rplu_ctx* ctx, int32_t p, int64_t n, int64_t m, const void* x,
                          const void* y, const void* G, const void* Bt, double* out,
                          void* stream);

/* ------------------------------------------------------------------------ */
/* Matrix-free CUR-form Alg 2 (cur_build) for the Gaussian-kernel operator
 * A_ij = exp(-|p_i - q_j|^2 / (2 h^2)).  The Python driver
 * (paper_2601_22344_b200.lowmem_cur.cur_build, mirroring lowmem_cur.py:212-300)
 * sequences these device primitives; every vector is a device fp64 array. */

typedef struct rplu_gauss_op {
  int64_t n, m;
  const double* P;  /* device n x 3 row-major: points p_i */
  const double* Q;  /* device m x 3 row-major: points q_j */
  double h;         /* bandwidth (> 0) */
} rplu_gauss_op;

/* K7 full generated GEMV: adjoint=0: out[n] = A v[m]; adjoint=1: out[m] = A^T v[n]
 * (accessor apply / adjoint_apply, accessors.py:36-90).  *kernel_ms (optional)
 * receives the CUDA-event time of the generated-entry kernel. */
int rplu_gauss_apply(rplu_ctx* ctx, const rplu_gauss_op* op, int32_t adjoint, const double* v,
                     double* out, double* kernel_ms, void* stream);
/* squared row norms sum_j A_ij^2 into out[n] (row_norms()) */
int rplu_gauss_row_norms(rplu_ctx* ctx, const rplu_gauss_op* op, double* out, void* stream);
/* axis=0: out[m] = A[index, :];  axis=1: out[n] = A[:, index] */
int rplu_gauss_line(rplu_ctx* ctx, const rplu_gauss_op* op, int32_t axis, int64_t index,
                    double* out, void* stream);
/* K8 k-restricted products: axis=0: out[m] = A[sel, :]^T w;  axis=1: out[n] = A[:, sel] w
 * (sel: device int64[k], w: device fp64[k]); replaces lowmem_cur.py:174-187. */
int rplu_gauss_restricted(rplu_ctx* ctx, const rplu_gauss_op* op, int32_t axis,
                          const int64_t* sel, const double* w, int64_t k, double* out,
                          void* stream);
/* K9 row-norm downdate (lowmem_cur.py:277-285): nrow -= 2 (g - v) chat;
 * nrow += l2 chat^2; count entries < -floor; clip at 0; *total = sum(nrow). */
int rplu_cur_downdate(rplu_ctx* ctx, int64_t n, double* nrow, const double* g, const double* v,
                      const double* chat, double l2, double floor, int64_t* clamped,
                      double* total, void* stream);

/* K11 error evaluation: out_sq[0] = ||A - L U||_F^2 and
 * out_sq[1] = ||A||_F^2 in one fused FP64-tensor-core kernel (DMMA), with no
 * L U panel in memory.  Replaces the reconstruction the reference's error
 * measures form, EliminationTrace.approximation() = L @ U and
 * np.linalg.norm(dense - approx) (dense_pivots.py:82-83, cli.py:151-157,
 * :200-206).  A: device n x m row-major (lda elements), dtype F32 / F64 /
 * C128; L is passed transposed as Lt: device k x n (ldl) -- the layout
 * rplu_dense_run fills -- and U: device k x m (ldu), both of A's dtype.
 * *kernel_ms (optional): CUDA-event time of the product kernel(s). */
int rplu_lu_error(rplu_ctx* ctx, int32_t dtype, const void* A, int64_t lda, int64_t n, int64_t m,
                  const void* Lt, int64_t ldl, const void* U, int64_t ldu, int64_t k,
                  double* out_sq, double* kernel_ms, void* stream);

/* ------------------------------------------------------------------------ */
/* Device-resident matrix-free CUR-form Alg 2 (cur_build,                    */
/* lowmem_cur.py:212-300, with _rebuild_row_norms :204-209).                 */
/* The whole loop runs in the library: per step the row / column draws,      */
/* residual row and column (k-restricted generated products), the one full   */
/* operator pass g = A l, the row-norm downdate with clamp count, the core    */
/* extension (an O(k^2) LU update of W = A[I,J] in selection order instead   */
/* of the reference's per-step QR) and, on > 1% clamps, the rebuild -- one    */
/* host synchronisation per step, no host arithmetic.                        */

#define RPLU_MF_GAUSS3D 1  /* A_ij = exp(-|p_i - q_j|^2 / (2 h^2)), points P (n x 3), Q (m x 3) */
#define RPLU_MF_DENSE 2    /* real dense A (n x m row-major, lda), float64, device */

typedef struct rplu_mf_args {
  int32_t op_kind;   /* RPLU_MF_GAUSS3D | RPLU_MF_DENSE */
  int32_t rule;      /* RPLU_RULE_RPLU (rplu-cur) | RPLU_RULE_C2PLU (c2plu-cur) */
  int64_t n, m, rank;
  double stop_tol;
  const double* P;   /* device (GAUSS3D) */
  const double* Q;   /* device (GAUSS3D) */
  double h;          /* bandwidth (GAUSS3D) */
  const double* A;   /* device (DENSE) */
  int64_t lda;       /* DENSE */
  const double* uniforms; /* host: the caller's stream, row draw then column draw per step */
  int64_t n_uniforms;
  void* stream;
  int32_t flags;     /* RPLU_FLAG_TIME_KERNELS: time the full operator passes */
  int32_t reserved;
} rplu_mf_args;

typedef struct rplu_mf_out {
  int64_t* rows;            /* host [rank]: I in selection order */
  int64_t* cols;            /* host [rank]: J */
  double* total_sq_norms;   /* host [rank + 1]: sum of the maintained row norms */
  int64_t* clamped;         /* host [rank] (optional) */
  double* core;             /* host [rank * rank] (optional): W = A[I, J], row-major k x k */
  double* row_norms;        /* host [n] (optional): final maintained row norms */
  double* row_norms_dev;    /* device [n] (optional) */
  int64_t steps_done, uniforms_consumed, near_boundary_draws, rebuilds;
  int32_t degenerate_stop, tol_stop, core_fell_back, reserved;
  double gemv_ms;           /* summed CUDA-event time of the full operator passes (TIME flag) */
  int64_t kernel_launches;
} rplu_mf_out;

int rplu_mf_run(rplu_ctx* ctx, const rplu_mf_args* args, rplu_mf_out* out);

/* Copy `bytes` from a pageable host buffer to device memory through the
 * context's ring of page-locked slots (`threads` host threads fill a slot
 * while the previous one is in flight).  Ordered on `stream`; the source is
 * no longer read on return.  The Python layer uses it for numpy inputs (the
 * reference's callers pass plain arrays, dense_pivots.py:86-89). */
int rplu_upload(rplu_ctx* ctx, void* dst, const void* src, int64_t bytes, int32_t threads,
                void* stream);

/* Diagnostic: measured FP64 FMA-pipe throughput of the context's GPU
 * (TFLOP/s, best of 5), the roofline denominator of the generated-entry
 * (Cauchy-like, Gaussian-kernel) kernels. */
int rplu_diag_fp64_peak(rplu_ctx* ctx, double* tflops, double* best_ms);

/* Diagnostic: measured FP64 tensor-core (DMMA m8n8k4) throughput, the K11
 * roofline denominator (TFLOP/s, best of 5). */
int rplu_diag_dmma_peak(rplu_ctx* ctx, double* tflops, double* best_ms);

/* sample_index(weights, u) on a device weight vector (rng.py:50-74):
 * first index whose running sum exceeds u*total, top clamp, walk-back over
 * zero weights.  RPLU_ERR_ARG for empty / negative / all-zero weights.
 * *near_boundary (optional) is set to 1 if the draw is within 1e-12*total of
 * a CDF boundary. */
int rplu_sample_index(rplu_ctx* ctx, const double* weights, int64_t n, double u,
                      int64_t* out_index, int32_t* near_boundary, void* stream);
/* The same draw plus the element gather[index] of a device complex128 array
 * (value[0..1] = re, im) in one host synchronisation: the plan path's column
 * draw and pivot value. */
int rplu_sample_index_gather(rplu_ctx* ctx, const double* weights, int64_t n, double u,
                             const void* gather, int64_t* out_index, int32_t* near_boundary,
                             double* value, void* stream);

/* The same search against an ABSOLUTE target in [0, total] (first index whose
 * running sum exceeds target; clamp / walk-back as above): the owner shard's
 * local draw in a row-sharded elimination, where target = u*T_global minus
 * the totals of the shards before it. */
int rplu_sample_target(rplu_ctx* ctx, const double* weights, int64_t n, double target,
                       int64_t* out_index, int32_t* near_boundary, void* stream);

/* Total of the weights in the CDF code's summation order (the per-shard
 * totals the shard CDF is formed from); host result. */
int rplu_cdf_total(rplu_ctx* ctx, const double* weights, int64_t n, double* total, void* stream);


/* ------------------------------------------------------------------------ */
/* Downstream consumers of the pivots and the CUR core.
 * All vectors are device complex128 ({re, im} double pairs). */

/* Loewner (divided-difference) matrix, row-major no x k:
 * out[i*k + j] = (fo[i] - fs[j]) / (zo[i] - zs[j])  (numpy-exact elementwise
 * arithmetic).  Replaces the matrix build of rplu.rational._loewner_weights
 * (rational.py:124-127); the weights are its smallest right singular vector. */
int rplu_loewner_fill(rplu_ctx* ctx, const void* zo, const void* fo, int64_t no, const void* zs,
                      const void* fs, int64_t k, void* out, void* stream);

/* Barycentric evaluation r(z) = sum_j w_j f_j/(z - t_j) / sum_j w_j/(z - t_j)
 * with the Cauchy entries generated on the fly (no nz x k matrix in HBM).
 * mode 0 = BarycentricRational.__call__ / eval_flagged (rational.py:63-80):
 *   |z - t_j| <= hit_tol returns f_j (last such j); near_pole[i] = 1 when
 *   |den| < 1e3 * DBL_MIN or the quotient is not finite (and no hit).
 * mode 1 = the AAA refit (rational.py:165-169): non-finite quotients -> 0,
 *   near_pole unused (may be NULL). */
int rplu_bary_eval(rplu_ctx* ctx, const void* z, int64_t nz, const void* t, const void* f,
                   const void* w, int64_t k, double hit_tol, int32_t mode, void* out,
                   int32_t* near_pole, void* stream);

/* One modified Gram-Schmidt Arnoldi step of restarted GMRES
 * (rplu.precond.gmres inner loop, precond.py:160-166), one cooperative
 * launch: for t = 0..j: h[t] = <V_t, w>, w -= h[t] V_t (MGS order);
 * h[j+1] = ||w|| (imaginary part 0); if h[j+1] > 0 and vnext != NULL,
 * vnext = w / h[j+1].  V: (j+1) contiguous rows of n complex128 (row t =
 * basis vector t); w updated in place; h: device complex128[j+2]. */
int rplu_mgs_arnoldi(rplu_ctx* ctx, const void* V, int64_t n, int32_t j, void* w, void* vnext,
                     void* h, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RPLU_B200_H */
