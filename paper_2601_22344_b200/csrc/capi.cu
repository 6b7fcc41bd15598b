// C ABI entry points (include/rplu_b200.h): context, errors, argument
// validation with the reference's error classes, dispatch to the paths.
#include <cuda_runtime.h>
#include <algorithm>
#include <stdio.h>
#include <stdlib.h>

#include <string>

#include "rplu_internal.h"

#include <atomic>
namespace rplu {
static std::atomic<long long> g_launches{0};
void count_launches(long long k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
}  // namespace rplu
namespace rplu {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                 cudaGetErrorString(e) + ") at " + where;
  return RPLU_ERR_CUDA;
}

int DevBuf::ensure(size_t want) {
  if (want <= bytes && ptr) return RPLU_OK;
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
  size_t b = want < 256 ? 256 : want;
  cudaError_t e = cudaMalloc(&ptr, b);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(workspace)");
  bytes = b;
  return RPLU_OK;
}

void DevBuf::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
}

int run_maybe_graph(rplu_ctx* ctx, cudaStream_t user, bool use_graph, int slot,
                    const std::function<int(cudaStream_t)>& enqueue) {
  if (!use_graph) return enqueue(user);
  if (!ctx->priv) {
    RPLU_CUDA(cudaStreamCreateWithFlags(&ctx->priv, cudaStreamNonBlocking));
    RPLU_CUDA(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
    RPLU_CUDA(cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming));
  }
  RPLU_CUDA(cudaEventRecord(ctx->ev_in, user));
  RPLU_CUDA(cudaStreamWaitEvent(ctx->priv, ctx->ev_in, 0));
  RPLU_CUDA(cudaStreamBeginCapture(ctx->priv, cudaStreamCaptureModeThreadLocal));
  int rc = enqueue(ctx->priv);
  cudaGraph_t g = nullptr;
  cudaError_t ec = cudaStreamEndCapture(ctx->priv, &g);
  if (rc != RPLU_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (ec != cudaSuccess) return cuda_fail(ec, "cudaStreamEndCapture");
  cudaGraphExec_t& ex = ctx->graph_exec[slot];
  static const bool debug = getenv("RPLU_DEBUG_GRAPH") != nullptr;
  if (ex) {
    cudaGraphExecUpdateResultInfo info;
    cudaError_t ue = cudaGraphExecUpdate(ex, g, &info);
    if (ue != cudaSuccess) {
      if (debug)
        fprintf(stderr, "[rplu] graph slot %d: exec update failed (%s, result %d)\n", slot,
                cudaGetErrorName(ue), (int)info.result);
      cudaGetLastError();  // clear the non-sticky update error
      cudaGraphExecDestroy(ex);
      ex = nullptr;
    }
  }
  if (!ex) {
    if (debug) fprintf(stderr, "[rplu] graph slot %d: instantiate\n", slot);
    ec = cudaGraphInstantiate(&ex, g, 0);
    if (ec != cudaSuccess) {
      cudaGraphDestroy(g);
      ex = nullptr;
      return cuda_fail(ec, "cudaGraphInstantiate");
    }
  }
  cudaGraphDestroy(g);
  RPLU_CUDA(cudaGraphLaunch(ex, ctx->priv));
  RPLU_CUDA(cudaEventRecord(ctx->ev_out, ctx->priv));
  RPLU_CUDA(cudaStreamWaitEvent(user, ctx->ev_out, 0));
  return RPLU_OK;
}

int dense_run_impl(rplu_ctx* ctx, const rplu_dense_args* a, rplu_dense_out* out);
int row_masses_impl(rplu_ctx* ctx, int dtype, const void* R, long long n, long long m,
                    long long ld, double* masses, cudaStream_t s);
int sample_index_impl(rplu_ctx* ctx, const double* w, long long n, double u, int mode,
                      long long* idx, int* near, double* total, cudaStream_t s);
int cauchy_run_impl(rplu_ctx* ctx, const rplu_cauchy_args* a, rplu_cauchy_out* out);
int fp64_peak_impl(rplu_ctx* ctx, double* tflops, double* ms_out);
int tree_bounds_impl(rplu_ctx* ctx, const rplu_tree_plan* plan, const void* x, const void* y,
                     const void* G, const void* Bt, double* u, cudaStream_t s);
int gauss_gemv_impl(rplu_ctx* ctx, const GaussOp& op, const double* v, double* out, bool square,
                    cudaStream_t s, float* ms);
int gauss_line_impl(const double* pts, long long count, const double* base, double c, double* out,
                    cudaStream_t s);
int gauss_restricted_impl(rplu_ctx* ctx, const double* targets, long long count,
                          const double* selpts, const long long* sel, const double* w,
                          long long k, double c, double* out, cudaStream_t s);
int cur_downdate_impl(rplu_ctx* ctx, long long n, double* nrow, const double* g, const double* v,
                      const double* chat, double l2, double floor, long long* clamped,
                      double* total, cudaStream_t s);

int loewner_fill_impl(const void* zo, const void* fo, long long no, const void* zs,
                      const void* fs, long long k, void* out, cudaStream_t s);
int bary_eval_impl(const void* z, long long nz, const void* t, const void* f, const void* w,
                   long long k, double hit_tol, int mode, void* out, int32_t* near_pole,
                   cudaStream_t s);
int mgs_arnoldi_impl(rplu_ctx* ctx, const void* V, long long n, int j, void* w, void* vnext,
                     void* h, cudaStream_t s);

int cauchy_plan_row_impl(rplu_ctx* ctx, int p, long long n, long long m, const void* x,
                         const void* y, void* G, void* Bt, long long i, void* rbuf, double* wbuf,
                         const double* bounds, double* host3, cudaStream_t s);
int cauchy_plan_update_impl(rplu_ctx* ctx, int p, long long n, long long m, const void* x,
                            const void* y, void* G, void* Bt, long long i, long long j, void* rbuf,
                            void* Cout, void* Rout, cudaStream_t s);

static int gauss_check(const rplu_gauss_op* op) {
  if (!op || op->n < 1 || op->m < 1 || !op->P || !op->Q || !(op->h > 0.0)) {
    set_error("invalid Gaussian-kernel operator");
    return RPLU_ERR_ARG;
  }
  return RPLU_OK;
}

// coordinate scale 1/(sqrt(2) h): |sc p - sc q|^2 = |p - q|^2 / (2 h^2)
static double gauss_scale(double h) { return 1.0 / (1.4142135623730951 * h); }

static GaussOp gauss_of(const rplu_gauss_op* op, bool adjoint) {
  GaussOp g;
  g.n = adjoint ? op->m : op->n;
  g.m = adjoint ? op->n : op->m;
  g.P = adjoint ? op->Q : op->P;
  g.Q = adjoint ? op->P : op->Q;
  g.c = gauss_scale(op->h);
  return g;
}
int cauchy_norms_impl(rplu_ctx* ctx, int p, long long n, long long m, const void* x, const void* y,
                      const void* G, const void* Bt, double* out, cudaStream_t s);

// Bind the calling thread to the context's device for the duration of a call.
struct DeviceGuard {
  int prev = -1;
  int rc = RPLU_OK;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) {
      cudaError_t e = cudaSetDevice(dev);
      if (e != cudaSuccess) rc = cuda_fail(e, "cudaSetDevice");
    }
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace rplu

using namespace rplu;

extern "C" {

int rplu_abi_version(void) { return RPLU_B200_ABI_VERSION; }

int64_t rplu_kernel_launch_count(void) { return g_launches.load(); }

const char* rplu_last_error(void) { return g_last_error.c_str(); }

int rplu_ctx_create(int device, rplu_ctx** out) {
  if (!out) { set_error("rplu_ctx_create: out is NULL"); return RPLU_ERR_ARG; }
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) {
    set_error("rplu_ctx_create: device " + std::to_string(device) + " out of range [0, " +
              std::to_string(ndev) + ")");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(device);
  if (g.rc) return g.rc;
  rplu_ctx* c = new rplu_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  *out = c;
  return RPLU_OK;
}

int rplu_ctx_destroy(rplu_ctx* ctx) {
  if (!ctx) return RPLU_OK;
  {
    DeviceGuard g(ctx->device);
    ctx->state.release();
    ctx->masses.release();
    ctx->rowmax.release();
    ctx->rowarg.release();
    ctx->uniforms.release();
    ctx->pivots.release();
    ctx->resid.release();
    ctx->masses2.release();
    ctx->gbar.release();
    ctx->csync.release();
    ctx->krylov.release();
    ctx->lu_pad.release();
    ctx->lu_part.release();
    ctx->mf_buf.release();
    ctx->gram.release();
    if (ctx->ring) cudaFreeHost(ctx->ring);
    for (auto& e : ctx->ring_ev)
      if (e) cudaEventDestroy(e);
    for (auto& b : ctx->scratch) b.release();
    for (auto& e : ctx->graph_exec)
      if (e) cudaGraphExecDestroy(e);
    if (ctx->priv) cudaStreamDestroy(ctx->priv);
    if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
    if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
  }
  delete ctx;
  return RPLU_OK;
}

// Argument validation mirrors eliminate (dense_pivots.py:142-145) and
// PivotRule (:56-59); the Python wrapper raises the same exception classes.
int rplu_dense_run(rplu_ctx* ctx, const rplu_dense_args* a, rplu_dense_out* out) {
  if (!ctx || !a || !out) { set_error("rplu_dense_run: NULL argument"); return RPLU_ERR_ARG; }
  if (a->dtype != RPLU_F32 && a->dtype != RPLU_F64 && a->dtype != RPLU_C128) {
    set_error("rplu_dense_run: unknown dtype " + std::to_string(a->dtype));
    return RPLU_ERR_ARG;
  }
  if (a->rule != RPLU_RULE_RPLU && a->rule != RPLU_RULE_C2PLU && a->rule != RPLU_RULE_CPLU) {
    set_error("unknown pivot rule id " + std::to_string(a->rule));
    return RPLU_ERR_ARG;
  }
  if (a->n < 1 || a->m < 1 || a->ld < a->m || a->ldu < a->m) {
    set_error("rplu_dense_run: bad shape n=" + std::to_string(a->n) + " m=" +
              std::to_string(a->m) + " ld=" + std::to_string(a->ld));
    return RPLU_ERR_ARG;
  }
  const int64_t kmax = a->n < a->m ? a->n : a->m;
  if (a->steps < 0 || a->steps > kmax) {
    set_error("steps " + std::to_string(a->steps) + " out of range [0, " + std::to_string(kmax) +
              "]");
    return RPLU_ERR_ARG;
  }
  if (!(a->stop_tol >= 0.0)) { set_error("stop_tol must be nonnegative"); return RPLU_ERR_ARG; }
  if (!a->R || (a->steps > 0 && (!a->Lt || !a->U))) {
    set_error("rplu_dense_run: NULL device buffer");
    return RPLU_ERR_ARG;
  }
  if (a->rule == RPLU_RULE_RPLU && a->steps > 0 && (!a->uniforms || a->n_uniforms < 2)) {
    set_error("rule 'rplu' needs an RngState (uniform stream)");
    return RPLU_ERR_ARG;
  }
  if (!out->pivots && a->steps > 0) { set_error("rplu_dense_run: out->pivots is NULL"); return RPLU_ERR_ARG; }
  if (!out->resid_fro) { set_error("rplu_dense_run: out->resid_fro is NULL"); return RPLU_ERR_ARG; }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  int st = dense_run_impl(ctx, a, out);
  if (st == RPLU_ERR_CUDA || st == RPLU_ERR_ARG) return st;
  if (st == kZeroPivot) {
    set_error("pivot (" + std::to_string(out->zero_pivot_i) + ", " +
              std::to_string(out->zero_pivot_j) + ") has exactly zero value after resampling");
    return RPLU_ERR_ZERO_PIVOT;
  }
  if (st == kUniformsExhausted) {
    set_error("uniform stream exhausted (pass at least 4*steps uniforms)");
    return RPLU_ERR_ARG;
  }
  return RPLU_OK;
}

int rplu_row_masses(rplu_ctx* ctx, int32_t dtype, const void* R, int64_t n, int64_t m, int64_t ld,
                    double* masses, void* stream) {
  if (!ctx || !R || !masses || n < 0 || m < 0 || ld < m) {
    set_error("rplu_row_masses: bad argument");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return row_masses_impl(ctx, dtype, R, n, m, ld, masses, reinterpret_cast<cudaStream_t>(stream));
}

// Validation mirrors structured_eliminate (cauchy.py:193-199) and
// CauchyLikeMatrix (:59-66).
int rplu_cauchy_run(rplu_ctx* ctx, const rplu_cauchy_args* a, rplu_cauchy_out* out) {
  if (!ctx || !a || !out) { set_error("rplu_cauchy_run: NULL argument"); return RPLU_ERR_ARG; }
  if (a->rule != RPLU_RULE_RPLU && a->rule != RPLU_RULE_C2PLU) {
    set_error("unknown structured rule id " + std::to_string(a->rule));
    return RPLU_ERR_ARG;
  }
  if (a->p < 1 || a->p > 8) {
    set_error("displacement rank " + std::to_string(a->p) + " exceeds 8");
    return RPLU_ERR_ARG;
  }
  if (a->n < 1 || a->m < 1) { set_error("rplu_cauchy_run: empty shape"); return RPLU_ERR_ARG; }
  const int64_t kmax = a->n < a->m ? a->n : a->m;
  if (a->rank < 0 || a->rank > kmax) {
    set_error("rank " + std::to_string(a->rank) + " out of range [0, " + std::to_string(kmax) +
              "]");
    return RPLU_ERR_ARG;
  }
  if (!a->x || !a->y || !a->G || !a->Bt) {
    set_error("rplu_cauchy_run: NULL generator buffer");
    return RPLU_ERR_ARG;
  }
  if (a->rule == RPLU_RULE_RPLU && a->rank > 0 && (!a->uniforms || a->n_uniforms < 2)) {
    set_error("structured rplu needs an RngState");
    return RPLU_ERR_ARG;
  }
  if (a->rank > 0 && (!out->rows || !out->cols || !out->bound_maxes || !out->bound_sums)) {
    set_error("rplu_cauchy_run: NULL output array");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  if (a->rank == 0) {
    out->steps_done = out->bounds_recorded = 0;
    out->uniforms_consumed = out->near_boundary_draws = 0;
    out->tol_stop = out->degenerate_stop = 0;
    out->kernel_launches = 0;
    return RPLU_OK;
  }
  int st = cauchy_run_impl(ctx, a, out);
  if (st == RPLU_ERR_CUDA || st == RPLU_ERR_ARG) return st;
  if (st == kZeroPivot) {
    set_error("pivot (" + std::to_string(out->zero_pivot_i) + ", " +
              std::to_string(out->zero_pivot_j) + ") is numerically zero" +
              (a->rule == RPLU_RULE_RPLU ? " after resampling" : ""));
    return RPLU_ERR_ZERO_PIVOT;
  }
  if (st == kUniformsExhausted) {
    set_error("uniform stream exhausted (pass at least 3*rank uniforms)");
    return RPLU_ERR_ARG;
  }
  return RPLU_OK;
}

int rplu_cauchy_row_norms(rplu_ctx* ctx, int32_t p, int64_t n, int64_t m, const void* x,
                          const void* y, const void* G, const void* Bt, double* out,
                          void* stream) {
  if (!ctx || !x || !y || !G || !Bt || !out || n < 1 || m < 1 || p < 1 || p > 8) {
    set_error("rplu_cauchy_row_norms: bad argument");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return cauchy_norms_impl(ctx, p, n, m, x, y, G, Bt, out, reinterpret_cast<cudaStream_t>(stream));
}

static int shard_check(rplu_ctx* ctx, const rplu_shard_args* a) {
  if (!ctx || !a || a->world < 1 || a->rank < 0 || a->rank >= a->world || a->n_local < 0 ||
      a->m < 1 || a->ld < a->m || a->ldu < a->m || a->steps < 0 || !a->U ||
      (a->n_local > 0 && !a->R)) {
    set_error("rplu_shard: bad arguments");
    return RPLU_ERR_ARG;
  }
  if (a->dtype != RPLU_F32 && a->dtype != RPLU_F64 && a->dtype != RPLU_C128) {
    set_error("rplu_shard: unknown dtype");
    return RPLU_ERR_ARG;
  }
  if (a->lazy_block != 0) {
    const long long vec = 16 / (a->dtype == RPLU_F32 ? 4 : (a->dtype == RPLU_F64 ? 8 : 16));
    if (a->lazy_block > kLazyMaxBlock || a->ld % vec || a->ldu % vec ||
        (uintptr_t)a->R % 16 || (uintptr_t)a->U % 16 || !a->Lt) {
      set_error("rplu_shard: lazy_block needs <= 16, 16-byte aligned rows of R and U, and Lt");
      return RPLU_ERR_ARG;
    }
  }
  return RPLU_OK;
}

// fp64 delayed-update shards use the Gram-form masses (RPLU_GRAM=0 disables)
static bool shard_gram(const rplu_shard_args* a) {
  static const bool env = [] {
    const char* e = getenv("RPLU_GRAM");
    return !(e && e[0] == '0');
  }();
  return env && a->dtype == RPLU_F64 && a->lazy_block != 0;
}

static int shard_block(const rplu_shard_args* a) {
  if (a->lazy_block >= 0) return a->lazy_block;
  return shard_gram(a) ? dense_gram_block() : dense_lazy_block_default(a->dtype);
}

static double* shard_gram_buf(rplu_ctx* ctx, const rplu_shard_args* a, int* rc) {
  *rc = RPLU_OK;
  if (!shard_gram(a)) return nullptr;
  if ((*rc = ctx->gram.ensure(sizeof(double) * (3 * (size_t)std::max<long long>(a->n_local, 1) +
                                                256))))
    return nullptr;
  return reinterpret_cast<double*>(ctx->gram.ptr);
}

static ShardParams shard_params(rplu_ctx* ctx, const rplu_shard_args* a) {
  ShardParams p{};
  p.dtype = a->dtype;
  p.R = a->R;
  p.ld = a->ld;
  p.n_local = a->n_local;
  p.m = a->m;
  p.row_offset = a->row_offset;
  p.steps = a->steps;
  p.U = a->U;
  p.ldu = a->ldu;
  p.masses = reinterpret_cast<double*>(ctx->masses.ptr);
  p.st = reinterpret_cast<DevState*>(ctx->state.ptr);
  p.world = a->world;
  p.rank = a->rank;
  p.uniforms = reinterpret_cast<const double*>(ctx->uniforms.ptr);
  p.n_uniforms = a->n_uniforms;
  p.resid = reinterpret_cast<double*>(ctx->resid.ptr);
  p.pivots = reinterpret_cast<long long*>(ctx->pivots.ptr);
  p.stop_tol = a->stop_tol;
  p.Lt = a->Lt;
  p.lazy_block = shard_block(a);
  return p;
}

__global__ void shard_init_state(DevState* st) {
  st->ucount = 0;
  st->near_boundary = 0;
  st->pi = st->pj = -1;
  st->err_i = st->err_j = -1;
  st->active = 1;
  st->status = 0;
  st->fro0 = 0.0;
  st->done = 0;
  st->step = 0;
}

int rplu_shard_begin(rplu_ctx* ctx, const rplu_shard_args* a, double* local_total) {
  int rc;
  if ((rc = shard_check(ctx, a))) return rc;
  if (!local_total || !a->uniforms || a->n_uniforms < 2) {
    set_error("rplu_shard_begin: needs local_total and a uniform stream");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(a->stream);
  if ((rc = ctx->state.ensure(sizeof(DevState)))) return rc;
  if ((rc = ctx->masses.ensure(sizeof(double) * (size_t)(a->n_local > 0 ? a->n_local : 1)))) return rc;
  if ((rc = ctx->pivots.ensure(sizeof(long long) * (size_t)(2 * a->steps + 2)))) return rc;
  if ((rc = ctx->resid.ensure(sizeof(double) * (size_t)(a->steps + 1)))) return rc;
  if ((rc = ctx->uniforms.ensure(sizeof(double) * (size_t)a->n_uniforms))) return rc;
  RPLU_CUDA(cudaMemcpyAsync(ctx->uniforms.ptr, a->uniforms, sizeof(double) * a->n_uniforms,
                            cudaMemcpyHostToDevice, s));
  shard_init_state<<<1, 1, 0, s>>>(reinterpret_cast<DevState*>(ctx->state.ptr));
  double* masses = reinterpret_cast<double*>(ctx->masses.ptr);
  if (a->n_local > 0) {
    if ((rc = dense_sweep_launch(a->dtype, a->R, a->ld, a->n_local, a->m, a->Lt, a->U, a->ldu,
                                 masses, nullptr, 0, false, s)))
      return rc;
    double* gram = shard_gram_buf(ctx, a, &rc);
    if (rc) return rc;
    if (gram && (rc = dense_gram_reset_launch(a->n_local, masses, gram, s))) return rc;
  }
  return shard_total_impl(masses, a->n_local, local_total, nullptr, s);
}

int rplu_shard_select(rplu_ctx* ctx, const rplu_shard_args* a, int64_t t, const double* totals,
                      void* msg) {
  int rc;
  if ((rc = shard_check(ctx, a))) return rc;
  if (!totals || !msg || t > a->steps) {
    set_error("rplu_shard_select: bad arguments");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  ShardParams p = shard_params(ctx, a);
  p.t = t < 0 ? -1 : t;
  p.totals = totals;
  p.msg = msg;
  if (p.lazy_block > 0)   // t < 0: the step comes from the device counter (captured blocks)
    return shard_lazy_select_impl(p, reinterpret_cast<cudaStream_t>(a->stream));
  return shard_select_impl(p, reinterpret_cast<cudaStream_t>(a->stream));
}

int rplu_shard_update(rplu_ctx* ctx, const rplu_shard_args* a, int64_t t, const void* msg,
                      double* local_total) {
  int rc;
  if ((rc = shard_check(ctx, a))) return rc;
  if (!msg || !local_total || t >= a->steps) {
    set_error("rplu_shard_update: bad arguments");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(a->stream);
  ShardParams p = shard_params(ctx, a);
  p.t = t < 0 ? -1 : t;
  p.msg = const_cast<void*>(msg);
  // Delayed-update shards with t < 0 (captured blocks): -1 - t is the step's
  // position inside its block; the absolute step comes from the device
  // counter, so one captured block of lazy_block steps can be replayed.  Only
  // whole blocks run this way (the flush sits at the block's last position).
  const long long b = p.lazy_block;
  const long long pos = t < 0 ? -1 - t : t % (b > 0 ? b : 1);
  if (b > 0 && pos >= b) {
    set_error("rplu_shard_update: block position out of range");
    return RPLU_ERR_ARG;
  }
  if ((rc = shard_post_impl(p, s))) return rc;
  if (b > 0) {
    const bool rel = t < 0;
    const bool flush = (pos + 1 == b) || (!rel && t == a->steps - 1);
    double* gram = shard_gram_buf(ctx, a, &rc);
    if (rc) return rc;
    if ((rc = dense_lazy_step_launch(a->dtype, a->R, a->ld, a->n_local, a->m, a->Lt, a->U,
                                     a->ldu, p.masses, p.st, rel ? pos : t, rel ? 0 : t - pos,
                                     true, flush, false, s, gram, rel, a->steps)))
      return rc;
  } else if (a->n_local > 0) {
    if ((rc = dense_sweep_launch(a->dtype, a->R, a->ld, a->n_local, a->m, a->Lt, a->U, a->ldu,
                                 p.masses, p.st, p.t, true, s)))
      return rc;
  }
  return shard_total_impl(p.masses, a->n_local, local_total, p.st, s);
}

int rplu_shard_lazy_block(const rplu_shard_args* a) { return a ? shard_block(a) : 0; }

int rplu_shard_active(rplu_ctx* ctx, const rplu_shard_args* a, int32_t* active) {
  int rc;
  if ((rc = shard_check(ctx, a))) return rc;
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(a->stream);
  DevState hs;
  RPLU_CUDA(cudaMemcpyAsync(&hs, ctx->state.ptr, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaStreamSynchronize(s));
  *active = hs.active;
  return RPLU_OK;
}

int rplu_shard_finish(rplu_ctx* ctx, const rplu_shard_args* a, rplu_dense_out* out) {
  int rc;
  if ((rc = shard_check(ctx, a))) return rc;
  if (!out || !out->resid_fro || (a->steps > 0 && !out->pivots)) {
    set_error("rplu_shard_finish: bad output");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(a->stream);
  DevState hs;
  RPLU_CUDA(cudaMemcpyAsync(&hs, ctx->state.ptr, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaStreamSynchronize(s));
  const long long done = hs.done;
  const int block = shard_block(a);
  out->lazy_block = block;
  if (block > 0 && done < a->steps) {
    // early stop: the local rows hold R^(t0) of the last flush
    const long long t0 = (done / block) * block;
    if (done > t0) {
      if ((rc = dense_lazy_step_launch(a->dtype, a->R, a->ld, a->n_local, a->m, a->Lt, a->U,
                                       a->ldu, reinterpret_cast<double*>(ctx->masses.ptr),
                                       reinterpret_cast<DevState*>(ctx->state.ptr), done - 1, t0,
                                       false, true, true, s)))
        return rc;
      RPLU_CUDA(cudaStreamSynchronize(s));
    }
  }
  if (done > 0)
    RPLU_CUDA(cudaMemcpy(out->pivots, ctx->pivots.ptr, sizeof(long long) * 2 * done,
                         cudaMemcpyDeviceToHost));
  RPLU_CUDA(cudaMemcpy(out->resid_fro, ctx->resid.ptr, sizeof(double) * (done + 1),
                       cudaMemcpyDeviceToHost));
  out->steps_done = done;
  out->uniforms_consumed = hs.ucount;
  out->near_boundary_draws = hs.near_boundary;
  out->clean_early_stop = hs.status == kCleanStop;
  out->tol_stop = hs.status == kTolStop;
  out->zero_pivot_i = hs.err_i;
  out->zero_pivot_j = hs.err_j;
  if (hs.status == kZeroPivot) {
    set_error("pivot (" + std::to_string(hs.err_i) + ", " + std::to_string(hs.err_j) +
              ") has exactly zero value (no resample on the sharded path)");
    return RPLU_ERR_ZERO_PIVOT;
  }
  if (hs.status == kUniformsExhausted) {
    set_error("uniform stream exhausted");
    return RPLU_ERR_ARG;
  }
  return RPLU_OK;
}

static int cauchy_shard_check(rplu_ctx* ctx, const rplu_cauchy_shard_args* a) {
  if (!ctx || !a || a->world < 1 || a->rank < 0 || a->rank >= a->world || a->n_local < 0 ||
      a->m < 1 || a->p < 1 || a->p > 8 || a->steps < 0 || !a->y || !a->Bt ||
      (a->n_local > 0 && (!a->x || !a->G)) || a->row_offset < 0) {
    set_error("rplu_cauchy_shard: bad arguments");
    return RPLU_ERR_ARG;
  }
  if (a->rule != RPLU_RULE_RPLU && a->rule != RPLU_RULE_C2PLU) {
    set_error("rplu_cauchy_shard: rule must be rplu or c2plu");
    return RPLU_ERR_ARG;
  }
  return RPLU_OK;
}

int rplu_cauchy_shard_begin(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, double* local_stats) {
  int rc;
  if ((rc = cauchy_shard_check(ctx, a))) return rc;
  if (!local_stats || (a->rule == RPLU_RULE_RPLU && (!a->uniforms || a->n_uniforms < 2))) {
    set_error("rplu_cauchy_shard_begin: needs local_stats and (rplu) a uniform stream");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return cauchy_shard_begin_impl(ctx, a, local_stats);
}

int rplu_cauchy_shard_select(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, int64_t t,
                             const double* totals, void* msg) {
  int rc;
  if ((rc = cauchy_shard_check(ctx, a))) return rc;
  if (!totals || !msg || t < 0 || t >= a->steps) {
    set_error("rplu_cauchy_shard_select: bad arguments (0 <= t < steps)");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return cauchy_shard_select_impl(ctx, a, t, totals, msg);
}

int rplu_cauchy_shard_update(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, int64_t t,
                             const void* msg, double* local_stats) {
  int rc;
  if ((rc = cauchy_shard_check(ctx, a))) return rc;
  if (!msg || !local_stats || t < 0 || t >= a->steps) {
    set_error("rplu_cauchy_shard_update: bad arguments (0 <= t < steps)");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return cauchy_shard_update_impl(ctx, a, t, msg, local_stats);
}

int rplu_cauchy_shard_active(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, int32_t* active) {
  int rc;
  if ((rc = cauchy_shard_check(ctx, a))) return rc;
  if (!active) { set_error("rplu_cauchy_shard_active: NULL active"); return RPLU_ERR_ARG; }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  int v = 0;
  if ((rc = cauchy_shard_active_impl(ctx, a, &v))) return rc;
  *active = v;
  return RPLU_OK;
}

int rplu_cauchy_shard_finish(rplu_ctx* ctx, const rplu_cauchy_shard_args* a,
                             rplu_cauchy_out* out) {
  int rc;
  if ((rc = cauchy_shard_check(ctx, a))) return rc;
  if (!out || (a->steps > 0 && (!out->rows || !out->cols || !out->bound_maxes ||
                                !out->bound_sums))) {
    set_error("rplu_cauchy_shard_finish: bad output");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  rc = cauchy_shard_finish_impl(ctx, a, out);
  if (rc == kZeroPivot) {
    set_error("pivot (" + std::to_string(out->zero_pivot_i) + ", " +
              std::to_string(out->zero_pivot_j) + ") is numerically zero after one resample");
    return RPLU_ERR_ZERO_PIVOT;
  }
  if (rc == kUniformsExhausted) {
    set_error("uniform stream exhausted");
    return RPLU_ERR_ARG;
  }
  return rc < 0 ? rc : RPLU_OK;
}

int rplu_gauss_apply(rplu_ctx* ctx, const rplu_gauss_op* op, int32_t adjoint, const double* v,
                     double* out, double* kernel_ms, void* stream) {
  int rc;
  if (!ctx || !v || !out) { set_error("rplu_gauss_apply: NULL argument"); return RPLU_ERR_ARG; }
  if ((rc = gauss_check(op))) return rc;
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  float ms = 0.f;
  rc = gauss_gemv_impl(ctx, gauss_of(op, adjoint != 0), v, out, false,
                       reinterpret_cast<cudaStream_t>(stream), kernel_ms ? &ms : nullptr);
  if (kernel_ms) *kernel_ms = ms;
  return rc;
}

int rplu_gauss_row_norms(rplu_ctx* ctx, const rplu_gauss_op* op, double* out, void* stream) {
  int rc;
  if (!ctx || !out) { set_error("rplu_gauss_row_norms: NULL argument"); return RPLU_ERR_ARG; }
  if ((rc = gauss_check(op))) return rc;
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return gauss_gemv_impl(ctx, gauss_of(op, false), nullptr, out, true,
                         reinterpret_cast<cudaStream_t>(stream), nullptr);
}

int rplu_gauss_line(rplu_ctx* ctx, const rplu_gauss_op* op, int32_t axis, int64_t index,
                    double* out, void* stream) {
  int rc;
  if (!ctx || !out) { set_error("rplu_gauss_line: NULL argument"); return RPLU_ERR_ARG; }
  if ((rc = gauss_check(op))) return rc;
  const int64_t lim = axis == 0 ? op->n : op->m;
  if (index < 0 || index >= lim) { set_error("index out of range"); return RPLU_ERR_ARG; }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  const double c = gauss_scale(op->h);
  if (axis == 0) return gauss_line_impl(op->Q, op->m, op->P + 3 * index, c, out,
                                        reinterpret_cast<cudaStream_t>(stream));
  return gauss_line_impl(op->P, op->n, op->Q + 3 * index, c, out,
                         reinterpret_cast<cudaStream_t>(stream));
}

int rplu_gauss_restricted(rplu_ctx* ctx, const rplu_gauss_op* op, int32_t axis,
                          const int64_t* sel, const double* w, int64_t k, double* out,
                          void* stream) {
  int rc;
  if (!ctx || !out || (k > 0 && (!sel || !w)) || k < 0) {
    set_error("rplu_gauss_restricted: bad argument");
    return RPLU_ERR_ARG;
  }
  if ((rc = gauss_check(op))) return rc;
  if (k > 12000) { set_error("restricted product supports k <= 12000"); return RPLU_ERR_ARG; }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  const double c = gauss_scale(op->h);
  const long long* s = reinterpret_cast<const long long*>(sel);
  if (axis == 0)  // out[m] = A[sel,:]^T w : targets Q, selected P[sel]
    return gauss_restricted_impl(ctx, op->Q, op->m, op->P, s, w, k, c, out,
                                 reinterpret_cast<cudaStream_t>(stream));
  return gauss_restricted_impl(ctx, op->P, op->n, op->Q, s, w, k, c, out,
                               reinterpret_cast<cudaStream_t>(stream));
}

int rplu_loewner_fill(rplu_ctx* ctx, const void* zo, const void* fo, int64_t no, const void* zs,
                      const void* fs, int64_t k, void* out, void* stream) {
  if (!ctx || no < 0 || k < 0 || (no * k > 0 && (!zo || !fo || !zs || !fs || !out))) {
    set_error("rplu_loewner_fill: bad argument");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return loewner_fill_impl(zo, fo, no, zs, fs, k, out, reinterpret_cast<cudaStream_t>(stream));
}

int rplu_bary_eval(rplu_ctx* ctx, const void* z, int64_t nz, const void* t, const void* f,
                   const void* w, int64_t k, double hit_tol, int32_t mode, void* out,
                   int32_t* near_pole, void* stream) {
  if (!ctx || nz < 0 || k < 1 || k > (1 << 30) || (mode != 0 && mode != 1) ||
      (nz > 0 && (!z || !t || !f || !w || !out || (mode == 0 && !near_pole)))) {
    set_error("rplu_bary_eval: bad argument");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return bary_eval_impl(z, nz, t, f, w, k, hit_tol, mode, out, near_pole,
                        reinterpret_cast<cudaStream_t>(stream));
}

int rplu_mgs_arnoldi(rplu_ctx* ctx, const void* V, int64_t n, int32_t j, void* w, void* vnext,
                     void* h, void* stream) {
  if (!ctx || n < 1 || j < 0 || !V || !w || !h) {
    set_error("rplu_mgs_arnoldi: bad argument");
    return RPLU_ERR_ARG;
  }
  if (((uintptr_t)V | (uintptr_t)w | (uintptr_t)vnext) % 16) {
    set_error("rplu_mgs_arnoldi: vectors must be 16-byte aligned");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return mgs_arnoldi_impl(ctx, V, n, j, w, vnext, h, reinterpret_cast<cudaStream_t>(stream));
}

int rplu_cur_downdate(rplu_ctx* ctx, int64_t n, double* nrow, const double* g, const double* v,
                      const double* chat, double l2, double floor, int64_t* clamped,
                      double* total, void* stream) {
  if (!ctx || !nrow || !g || !v || !chat || !clamped || !total || n < 1) {
    set_error("rplu_cur_downdate: bad argument");
    return RPLU_ERR_ARG;
  }
  DeviceGuard gd(ctx->device);
  if (gd.rc) return gd.rc;
  long long c = 0;
  int rc = cur_downdate_impl(ctx, n, nrow, g, v, chat, l2, floor, &c, total,
                             reinterpret_cast<cudaStream_t>(stream));
  *clamped = c;
  return rc;
}

int rplu_tree_bounds(rplu_ctx* ctx, const rplu_tree_plan* plan, const void* x, const void* y,
                     const void* G, const void* Bt, double* u, void* stream) {
  if (!ctx || !plan || !x || !y || !G || !Bt || !u || plan->n < 1 || plan->m < 1 ||
      plan->p < 1 || plan->p > 8 || plan->n_tleaves < 1 || plan->n_snodes < 1 ||
      plan->n_sleaves < 1 || !plan->cstart || !plan->leaf_node || plan->n_levels < 0 ||
      (plan->n_levels > 0 && (!plan->lvl_nodes || !plan->lvl_start))) {
    set_error("rplu_tree_bounds: bad argument");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return tree_bounds_impl(ctx, plan, x, y, G, Bt, u, reinterpret_cast<cudaStream_t>(stream));
}

int rplu_cauchy_plan_row(rplu_ctx* ctx, int32_t p, int64_t n, int64_t m, const void* x,
                         const void* y, void* G, void* Bt, int64_t i, void* rbuf, double* wbuf,
                         const double* bounds, double* out3, void* stream) {
  if (!ctx || p < 1 || p > 8 || n < 1 || m < 1 || !x || !y || !G || !Bt || !rbuf || !wbuf ||
      !out3 || i < 0 || i >= n) {
    set_error("rplu_cauchy_plan_row: bad argument");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return cauchy_plan_row_impl(ctx, p, n, m, x, y, G, Bt, i, rbuf, wbuf, bounds, out3,
                              reinterpret_cast<cudaStream_t>(stream));
}

int rplu_cauchy_plan_update(rplu_ctx* ctx, int32_t p, int64_t n, int64_t m, const void* x,
                            const void* y, void* G, void* Bt, int64_t i, int64_t j,
                            const void* rbuf, void* Cout, void* Rout, void* stream) {
  if (!ctx || p < 1 || p > 8 || n < 1 || m < 1 || !x || !y || !G || !Bt || !rbuf || i < 0 ||
      i >= n || j < 0 || j >= m) {
    set_error("rplu_cauchy_plan_update: bad argument");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return cauchy_plan_update_impl(ctx, p, n, m, x, y, G, Bt, i, j, const_cast<void*>(rbuf), Cout,
                                 Rout, reinterpret_cast<cudaStream_t>(stream));
}

int rplu_upload(rplu_ctx* ctx, void* dst, const void* src, int64_t bytes, int32_t threads,
                void* stream) {
  if (!ctx) { set_error("rplu_upload: NULL context"); return RPLU_ERR_ARG; }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return upload_impl(ctx, dst, src, bytes, threads, static_cast<cudaStream_t>(stream));
}

int rplu_mf_run(rplu_ctx* ctx, const rplu_mf_args* args, rplu_mf_out* out) {
  if (!ctx || !args || !out) { set_error("rplu_mf_run: NULL argument"); return RPLU_ERR_ARG; }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return mf_run_impl(ctx, args, out);
}

int rplu_lu_error(rplu_ctx* ctx, int32_t dtype, const void* A, int64_t lda, int64_t n, int64_t m,
                  const void* Lt, int64_t ldl, const void* U, int64_t ldu, int64_t k,
                  double* out_sq, double* kernel_ms, void* stream) {
  if (!ctx || !A || !out_sq || (k > 0 && (!Lt || !U))) {
    set_error("rplu_lu_error: NULL argument");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return lu_error_impl(ctx, dtype, A, lda, n, m, Lt, ldl, U, ldu, k, out_sq, kernel_ms,
                       static_cast<cudaStream_t>(stream));
}

int rplu_diag_dmma_peak(rplu_ctx* ctx, double* tflops, double* best_ms) {
  if (!ctx || !tflops) { set_error("rplu_diag_dmma_peak: NULL argument"); return RPLU_ERR_ARG; }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return dmma_peak_impl(ctx, tflops, best_ms);
}

int rplu_diag_fp64_peak(rplu_ctx* ctx, double* tflops, double* best_ms) {
  if (!ctx || !tflops) { set_error("rplu_diag_fp64_peak: NULL argument"); return RPLU_ERR_ARG; }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return fp64_peak_impl(ctx, tflops, best_ms);
}

int rplu_sample_index(rplu_ctx* ctx, const double* weights, int64_t n, double u,
                      int64_t* out_index, int32_t* near_boundary, void* stream) {
  if (!ctx || !out_index) { set_error("rplu_sample_index: NULL argument"); return RPLU_ERR_ARG; }
  if (n <= 0 || !weights) { set_error("weights must be a nonempty 1-D array"); return RPLU_ERR_ARG; }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  long long idx = -1;
  int near = 0;
  int rc = sample_index_impl(ctx, weights, n, u, 0, &idx, &near, nullptr,
                             reinterpret_cast<cudaStream_t>(stream));
  if (rc) return rc;
  *out_index = idx;
  if (near_boundary) *near_boundary = near;
  return RPLU_OK;
}

int rplu_sample_index_gather(rplu_ctx* ctx, const double* weights, int64_t n, double u,
                             const void* gather, int64_t* out_index, int32_t* near_boundary,
                             double* value, void* stream) {
  if (!ctx || !out_index || !gather || !value) {
    set_error("rplu_sample_index_gather: NULL argument");
    return RPLU_ERR_ARG;
  }
  if (n <= 0 || !weights) { set_error("weights must be a nonempty 1-D array"); return RPLU_ERR_ARG; }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  long long idx = -1;
  int near = 0;
  int rc = sample_index_gather_impl(ctx, weights, n, u, gather, &idx, &near, value,
                                    reinterpret_cast<cudaStream_t>(stream));
  if (rc) return rc;
  *out_index = idx;
  if (near_boundary) *near_boundary = near;
  return RPLU_OK;
}

int rplu_cauchy_plan_propose(rplu_ctx* ctx, int32_t p, int64_t n, int64_t m, const void* x,
                             const void* y, void* G, void* Bt, const double* bounds, double u,
                             void* rbuf, double* wbuf, double* out5, void* stream) {
  if (!ctx || p < 1 || p > 8 || n < 1 || m < 1 || !x || !y || !G || !Bt || !rbuf || !wbuf ||
      !out5 || !bounds) {
    set_error("rplu_cauchy_plan_propose: bad argument");
    return RPLU_ERR_ARG;
  }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return cauchy_plan_propose_impl(ctx, p, n, m, x, y, G, Bt, bounds, u, rbuf, wbuf, out5,
                                  reinterpret_cast<cudaStream_t>(stream));
}

int rplu_sample_target(rplu_ctx* ctx, const double* weights, int64_t n, double target,
                       int64_t* out_index, int32_t* near_boundary, void* stream) {
  if (!ctx || !out_index) { set_error("rplu_sample_target: NULL argument"); return RPLU_ERR_ARG; }
  if (n <= 0 || !weights) { set_error("weights must be a nonempty 1-D array"); return RPLU_ERR_ARG; }
  if (!(target >= 0.0)) { set_error("rplu_sample_target: target must be >= 0"); return RPLU_ERR_ARG; }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  long long idx = -1;
  int near = 0;
  int rc = sample_index_impl(ctx, weights, n, target, 1, &idx, &near, nullptr,
                             reinterpret_cast<cudaStream_t>(stream));
  if (rc) return rc;
  *out_index = idx;
  if (near_boundary) *near_boundary = near;
  return RPLU_OK;
}

int rplu_cdf_total(rplu_ctx* ctx, const double* weights, int64_t n, double* total, void* stream) {
  if (!ctx || !total) { set_error("rplu_cdf_total: NULL argument"); return RPLU_ERR_ARG; }
  if (n < 0 || (n > 0 && !weights)) { set_error("rplu_cdf_total: bad weights"); return RPLU_ERR_ARG; }
  if (n == 0) { *total = 0.0; return RPLU_OK; }
  DeviceGuard g(ctx->device);
  if (g.rc) return g.rc;
  return sample_index_impl(ctx, weights, n, 0.0, 2, nullptr, nullptr, total,
                           reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
