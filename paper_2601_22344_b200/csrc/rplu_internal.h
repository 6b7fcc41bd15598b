// Internal (non-exported) declarations shared by the CUDA translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <functional>
#include <string>

#include "../../include/rplu_b200.h"

namespace rplu {

// Per-run device-resident control block.  One instance lives in device memory
// for the whole pivot loop so no step needs a host round trip.
struct DevState {
  long long ucount;         // uniforms consumed so far
  long long near_boundary;  // draws within 1e-12*total of a CDF boundary
  long long pi, pj;         // pivot of the current step
  long long err_i, err_j;   // zero pivot location
  long long done;           // pivots committed
  long long step;           // device step counter (sharded graph replay)
  int active;               // 1 while the loop runs
  int status;               // 0 running/ok, 1 clean stop, 2 tol stop, 3 degenerate,
                            // -2 zero pivot, -1 uniform stream exhausted
  double fro0;              // residual Frobenius norm at step 0 (or u0_max / total0)
  // pivot coefficients of the current step
  double inv_d;             // 1/a (real fp64)
  float inv_f;              // 1/a (fp32)
  int branch;               // complex Smith branch
  double rat, scl;          // complex Smith coefficients
  double a_re, a_im;        // pivot value
  double aux[8];            // path-specific scratch (Cauchy / CUR)
};

enum Status {
  kRunning = 0,
  kCleanStop = 1,
  kTolStop = 2,
  kDegenerate = 3,
  kUniformsExhausted = -1,
  kZeroPivot = -2,
};

// Gaussian-kernel operator as the kernels see it (rows P, columns Q,
// c = coordinate scale 1/(sqrt(2) h) applied as points are loaded); the
// adjoint swaps P and Q.
struct GaussOp {
  long long n, m;
  const double* P;  // n x 3
  const double* Q;  // m x 3
  double c;
};

// Sharded dense step (shard.cu).
struct ShardParams {
  int dtype;
  void* R;
  long long ld, n_local, m, row_offset, steps;
  void* U;
  long long ldu;
  double* masses;
  DevState* st;
  long long t;
  const double* totals;  // [world] allgathered shard totals
  int world, rank;
  const double* uniforms;
  long long n_uniforms;
  void* msg;  // [i_global, j, a_re, a_im] (fp64) followed by the pivot row (T)
  double* resid;
  long long* pivots;
  double stop_tol;
  void* Lt;        // [steps][n_local] local L columns
  int lazy_block;  // 0: eager; > 0: delayed-update block (host step loop)
};
int shard_select_impl(const ShardParams& p, cudaStream_t s);
int shard_lazy_select_impl(const ShardParams& p, cudaStream_t s);
int shard_post_impl(const ShardParams& p, cudaStream_t s);
int shard_total_impl(const double* masses, long long n, double* out, DevState* advance,
                     cudaStream_t s);

// K1 (update=false) / K3 (update=true) on a row block, from dense.cu; the
// pivot (pj, coefficients) is read from *st and the pivot row from U[t,:].
int dense_sweep_launch(int dtype, void* R, long long ld, long long n, long long m, void* Lt,
                       void* U, long long ldu, double* masses, DevState* st, long long t,
                       bool update, cudaStream_t s);

constexpr int kLazyMaxBlock = 16;  // longest delayed-update block

// Delayed-update pieces on a row block, from dense.cu: (pivcol) the pivot
// column L[:,t] rebuilt from R^(t0) and the pending terms, then the pass
// (masses of R^(t+1); flush writes it).  force runs the pass after a stop.
// gram (fp64 only; nullptr: applied-term masses): [m0 | lin | quad](n) + 256
// doubles of U Gram -- the Gram-form masses of dense.cu (non-flush steps
// run the dot pass, flushes reset m0 / lin / quad)
int dense_lazy_step_launch(int dtype, void* R, long long ld, long long n, long long m, void* Lt,
                           void* U, long long ldu, double* masses, DevState* st, long long t,
                           long long t0, bool pivcol, bool flush, bool force, cudaStream_t s,
                           double* gram = nullptr, bool rel = false, long long u_rows = 0);
int dense_gram_reset_launch(long long n, double* masses, double* gram, cudaStream_t s);
int dense_gram_block();
int dense_lazy_block_default(int dtype, bool fused = false);

// Sharded Cauchy-like steps (cauchy.cu).
int cauchy_shard_begin_impl(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, double* stats);
int cauchy_shard_select_impl(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, long long t,
                             const double* totals, void* msg);
int cauchy_shard_update_impl(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, long long t,
                             const void* msg, double* stats);
int cauchy_shard_finish_impl(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, rplu_cauchy_out* out);
int cauchy_shard_active_impl(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, int* active);

void set_error(const std::string& msg);

// Process-wide count of kernels launched by the standalone primitives
// (Gaussian-kernel, sample-index, consumer kernels) for bench.py's
// gpu_launches claim; the pivot-loop drivers report theirs in *_out.
void count_launches(long long k);

// standalone draw (dense.cu): mode 0 u*total, 1 absolute target, 2 total only
// draws chained on the device (dense.cu): see sample_index_launch
constexpr size_t kSampleOutBytes = 24;   // sizeof(SampleOut)
int sample_index_gather_impl(rplu_ctx* ctx, const double* w, long long n, double u,
                             const void* gather, long long* idx, int* near, double* value2,
                             cudaStream_t s);
int sample_two_launch(rplu_ctx* ctx, const double* w0, long long n0, double u0,
                      const std::function<int(const void*)>& after_draw, const double* w1,
                      long long n1, cudaStream_t s, const void** d0, const void** d1);
int sample_out_unpack(const void* host_copy, long long* idx, int* near, double* total);
int cauchy_plan_propose_impl(rplu_ctx* ctx, int p, long long n, long long m, const void* x,
                             const void* y, void* G, void* Bt, const double* bounds, double u,
                             void* rbuf, double* wbuf, double* host5, cudaStream_t s);
int sample_index_impl(rplu_ctx* ctx, const double* w, long long n, double u, int mode,
                      long long* idx, int* near, double* total, cudaStream_t s);
int cuda_fail(cudaError_t e, const char* where);

int dmma_peak_impl(rplu_ctx* ctx, double* tflops, double* ms_out);
int mf_run_impl(rplu_ctx* ctx, const rplu_mf_args* a, rplu_mf_out* out);
int upload_impl(rplu_ctx* ctx, void* dst, const void* src, long long bytes, int threads,
                cudaStream_t s);

// K11 fused ||A - X Y||_F^2, ||A||_F^2 (lu_error.cu); out_sq host[2]
int lu_error_impl(rplu_ctx* ctx, int dtype, const void* A, long long lda, long long n,
                  long long m, const void* Xt, long long ldx, const void* Y, long long ldy,
                  long long k, double* out_sq, double* kernel_ms, cudaStream_t s);

#define RPLU_CUDA(call)                                        \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return ::rplu::cuda_fail(_e, #call); \
  } while (0)

// Grow-only device workspace owned by a context.
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int ensure(size_t want);
  void release();
};

}  // namespace rplu

namespace rplu {
// Enqueue work either directly on `user` or captured into a CUDA graph on the
// context's private stream (one graph launch instead of one launch per
// kernel: the latency-bound configs are otherwise host-launch bound).  The
// graph is ordered after earlier work on `user` and before later work on it;
// the instantiated graph of each slot is cached and updated in place.
int run_maybe_graph(rplu_ctx* ctx, cudaStream_t user, bool use_graph, int slot,
                    const std::function<int(cudaStream_t)>& enqueue);
}  // namespace rplu

struct rplu_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t priv = nullptr;       // capture stream
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaGraphExec_t graph_exec[4] = {nullptr, nullptr, nullptr, nullptr};
  rplu::DevBuf state;       // DevState
  rplu::DevBuf masses;      // n doubles
  rplu::DevBuf rowmax;      // n doubles (CPLU)
  rplu::DevBuf rowarg;      // n int64 (CPLU)
  rplu::DevBuf uniforms;    // device copy of the uniform stream
  rplu::DevBuf pivots;      // 2*steps int64
  rplu::DevBuf resid;       // steps+1 doubles
  rplu::DevBuf scratch[8];  // path-specific
  rplu::DevBuf masses2;     // n doubles (persistent dense loop: double-buffered masses)
  rplu::DevBuf gbar;        // grid-barrier counters (persistent dense loop)
  rplu::DevBuf csync;       // Cauchy loop: split-arrival counters + row max slot
  rplu::DevBuf krylov;      // MGS Arnoldi: per-CTA partials + grid barrier
  rplu::DevBuf lu_pad;      // K11: zero-padded fp64 factor panels
  rplu::DevBuf lu_part;     // K11: per-CTA partial sums
  rplu::DevBuf mf_buf;      // rplu_mf_run workspace (vectors, core factors, histories)
  rplu::DevBuf gram;        // dense Gram-mass delayed updates: m0, lin, quad, U Gram
  void* ring = nullptr;     // rplu_upload: page-locked staging slots
  cudaEvent_t ring_ev[4] = {nullptr, nullptr, nullptr, nullptr};
};
