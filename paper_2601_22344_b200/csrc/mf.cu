// Device-resident matrix-free CUR-form RPLU (Alg 2): rplu_mf_run.
//
// Reference: rplu.lowmem_cur.cur_build (pkg/src/rplu/lowmem_cur.py:212-300)
// with the residual row / column helpers (:161-201), the QR core
// (:43-133) and the rebuild (:204-209).  The whole step is enqueued from
// this C++ loop with every scalar decision taken on the device, so a step
// costs one host synchronisation (the control block, read back so the loop
// can stop or rebuild) and no Python at all:
//
//   1. row draw      i ~ n_row (u1) or argmax; single-CTA or two-level CDF
//   2. residual row  r = A[i,:],  rhat = r - A[I,:]^T W^{-T} r[J]     (K8)
//                    energy check, one redraw (u1'), degenerate stop
//   3. column draw   j ~ |rhat|^2 (u2) or argmax |rhat|
//   4. residual col  c = A[:,j],  chat = c - A[:,J] W^{-1} c[I]      (K8)
//   5. l = rhat / a (real: rhat * (1/a)),  g = A l                 (K7)
//   6. v = A[:,J] W^{-1} g[I]                                       (K8)
//   7. downdate      n_row -= 2 (g - v) chat; += |l|^2 chat^2; clamp (K9)
//   8. core extend   W = [[W, c[I]], [r[J], r[j]]]
//   9. rebuild       (clamps > 1% of n) n_row from m residual columns
//  10. tol stop      sum n_row <= tol^2 total0
//
// The core is kept as an unpivoted LU in selection order, W = L_W U_W, grown
// by one row / column per step in O(k^2): the new row of L_W is p = U_W^{-T}
// r[J] and the new column of U_W is q = L_W^{-1} c[I] -- exactly the
// intermediates of the two residual solves of step 2 and 4 -- and the new
// diagonal is r[j] - p.q (the pivot's Schur complement).  Its pivots are the
// elimination's own residual pivots; the reference refactors a QR of W every
// step (lowmem_cur.py:126-133, O(k^3) per step), which agrees to rounding.
// Triangular solves run in one CTA, column-oriented against row- and
// column-major copies of both factors (coalesced reads, one barrier per
// column).  Operators: the Gaussian kernel of BASELINE configs[4] (points
// P, Q; generated entries, no matrix in HBM) and a dense real matrix in HBM.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "gauss.cuh"
#include "rplu_common.cuh"
#include "rplu_internal.h"

namespace rplu {

int gauss_gemv_impl(rplu_ctx* ctx, const GaussOp& op, const double* v, double* out, bool square,
                    cudaStream_t s, float* ms);
int gauss_restricted_impl(rplu_ctx* ctx, const double* targets, long long count,
                          const double* selpts, const long long* sel, const double* w,
                          long long k, double c, double* out, cudaStream_t s);

namespace {

constexpr double kEps = 2.220446049250313e-16;  // np.finfo(float).eps
constexpr int kSolveThreads = 1024;
constexpr int kSolvePer = 8;                     // rank <= 8192
constexpr int kRedThreads = 256;

enum MfStatus { kMfRunning = 0, kMfDegenerate = 3, kMfTol = 2, kMfUniforms = -1 };

// Device control block: every per-step scalar the reference keeps in Python.
struct MfCtl {
  long long ucount, near;
  long long step;          // pivots committed (= core size k)
  long long i, j;
  long long clamped;
  int status;              // MfStatus
  int skip;                // 1 once stopped: gated kernels return at once
  int one;                 // constant 1 (the main path's gate)
  int redraw;              // 1 when the row must be redrawn (degenerate residual row)
  int fell_back;           // inverse mode would have fallen back to QR
  int pad;
  double total0, total, prev_total;
  double energy, a, inv_a, l2;
};

// Operator as the kernels see it.  kind 0: Gaussian kernel (entries from
// points scaled by c = 1/(sqrt(2) h)); kind 1: dense row-major A (lda).
struct MfOp {
  int kind;
  long long n, m;
  const double* P;
  const double* Q;
  double c;
  const double* A;
  long long lda;
};

__device__ __forceinline__ bool gated(const MfCtl* ctl, const int* gate) {
  return !ctl->skip && *gate;
}

// ---------------------------------------------------------------------------
// draws

// totals of 32768-weight chunks (two-level CDF, n >= kChunkedMinN)
__global__ void __launch_bounds__(1024) mf_chunk_totals_kernel(const MfCtl* ctl, const int* gate,
                                                               const double* w, long long n,
                                                               double* ctot, int* neg) {
  if (!gated(ctl, gate)) return;
  chunk_totals_block(w, n, ctot, neg);
}

// sample_index(w, u) (rng.py:50-74) with u = uniforms[ucount] (rplu) or the
// first argmax (greedy); the index goes to ctl->i (which == 0) or ctl->j.
__global__ void __launch_bounds__(1024) mf_draw_kernel(MfCtl* ctl, const int* gate,
                                                       const double* w, long long n,
                                                       const double* uniforms,
                                                       long long n_uniforms, int greedy,
                                                       int which, const double* ctot,
                                                       long long nch) {
  constexpr int B = 1024;
  __shared__ CdfSmem<B> sm;
  if (!gated(ctl, gate)) return;
  long long idx;
  int near = 0;
  if (greedy) {
    auto wf = [&](long long k) { return w[k]; };
    idx = block_argmax<B>(wf, n, nullptr);
  } else {
    const long long uc = ctl->ucount;
    if (uc >= n_uniforms) {
      if (threadIdx.x == 0) { ctl->status = kMfUniforms; ctl->skip = 1; }
      return;
    }
    const double u = uniforms[uc];
    if (ctot) {
      double total;
      idx = chunked_draw_block(w, n, u, 0, ctot, nch, sm, &total, &near);
    } else {
      auto wf = [&](long long k) { return w[k]; };
      Cdf<B> c = cdf_build<B>(wf, n, sm);
      const double tg = u * c.total;
      idx = cdf_find_target<B>(wf, n, c, tg, sm);
      const double tol = kNearBoundaryRel * c.total;
      near = (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) ? 1 : 0;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (which == 0) ctl->i = idx; else ctl->j = idx;
    if (!greedy) {
      ctl->ucount += 1;
      ctl->near += near;
    }
  }
}

// ---------------------------------------------------------------------------
// operator lines: axis 0 -> out[m] = A[ctl->i, :], axis 1 -> out[n] = A[:, ctl->j]
__global__ void __launch_bounds__(256) mf_line_kernel(MfOp op, const MfCtl* ctl, const int* gate,
                                                      int axis, double* out) {
  if (!gated(ctl, gate)) return;
  const long long count = axis == 0 ? op.m : op.n;
  const long long idx = axis == 0 ? ctl->i : ctl->j;
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (op.kind == 0) {
    const double* pts = axis == 0 ? op.Q : op.P;
    const double* base = (axis == 0 ? op.P : op.Q) + 3 * idx;
    const double bx = op.c * base[0], by = op.c * base[1], bz = op.c * base[2];
    const ExpTab tl = exp2tab_lane();
    for (long long k0 = (long long)blockIdx.x * blockDim.x; k0 < count; k0 += stride) {
      const long long k = k0 + threadIdx.x;
      const long long kk = k < count ? k : count - 1;
      const double e = gauss_entry(bx, by, bz, op.c * pts[kk * 3], op.c * pts[kk * 3 + 1],
                                   op.c * pts[kk * 3 + 2], tl);
      if (k < count) out[k] = e;
    }
  } else {
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride)
      out[k] = axis == 0 ? op.A[idx * op.lda + k] : op.A[k * op.lda + idx];
  }
}

// dense K8: axis 0 out[t] = sum_s A[I_s, t] y_s (t < m);
//           axis 1 out[t] = sum_s A[t, J_s] y_s (t < n)
__global__ void __launch_bounds__(256) mf_dense_restricted_kernel(MfOp op, int axis,
                                                                  const long long* sel,
                                                                  const double* y, long long k,
                                                                  double* out) {
  const long long count = axis == 0 ? op.m : op.n;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    if (axis == 0)
      for (long long s = 0; s < k; ++s) acc = fma(op.A[sel[s] * op.lda + t], y[s], acc);
    else
      for (long long s = 0; s < k; ++s) acc = fma(op.A[t * op.lda + sel[s]], y[s], acc);
    out[t] = acc;
  }
}

// dense K7: out[i] = sum_j A[i, j] v_j (one warp per row); square: A[i,j]^2
__global__ void __launch_bounds__(256) mf_dense_gemv_kernel(MfOp op, const double* v, int square,
                                                            double* out) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < op.n;
       i += warps) {
    const double* a = op.A + i * op.lda;
    double acc = 0.0;
    for (long long j = lane; j < op.m; j += 32)
      acc = square ? fma(a[j], a[j], acc) : fma(a[j], v[j], acc);
    acc = warp_sum(acc);
    if (lane == 0) out[i] = acc;
  }
}

// ---------------------------------------------------------------------------
// core solves (one CTA).  Factors of the k x k core: Lr / Lc (unit lower,
// row- / column-major), Ur / Uc (upper, row- / column-major), leading
// dimension kmax.  mode 0: W x = src[sel] -> inter = L^{-1} b (the new U
// column when src is c), x = U^{-1} inter.  mode 1: W^T y = src[sel] ->
// inter = U^{-T} z (the new L row when src is r), y = L^{-T} inter.
__global__ void __launch_bounds__(kSolveThreads) mf_solve_kernel(
    const MfCtl* ctl, const int* gate, int mode, const double* Lr, const double* Lc,
    const double* Ur, const double* Uc, long long kmax, long long k, const double* src,
    const long long* sel, double* inter, double* x) {
  if (!gated(ctl, gate)) return;
  __shared__ double sx[2];
  const int tid = threadIdx.x;
  double b[kSolvePer];
#pragma unroll
  for (int r = 0; r < kSolvePer; ++r) {
    const long long s = tid + (long long)r * kSolveThreads;
    b[r] = s < k ? src[sel[s]] : 0.0;
  }
  // forward: (mode 0) L q = b, unit diagonal, columns of L = Lc rows;
  //          (mode 1) U^T p = z, diagonal U_tt, columns of U^T = rows of U (Ur)
  const double* Fc = mode == 0 ? Lc : Ur;
  for (long long t = 0; t < k; ++t) {
    const int owner = (int)(t % kSolveThreads), slot = (int)(t / kSolveThreads);
    if (tid == owner) {
      double v = 0.0;
#pragma unroll
      for (int r = 0; r < kSolvePer; ++r)
        if (r == slot) v = b[r];
      if (mode == 1) v = v / Ur[t * kmax + t];
#pragma unroll
      for (int r = 0; r < kSolvePer; ++r)
        if (r == slot) b[r] = v;
      sx[t & 1] = v;
    }
    __syncthreads();
    const double xt = sx[t & 1];
    const double* col = Fc + t * kmax;  // entries s > t of column t
#pragma unroll
    for (int r = 0; r < kSolvePer; ++r) {
      const long long s = tid + (long long)r * kSolveThreads;
      if (s > t && s < k) b[r] = fma(-col[s], xt, b[r]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kSolvePer; ++r) {
    const long long s = tid + (long long)r * kSolveThreads;
    if (s < k && inter) inter[s] = b[r];
  }
  // backward: (mode 0) U x = q, columns of U = Uc rows;
  //           (mode 1) L^T y = p, unit diagonal, columns of L^T = rows of L (Lr)
  const double* Bc = mode == 0 ? Uc : Lr;
  for (long long t = k - 1; t >= 0; --t) {
    const int owner = (int)(t % kSolveThreads), slot = (int)(t / kSolveThreads);
    if (tid == owner) {
      double v = 0.0;
#pragma unroll
      for (int r = 0; r < kSolvePer; ++r)
        if (r == slot) v = b[r];
      if (mode == 0) v = v / Uc[t * kmax + t];
#pragma unroll
      for (int r = 0; r < kSolvePer; ++r)
        if (r == slot) b[r] = v;
      sx[t & 1] = v;
    }
    __syncthreads();
    const double xt = sx[t & 1];
    const double* col = Bc + t * kmax;  // entries s < t of column t
#pragma unroll
    for (int r = 0; r < kSolvePer; ++r) {
      const long long s = tid + (long long)r * kSolveThreads;
      if (s < t) b[r] = fma(-col[s], xt, b[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < kSolvePer; ++r) {
    const long long s = tid + (long long)r * kSolveThreads;
    if (s < k) x[s] = b[r];
  }
}

// ---------------------------------------------------------------------------
// elementwise + reductions (per-CTA partials, summed in a fixed order by a
// one-CTA finish kernel: deterministic)

__device__ __forceinline__ double block_sum256(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kRedThreads / 32; ++w) t += red[w];
  return t;
}

// rhat = r - t; w = rhat^2; partial sums of w
__global__ void __launch_bounds__(kRedThreads) mf_resid_row_kernel(const MfCtl* ctl,
                                                                   const int* gate, long long m,
                                                                   const double* r,
                                                                   const double* t, double* rhat,
                                                                   double* w, double* part) {
  __shared__ double red[kRedThreads / 32];
  if (!gated(ctl, gate)) return;
  double s = 0.0;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < m;
       q += (long long)gridDim.x * blockDim.x) {
    const double v = __dsub_rn(r[q], t[q]);
    rhat[q] = v;
    const double ww = __dmul_rn(v, v);
    w[q] = ww;
    s += ww;
  }
  const double b = block_sum256(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = b;
}

// energy = sum of the partials; first pass: energy <= eps^2 total0 asks for
// a redraw; second pass (the redraw): a degenerate row stops the build
// (lowmem_cur.py:253-259)
__global__ void mf_energy_kernel(MfCtl* ctl, const int* gate, const double* part, int parts,
                                 int second) {
  if (!gated(ctl, gate)) return;
  if (threadIdx.x != 0) return;
  double e = 0.0;
  for (int q = 0; q < parts; ++q) e += part[q];
  ctl->energy = e;
  const bool degenerate = e <= kEps * kEps * ctl->total0;
  if (!second) {
    ctl->redraw = degenerate ? 1 : 0;
  } else {
    ctl->redraw = 0;
    if (degenerate) { ctl->status = kMfDegenerate; ctl->skip = 1; }
  }
}

// a = rhat[j], 1/a
__global__ void mf_pivot_kernel(MfCtl* ctl, const double* rhat) {
  if (ctl->skip || threadIdx.x != 0) return;
  const double a = rhat[ctl->j];
  ctl->a = a;
  ctl->inv_a = 1.0 / a;
}

// chat = c - t
__global__ void __launch_bounds__(256) mf_resid_col_kernel(const MfCtl* ctl, long long n,
                                                           const double* c, const double* t,
                                                           double* chat) {
  if (ctl->skip) return;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x)
    chat[q] = __dsub_rn(c[q], t[q]);
}

// l = rhat * (1/a) (numpy's complex division by a real value), partial |l|^2
__global__ void __launch_bounds__(kRedThreads) mf_make_l_kernel(const MfCtl* ctl, long long m,
                                                                const double* rhat, double* l,
                                                                double* part) {
  __shared__ double red[kRedThreads / 32];
  if (ctl->skip) return;
  const double ia = ctl->inv_a;
  double s = 0.0;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < m;
       q += (long long)gridDim.x * blockDim.x) {
    const double v = __dmul_rn(rhat[q], ia);
    l[q] = v;
    s += __dmul_rn(v, v);
  }
  const double b = block_sum256(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = b;
}

__global__ void mf_l2_kernel(MfCtl* ctl, const double* part, int parts) {
  if (ctl->skip || threadIdx.x != 0) return;
  double e = 0.0;
  for (int q = 0; q < parts; ++q) e += part[q];
  ctl->l2 = e;
}

// K9 downdate (lowmem_cur.py:277-285) with the clamp count against
// eps * prev_total / n; one rounding per numpy ufunc
__global__ void __launch_bounds__(kRedThreads) mf_downdate_kernel(const MfCtl* ctl, long long n,
                                                                  double* nrow, const double* g,
                                                                  const double* v,
                                                                  const double* chat,
                                                                  double* psum,
                                                                  long long* pcnt) {
  __shared__ double red[kRedThreads / 32];
  __shared__ long long redc[kRedThreads / 32];
  if (ctl->skip) return;
  const double l2 = ctl->l2;
  const double floor = kEps * ctl->total / (double)n;
  double s = 0.0;
  long long cnt = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double ch = chat[i];
    double x = nrow[i];
    x = __dsub_rn(x, __dmul_rn(2.0, __dmul_rn(__dsub_rn(g[i], v[i]), ch)));
    x = __dadd_rn(x, __dmul_rn(l2, __dmul_rn(ch, ch)));
    if (x < -floor) ++cnt;
    x = x > 0.0 ? x : 0.0;
    nrow[i] = x;
    s += x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0) redc[threadIdx.x >> 5] = cnt;
  const double b = block_sum256(s, red);
  if (threadIdx.x == 0) {
    long long c = 0;
    for (int w = 0; w < kRedThreads / 32; ++w) c += redc[w];
    psum[blockIdx.x] = b;
    pcnt[blockIdx.x] = c;
  }
}

// the new total and clamp count; the history rows of this step
__global__ void mf_total_kernel(MfCtl* ctl, const double* psum, const long long* pcnt, int parts,
                                double* total_hist, long long* clamp_hist) {
  if (ctl->skip || threadIdx.x != 0) return;
  double t = 0.0;
  long long c = 0;
  for (int q = 0; q < parts; ++q) { t += psum[q]; c += pcnt[q]; }
  ctl->prev_total = ctl->total;
  ctl->total = t;
  ctl->clamped = c;
  clamp_hist[ctl->step] = c;
  total_hist[ctl->step + 1] = t;
}

// Core extension W -> [[W, c[I]], [r[J], r[j]]] with the LU update, the
// index sets and the inverse-mode degeneracy test (lowmem_cur.py:106-125:
// |sigma| <= 1e-14 (|omega| + |z| |W^{-1} w|), sigma = omega - z W^{-1} w).
__global__ void __launch_bounds__(256) mf_extend_kernel(MfCtl* ctl, long long kmax,
                                                        double* Lr, double* Lc, double* Ur,
                                                        double* Uc, double* W, long long* I,
                                                        long long* J, long long* rows,
                                                        long long* cols, const double* r,
                                                        const double* c, const double* p,
                                                        const double* q, const double* xw) {
  __shared__ double red[kRedThreads / 32];
  __shared__ long long s_i, s_j, s_k;
  if (ctl->skip) return;
  if (threadIdx.x == 0) { s_i = ctl->i; s_j = ctl->j; s_k = ctl->step; }
  __syncthreads();
  const long long k = s_k, i = s_i, j = s_j;
  double pq = 0.0, zz = 0.0, xx = 0.0;
  for (long long s = threadIdx.x; s < k; s += blockDim.x) {
    const double ps = p[s], qs = q[s];
    Lr[k * kmax + s] = ps;           // row k of L
    Lc[s * kmax + k] = ps;           // column s of L, entry k
    Ur[s * kmax + k] = qs;           // row s of U, entry k
    Uc[k * kmax + s] = qs;           // column k of U
    const double z = r[J[s]], w = c[I[s]];
    W[k * kmax + s] = z;             // new core row A[i, J]
    W[s * kmax + k] = w;             // new core column A[I, j]
    pq = fma(ps, qs, pq);
    zz = fma(z, z, zz);
    xx = fma(xw[s], xw[s], xx);
  }
  pq = block_sum256(pq, red);
  __syncthreads();
  zz = block_sum256(zz, red);
  __syncthreads();
  xx = block_sum256(xx, red);
  if (threadIdx.x == 0) {
    const double omega = r[j];
    const double delta = omega - pq;
    Lr[k * kmax + k] = 1.0;
    Lc[k * kmax + k] = 1.0;
    Ur[k * kmax + k] = delta;
    Uc[k * kmax + k] = delta;
    W[k * kmax + k] = omega;
    I[k] = i;
    J[k] = j;
    rows[k] = i;
    cols[k] = j;
    const double guard = fabs(omega) + sqrt(zz) * sqrt(xx);
    if (fabs(delta) <= 1e-14 * fmax(guard, 1e-300)) ctl->fell_back = 1;
    ctl->step = k + 1;
  }
}

// tol stop on the current total (lowmem_cur.py:294-297)
__global__ void mf_tol_kernel(MfCtl* ctl, double stop_tol) {
  if (ctl->skip || threadIdx.x != 0) return;
  if (stop_tol > 0.0 && ctl->total <= stop_tol * stop_tol * ctl->total0) {
    ctl->status = kMfTol;
    ctl->skip = 1;
  }
}

// degenerate stop at the top of a step (sum(n_row) <= 0)
__global__ void mf_begin_kernel(MfCtl* ctl) {
  if (ctl->skip || threadIdx.x != 0) return;
  ctl->redraw = 0;
  if (!(ctl->total > 0.0)) { ctl->status = kMfDegenerate; ctl->skip = 1; }
}

__global__ void mf_init_kernel(MfCtl* ctl, const double* part, int parts, double* total_hist) {
  if (threadIdx.x != 0) return;
  double t = 0.0;
  for (int q = 0; q < parts; ++q) t += part[q];
  memset(ctl, 0, sizeof(MfCtl));
  ctl->one = 1;
  ctl->total0 = t;
  ctl->total = t;
  ctl->prev_total = t;
  total_hist[0] = t;
  if (t == 0.0) { ctl->status = kMfDegenerate; ctl->skip = 1; }  // lowmem_cur.py:237-240
}

// partial sums of a vector (initial total of the row norms)
__global__ void __launch_bounds__(kRedThreads) mf_sum_kernel(const double* x, long long n,
                                                             double* part) {
  __shared__ double red[kRedThreads / 32];
  double s = 0.0;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x)
    s += x[q];
  const double b = block_sum256(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = b;
}

// ---------------------------------------------------------------------------
// rebuild (lowmem_cur.py:204-209): n_row_t = sum_j |A_tj - (A[:,J] M)_tj|^2,
// M = W^{-1} A[I, :], over column chunks of kRebuildCols.
constexpr int kRebuildCols = 32;

// M chunk (k x cb, row-major ld cb) = W^{-1} A[I, j0:j0+cb]: one CTA per column
__global__ void __launch_bounds__(kSolveThreads) mf_rebuild_solve_kernel(
    MfOp op, const double* Lc, const double* Uc, long long kmax, long long k,
    const long long* I, long long j0, int cb, double* M) {
  __shared__ double sx[2];
  const long long jc = j0 + blockIdx.x;
  if (jc >= op.m) return;
  const ExpTab tl = exp2tab_lane();
  const int tid = threadIdx.x;
  double b[kSolvePer];
#pragma unroll
  for (int r = 0; r < kSolvePer; ++r) {
    const long long s = tid + (long long)r * kSolveThreads;
    const long long ss = s < k ? s : 0;
    double e;
    if (op.kind == 0) {
      const double* pp = op.P + 3 * I[ss];
      const double* qq = op.Q + 3 * jc;
      e = gauss_entry(op.c * pp[0], op.c * pp[1], op.c * pp[2], op.c * qq[0], op.c * qq[1],
                      op.c * qq[2], tl);
    } else {
      e = op.A[I[ss] * op.lda + jc];
    }
    b[r] = s < k ? e : 0.0;
  }
  for (long long t = 0; t < k; ++t) {            // L q = b
    const int owner = (int)(t % kSolveThreads), slot = (int)(t / kSolveThreads);
    if (tid == owner) {
#pragma unroll
      for (int r = 0; r < kSolvePer; ++r)
        if (r == slot) sx[t & 1] = b[r];
    }
    __syncthreads();
    const double xt = sx[t & 1];
    const double* col = Lc + t * kmax;
#pragma unroll
    for (int r = 0; r < kSolvePer; ++r) {
      const long long s = tid + (long long)r * kSolveThreads;
      if (s > t && s < k) b[r] = fma(-col[s], xt, b[r]);
    }
  }
  __syncthreads();
  for (long long t = k - 1; t >= 0; --t) {       // U x = q
    const int owner = (int)(t % kSolveThreads), slot = (int)(t / kSolveThreads);
    if (tid == owner) {
#pragma unroll
      for (int r = 0; r < kSolvePer; ++r)
        if (r == slot) {
          b[r] = b[r] / Uc[t * kmax + t];
          sx[t & 1] = b[r];
        }
    }
    __syncthreads();
    const double xt = sx[t & 1];
    const double* col = Uc + t * kmax;
#pragma unroll
    for (int r = 0; r < kSolvePer; ++r) {
      const long long s = tid + (long long)r * kSolveThreads;
      if (s < t) b[r] = fma(-col[s], xt, b[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < kSolvePer; ++r) {
    const long long s = tid + (long long)r * kSolveThreads;
    if (s < k) M[s * cb + blockIdx.x] = b[r];
  }
}

// n_row_t += sum_{c < cb} (A_t,j0+c - sum_s A_t,J_s M[s][c])^2, thread per row t
__global__ void __launch_bounds__(256) mf_rebuild_rows_kernel(MfOp op, const long long* J,
                                                              long long k, const double* M,
                                                              long long j0, int cb,
                                                              double* nrow) {
  __shared__ double sm[64 * kRebuildCols];
  __shared__ double sq[64 * 4];
  const ExpTab tl = exp2tab_lane();
  const long long t0 = (long long)blockIdx.x * blockDim.x;
  const long long t = t0 + threadIdx.x;
  const long long tt = t < op.n ? t : op.n - 1;
  double px = 0, py = 0, pz = 0;
  if (op.kind == 0) {
    px = op.c * op.P[tt * 3];
    py = op.c * op.P[tt * 3 + 1];
    pz = op.c * op.P[tt * 3 + 2];
  }
  double acc[kRebuildCols];
#pragma unroll
  for (int c = 0; c < kRebuildCols; ++c) {
    const long long jc = j0 + c;
    double e = 0.0;
    if (c < cb) {
      if (op.kind == 0) {
        const double* qq = op.Q + 3 * jc;
        e = gauss_entry(px, py, pz, op.c * qq[0], op.c * qq[1], op.c * qq[2], tl);
      } else {
        e = op.A[tt * op.lda + jc];
      }
    }
    acc[c] = e;
  }
  for (long long s0 = 0; s0 < k; s0 += 64) {
    const int cnt = (int)min(64LL, k - s0);
    __syncthreads();
    for (int q = threadIdx.x; q < cnt * kRebuildCols; q += blockDim.x) {
      const int s = q / kRebuildCols, c = q % kRebuildCols;
      sm[q] = c < cb ? M[(s0 + s) * cb + c] : 0.0;
    }
    if (op.kind == 0)
      for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
        const double* qq = op.Q + 3 * J[s0 + q];
        sq[q * 4] = op.c * qq[0];
        sq[q * 4 + 1] = op.c * qq[1];
        sq[q * 4 + 2] = op.c * qq[2];
      }
    __syncthreads();
    for (int s = 0; s < cnt; ++s) {
      double e;
      if (op.kind == 0) e = gauss_entry(px, py, pz, sq[s * 4], sq[s * 4 + 1], sq[s * 4 + 2], tl);
      else e = op.A[tt * op.lda + J[s0 + s]];
#pragma unroll
      for (int c = 0; c < kRebuildCols; ++c) acc[c] = fma(-e, sm[s * kRebuildCols + c], acc[c]);
    }
  }
  double ssum = 0.0;
#pragma unroll
  for (int c = 0; c < kRebuildCols; ++c) ssum = fma(acc[c], acc[c], ssum);
  if (t < op.n) nrow[t] += ssum;
}

inline int blocks_for(long long n, int threads, int cap) {
  return (int)std::max<long long>(1, std::min<long long>((n + threads - 1) / threads, cap));
}

}  // namespace

int mf_run_impl(rplu_ctx* ctx, const rplu_mf_args* a, rplu_mf_out* out) {
  if (!a || !out) { set_error("rplu_mf_run: NULL argument"); return RPLU_ERR_ARG; }
  const long long n = a->n, m = a->m, rank = a->rank;
  if (n < 1 || m < 1 || rank < 0 || rank > std::min(n, m)) {
    set_error("rank out of range");
    return RPLU_ERR_ARG;
  }
  if (rank > (long long)kSolveThreads * kSolvePer) {
    set_error("rplu_mf_run: rank above 8192 is not supported by the device core solves");
    return RPLU_ERR_CAPABILITY;
  }
  if (a->rule != RPLU_RULE_RPLU && a->rule != RPLU_RULE_C2PLU) {
    set_error("unknown CUR rule");
    return RPLU_ERR_ARG;
  }
  const bool greedy = a->rule == RPLU_RULE_C2PLU;
  if (!greedy && (!a->uniforms || a->n_uniforms < 1) && rank > 0) {
    set_error("rplu-cur needs a uniform stream");
    return RPLU_ERR_ARG;
  }
  MfOp op{};
  op.n = n;
  op.m = m;
  if (a->op_kind == RPLU_MF_GAUSS3D) {
    if (!a->P || !a->Q || !(a->h > 0.0)) { set_error("invalid Gaussian-kernel operator"); return RPLU_ERR_ARG; }
    op.kind = 0;
    op.P = a->P;
    op.Q = a->Q;
    op.c = 1.0 / (1.4142135623730951 * a->h);
  } else if (a->op_kind == RPLU_MF_DENSE) {
    if (!a->A || a->lda < m) { set_error("invalid dense operator"); return RPLU_ERR_ARG; }
    op.kind = 1;
    op.A = a->A;
    op.lda = a->lda;
  } else {
    set_error("unknown matrix-free operator kind");
    return RPLU_ERR_CAPABILITY;
  }
  cudaStream_t s = static_cast<cudaStream_t>(a->stream);
  const long long kmax = std::max(rank, 1LL);
  const int red_blocks = 4 * ctx->sm_count;
  const long long nch_n = (n + kChunk - 1) / kChunk, nch_m = (m + kChunk - 1) / kChunk;
  const bool chunk_n = n >= kChunkedMinN, chunk_m = m >= kChunkedMinN;

  // workspace: vectors, core factors, histories, partials
  std::vector<std::pair<void**, size_t>> plan;
  double *nrow, *r, *rhat, *w, *tmpm, *l, *c, *chat, *g, *v, *tmpn;
  double *Lr, *Lc, *Ur, *Uc, *W, *pbuf, *qbuf, *xbuf, *ybuf, *zbuf, *total_hist, *part, *psum;
  double *uni, *ctot, *Mbuf;
  long long *I, *J, *rows, *cols, *clamp_hist, *pcnt;
  int* neg;
  MfCtl* ctl;
  const size_t kk = (size_t)kmax * kmax;
  const size_t cbuf = (size_t)std::max(nch_n, nch_m) + 1;
  size_t off = 0;
  auto carve = [&](auto** p, size_t bytes) {
    off = (off + 255) & ~(size_t)255;
    plan.push_back({reinterpret_cast<void**>(p), off});
    off += bytes;
  };
  carve(&nrow, 8 * n); carve(&r, 8 * m); carve(&rhat, 8 * m); carve(&w, 8 * m);
  carve(&tmpm, 8 * m); carve(&l, 8 * m); carve(&c, 8 * n); carve(&chat, 8 * n);
  carve(&g, 8 * n); carve(&v, 8 * n); carve(&tmpn, 8 * n);
  carve(&Lr, 8 * kk); carve(&Lc, 8 * kk); carve(&Ur, 8 * kk); carve(&Uc, 8 * kk);
  carve(&W, 8 * kk);
  carve(&pbuf, 8 * kmax); carve(&qbuf, 8 * kmax); carve(&xbuf, 8 * kmax);
  carve(&ybuf, 8 * kmax); carve(&zbuf, 8 * kmax);
  carve(&total_hist, 8 * (rank + 1)); carve(&part, 8 * red_blocks); carve(&psum, 8 * red_blocks);
  carve(&uni, 8 * std::max<long long>(a->n_uniforms, 1)); carve(&ctot, 8 * cbuf);
  carve(&Mbuf, 8 * kmax * kRebuildCols);
  carve(&I, 8 * kmax); carve(&J, 8 * kmax); carve(&rows, 8 * kmax); carve(&cols, 8 * kmax);
  carve(&clamp_hist, 8 * kmax); carve(&pcnt, 8 * red_blocks);
  carve(&neg, 16); carve(&ctl, sizeof(MfCtl));
  int rc;
  if ((rc = ctx->mf_buf.ensure(off + 256))) return rc;
  char* base = reinterpret_cast<char*>(ctx->mf_buf.ptr);
  for (auto& e : plan) *e.first = base + e.second;
  if (!greedy && a->n_uniforms > 0)
    RPLU_CUDA(cudaMemcpyAsync(uni, a->uniforms, sizeof(double) * a->n_uniforms,
                              cudaMemcpyHostToDevice, s));
  // L, U copies and W are carved consecutively: zero them in one call
  RPLU_CUDA(cudaMemsetAsync(Lr, 0, reinterpret_cast<char*>(W + kk) - reinterpret_cast<char*>(Lr),
                            s));
  long long launches = 0;
  GaussOp gop{n, m, op.P, op.Q, op.c};
  float gemv_total = 0.f;   // K7 time: the initial row-norm pass + one pass per step
  const bool time_gemv = (a->flags & RPLU_FLAG_TIME_KERNELS) != 0;

  // initial row norms (accessor row_norms(), lowmem_cur.py:235-236) and total0
  if (op.kind == 0) {
    float ms0 = 0.f;   // the row-norm pass is the same K7 kernel (squares)
    if ((rc = gauss_gemv_impl(ctx, gop, nullptr, nrow, true, s, time_gemv ? &ms0 : nullptr)))
      return rc;
    gemv_total += ms0;
    launches += 2;
  } else {
    mf_dense_gemv_kernel<<<blocks_for(n * 32, 256, 8 * ctx->sm_count), 256, 0, s>>>(op, nullptr,
                                                                                   1, nrow);
    ++launches;
  }
  mf_sum_kernel<<<red_blocks, kRedThreads, 0, s>>>(nrow, n, part);
  mf_init_kernel<<<1, 32, 0, s>>>(ctl, part, red_blocks, total_hist);
  launches += 2;
  RPLU_CUDA(cudaGetLastError());

  MfCtl h{};
  RPLU_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(MfCtl), cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaStreamSynchronize(s));
  long long rebuilds = 0;
  const int* one = &ctl->one;
  const int* redraw = &ctl->redraw;
  const int lblocks_m = blocks_for(m, 256, 4096), lblocks_n = blocks_for(n, 256, 4096);
  const int eb_m = blocks_for(m, kRedThreads, red_blocks);
  const int eb_n = blocks_for(n, kRedThreads, red_blocks);
  const double* uptr = greedy ? nullptr : uni;

  auto restricted = [&](int axis, const long long* sel, const double* y, long long k,
                        double* outv) -> int {
    if (op.kind == 0) {
      launches += 1;
      return axis == 0 ? gauss_restricted_impl(ctx, op.Q, m, op.P, sel, y, k, op.c, outv, s)
                       : gauss_restricted_impl(ctx, op.P, n, op.Q, sel, y, k, op.c, outv, s);
    }
    if (k == 0) {
      RPLU_CUDA(cudaMemsetAsync(outv, 0, 8 * (axis == 0 ? m : n), s));
      return RPLU_OK;
    }
    mf_dense_restricted_kernel<<<blocks_for(axis == 0 ? m : n, 256, 16 * ctx->sm_count), 256, 0,
                                 s>>>(op, axis, sel, y, k, outv);
    launches += 1;
    return RPLU_OK;
  };
  auto draw = [&](const int* gate, const double* wv, long long len, bool chunked, long long nch,
                  int which) {
    if (!greedy && chunked) {
      RPLU_CUDA(cudaMemsetAsync(neg, 0, sizeof(int), s));
      mf_chunk_totals_kernel<<<(unsigned)nch, 1024, 0, s>>>(ctl, gate, wv, len, ctot, neg);
      ++launches;
    }
    mf_draw_kernel<<<1, 1024, 0, s>>>(ctl, gate, wv, len, uptr, a->n_uniforms, greedy ? 1 : 0,
                                      which, (!greedy && chunked) ? ctot : nullptr, nch);
    ++launches;
    return RPLU_OK;
  };
  // residual row i: r, p = U^{-T} r[J], y = W^{-T} r[J], rhat, w, energy check
  auto residual_row = [&](const int* gate, long long k, int second) -> int {
    int e;
    if ((e = draw(gate, nrow, n, chunk_n, nch_n, 0))) return e;
    mf_line_kernel<<<lblocks_m, 256, 0, s>>>(op, ctl, gate, 0, r);
    ++launches;
    if (k > 0) {
      mf_solve_kernel<<<1, kSolveThreads, 0, s>>>(ctl, gate, 1, Lr, Lc, Ur, Uc, kmax, k, r, J,
                                                  pbuf, ybuf);
      ++launches;
    }
    if ((e = restricted(0, I, ybuf, k, tmpm))) return e;
    mf_resid_row_kernel<<<eb_m, kRedThreads, 0, s>>>(ctl, gate, m, r, tmpm, rhat, w, part);
    mf_energy_kernel<<<1, 32, 0, s>>>(ctl, gate, part, eb_m, second);
    launches += 2;
    return RPLU_OK;
  };

  long long k = 0;
  for (; k < rank && !h.skip; ) {
    mf_begin_kernel<<<1, 32, 0, s>>>(ctl);
    ++launches;
    if ((rc = residual_row(one, k, 0))) return rc;
    if ((rc = residual_row(redraw, k, 1))) return rc;     // runs only on a degenerate row
    // column draw and pivot
    if ((rc = draw(one, w, m, chunk_m, nch_m, 1))) return rc;
    mf_pivot_kernel<<<1, 32, 0, s>>>(ctl, rhat);
    mf_line_kernel<<<lblocks_n, 256, 0, s>>>(op, ctl, one, 1, c);
    launches += 2;
    if (k > 0) {
      mf_solve_kernel<<<1, kSolveThreads, 0, s>>>(ctl, one, 0, Lr, Lc, Ur, Uc, kmax, k, c, I,
                                                  qbuf, xbuf);
      ++launches;
    }
    if ((rc = restricted(1, J, xbuf, k, tmpn))) return rc;
    mf_resid_col_kernel<<<lblocks_n, 256, 0, s>>>(ctl, n, c, tmpn, chat);
    mf_make_l_kernel<<<eb_m, kRedThreads, 0, s>>>(ctl, m, rhat, l, part);
    mf_l2_kernel<<<1, 32, 0, s>>>(ctl, part, eb_m);
    launches += 3;
    // g = A l: the step's one full operator pass (K7)
    if (op.kind == 0) {
      float ms = 0.f;
      if ((rc = gauss_gemv_impl(ctx, gop, l, g, false, s, time_gemv ? &ms : nullptr))) return rc;
      gemv_total += ms;
      launches += 2;
    } else {
      mf_dense_gemv_kernel<<<blocks_for(n * 32, 256, 8 * ctx->sm_count), 256, 0, s>>>(op, l, 0,
                                                                                     g);
      ++launches;
    }
    if (k > 0) {
      mf_solve_kernel<<<1, kSolveThreads, 0, s>>>(ctl, one, 0, Lr, Lc, Ur, Uc, kmax, k, g, I,
                                                  nullptr, zbuf);
      ++launches;
    }
    if ((rc = restricted(1, J, zbuf, k, v))) return rc;
    mf_downdate_kernel<<<eb_n, kRedThreads, 0, s>>>(ctl, n, nrow, g, v, chat, psum, pcnt);
    mf_total_kernel<<<1, 32, 0, s>>>(ctl, psum, pcnt, eb_n, total_hist, clamp_hist);
    mf_extend_kernel<<<1, 256, 0, s>>>(ctl, kmax, Lr, Lc, Ur, Uc, W, I, J, rows, cols, r, c,
                                       pbuf, qbuf, xbuf);
    launches += 3;
    RPLU_CUDA(cudaGetLastError());
    RPLU_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(MfCtl), cudaMemcpyDeviceToHost, s));
    RPLU_CUDA(cudaStreamSynchronize(s));
    if (h.skip) break;           // degenerate row / uniforms exhausted: no pivot this step
    k = h.step;
    if ((double)h.clamped > 0.01 * (double)n) {
      // rebuild n_row from m residual columns (lowmem_cur.py:290-292)
      RPLU_CUDA(cudaMemsetAsync(nrow, 0, 8 * n, s));
      for (long long j0 = 0; j0 < m; j0 += kRebuildCols) {
        const int cb = (int)std::min<long long>(kRebuildCols, m - j0);
        mf_rebuild_solve_kernel<<<cb, kSolveThreads, 0, s>>>(op, Lc, Uc, kmax, k, I, j0, cb,
                                                             Mbuf);
        mf_rebuild_rows_kernel<<<blocks_for(n, 256, 1 << 30), 256, 0, s>>>(op, J, k, Mbuf, j0,
                                                                           cb, nrow);
        launches += 2;
      }
      mf_sum_kernel<<<red_blocks, kRedThreads, 0, s>>>(nrow, n, part);
      ++launches;
      RPLU_CUDA(cudaGetLastError());
      std::vector<double> hp(red_blocks);
      RPLU_CUDA(cudaMemcpyAsync(hp.data(), part, 8 * red_blocks, cudaMemcpyDeviceToHost, s));
      RPLU_CUDA(cudaStreamSynchronize(s));
      double t = 0.0;
      for (double x : hp) t += x;
      RPLU_CUDA(cudaMemcpyAsync(&total_hist[k], &t, 8, cudaMemcpyHostToDevice, s));
      RPLU_CUDA(cudaMemcpyAsync(&ctl->total, &t, 8, cudaMemcpyHostToDevice, s));
      ++rebuilds;
    }
    mf_tol_kernel<<<1, 32, 0, s>>>(ctl, a->stop_tol);
    ++launches;
    RPLU_CUDA(cudaMemcpyAsync(&h, ctl, sizeof(MfCtl), cudaMemcpyDeviceToHost, s));
    RPLU_CUDA(cudaStreamSynchronize(s));
  }
  k = h.step;
  // results
  out->steps_done = k;
  out->uniforms_consumed = h.ucount;
  out->near_boundary_draws = h.near;
  out->rebuilds = rebuilds;
  out->degenerate_stop = h.status == kMfDegenerate ? 1 : 0;
  out->tol_stop = h.status == kMfTol ? 1 : 0;
  out->core_fell_back = h.fell_back;
  out->gemv_ms = gemv_total;
  if (out->rows && k) RPLU_CUDA(cudaMemcpyAsync(out->rows, rows, 8 * k, cudaMemcpyDeviceToHost, s));
  if (out->cols && k) RPLU_CUDA(cudaMemcpyAsync(out->cols, cols, 8 * k, cudaMemcpyDeviceToHost, s));
  if (out->total_sq_norms)
    RPLU_CUDA(cudaMemcpyAsync(out->total_sq_norms, total_hist, 8 * (k + 1),
                              cudaMemcpyDeviceToHost, s));
  if (out->clamped && k)
    RPLU_CUDA(cudaMemcpyAsync(out->clamped, clamp_hist, 8 * k, cudaMemcpyDeviceToHost, s));
  if (out->core && k)
    RPLU_CUDA(cudaMemcpy2DAsync(out->core, 8 * k, W, 8 * kmax, 8 * k, k, cudaMemcpyDeviceToHost,
                                s));
  if (out->row_norms_dev)
    RPLU_CUDA(cudaMemcpyAsync(out->row_norms_dev, nrow, 8 * n, cudaMemcpyDeviceToDevice, s));
  if (out->row_norms)
    RPLU_CUDA(cudaMemcpyAsync(out->row_norms, nrow, 8 * n, cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaStreamSynchronize(s));
  if (h.status == kMfUniforms) {
    set_error("uniform stream exhausted");
    return RPLU_ERR_ARG;
  }
  out->kernel_launches = launches;
  count_launches(launches);
  return RPLU_OK;
}

}  // namespace rplu
