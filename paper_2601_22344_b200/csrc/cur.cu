// Matrix-free CUR-form RPLU (Alg 2) device kernels for the Gaussian-kernel
// operator A_ij = exp(-|p_i - q_j|^2 / (2 h^2)) (BASELINE configs[4]).
//
// Reference: rplu.lowmem_cur.cur_build (pkg/src/rplu/lowmem_cur.py:212-300).
// The reference touches A only through full applies (4 of A + 2 of A^T per
// step, :161-187, :266-275, :303-312).  Here:
//   K7  gauss_apply      full generated GEMV g = A l (the one O(nm) pass per
//                        step, :273), FP64-pipe bound: no matrix in HBM
//   K8  gauss_rows/cols  k-restricted products A[I,:]^T w and A[:,J] w
//                        (:174-187; the reference spends a full apply on a
//                        k-sparse vector), single rows/columns A[i,:], A[:,j]
//   K9  cur_downdate     n_row -= 2 Re((g-v) conj(chat)); += |l|^2 |chat|^2;
//                        clamp count against eps*prev/n; total (:277-285)
// All vectors are real fp64: the operator is real, so the reference's
// complex128 vectors carry zero imaginary parts throughout.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "rplu_common.cuh"
#include "rplu_internal.h"
#include "gauss.cuh"

namespace rplu {

// ---------------------------------------------------------------------------
// K7: out[i] (+split partial) = sum_j A_ij v_j, or sum_j A_ij^2 (SQUARE, v
// ignored) for row norms.  Row side in registers, column side (q_j, v_j) in
// shared-memory tiles; columns split across gridDim.y for small n.
template <int RPT, int TJ, bool SQUARE>
__global__ void __launch_bounds__(256) gauss_gemv_kernel(GaussOp op, const double* __restrict__ v,
                                                         double* __restrict__ partial, int splits) {
  constexpr int NT = 256;
  __shared__ double sq[TJ * 4];
  const long long row_base = (long long)blockIdx.x * NT * RPT;
  const long long cols_per = (op.m + splits - 1) / splits;
  const long long j0 = (long long)blockIdx.y * cols_per;
  const long long j1 = min(op.m, j0 + cols_per);
  const ExpTab tl = exp2tab_lane();
  double px[RPT], py[RPT], pz[RPT], acc[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    long long i = row_base + threadIdx.x + (long long)r * NT;
    long long ii = i < op.n ? i : 0;
    px[r] = op.c * op.P[ii * 3 + 0];
    py[r] = op.c * op.P[ii * 3 + 1];
    pz[r] = op.c * op.P[ii * 3 + 2];
    acc[r] = 0.0;
  }
  for (long long jt = j0; jt < j1; jt += TJ) {
    const int cnt = (int)min((long long)TJ, j1 - jt);
    __syncthreads();
    for (int cc = threadIdx.x; cc < cnt; cc += NT) {
      const long long j = jt + cc;
      sq[cc * 4 + 0] = op.c * op.Q[j * 3 + 0];
      sq[cc * 4 + 1] = op.c * op.Q[j * 3 + 1];
      sq[cc * 4 + 2] = op.c * op.Q[j * 3 + 2];
      sq[cc * 4 + 3] = SQUARE ? 1.0 : v[j];
    }
    __syncthreads();
#pragma unroll 4
    for (int cc = 0; cc < cnt; ++cc) {
      const double qx = sq[cc * 4 + 0], qy = sq[cc * 4 + 1], qz = sq[cc * 4 + 2];
      const double vj = sq[cc * 4 + 3];
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const double e = gauss_entry(px[r], py[r], pz[r], qx, qy, qz, tl);
        acc[r] = SQUARE ? fma(e, e, acc[r]) : fma(e, vj, acc[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    long long i = row_base + threadIdx.x + (long long)r * NT;
    if (i < op.n) partial[(long long)blockIdx.y * op.n + i] = acc[r];
  }
}

__global__ void reduce_splits_kernel(const double* partial, int splits, long long n, double* out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int k = 0; k < splits; ++k) s += partial[(long long)k * n + i];
  out[i] = s;
}

// K8: single row A[i,:] (m) or column A[:,j] (n) — out[k] = entry(base, pts[k])
__global__ void gauss_line_kernel(const double* __restrict__ pts, long long count,
                                  const double* __restrict__ base, double c, double* out) {
  const double bx = c * base[0], by = c * base[1], bz = c * base[2];
  const ExpTab tl = exp2tab_lane();
  const long long stride = (long long)gridDim.x * blockDim.x;
  // warp-uniform trip count (the exp's table shuffle needs every lane)
  for (long long k0 = (long long)blockIdx.x * blockDim.x; k0 < count; k0 += stride) {
    const long long k = k0 + threadIdx.x;
    const long long kk = k < count ? k : count - 1;
    const double e = gauss_entry(bx, by, bz, c * pts[kk * 3], c * pts[kk * 3 + 1],
                                 c * pts[kk * 3 + 2], tl);
    if (k < count) out[k] = e;
  }
}

// K8: out[t] = sum_s w_s A(sel_s, t) over `count` targets t, where the k
// selected points (rows I or columns J) and their weights are staged in smem.
// A[I,:]^T w: targets = Q (m), selected = P[I];  A[:,J] w: targets = P (n),
// selected = Q[J].  The kernel is symmetric in its point arguments.
__global__ void __launch_bounds__(256) gauss_restricted_kernel(
    const double* __restrict__ targets, long long count, const double* __restrict__ selpts,
    const long long* __restrict__ sel, const double* __restrict__ w, long long k, double c,
    double* out) {
  extern __shared__ double ss[];  // k * 4
  for (long long s = threadIdx.x; s < k; s += blockDim.x) {
    const long long ix = sel[s];
    ss[s * 4 + 0] = c * selpts[ix * 3 + 0];
    ss[s * 4 + 1] = c * selpts[ix * 3 + 1];
    ss[s * 4 + 2] = c * selpts[ix * 3 + 2];
    ss[s * 4 + 3] = w[s];
  }
  __syncthreads();
  const ExpTab tl = exp2tab_lane();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t0 = (long long)blockIdx.x * blockDim.x; t0 < count; t0 += stride) {
    const long long t = t0 + threadIdx.x;
    const long long tt = t < count ? t : count - 1;
    const double tx = c * targets[tt * 3], ty = c * targets[tt * 3 + 1],
                 tz = c * targets[tt * 3 + 2];
    double acc = 0.0;
    for (long long s = 0; s < k; ++s)
      acc = fma(gauss_entry(ss[s * 4], ss[s * 4 + 1], ss[s * 4 + 2], tx, ty, tz, tl),
                ss[s * 4 + 3], acc);
    if (t < count) out[t] = acc;
  }
}

// K9: row-norm downdate with clamp (lowmem_cur.py:277-285), per-CTA partial
// (sum, clamp count) written for a deterministic second-stage reduction.
__global__ void __launch_bounds__(256) cur_downdate_kernel(long long n, double* nrow,
                                                           const double* g, const double* v,
                                                           const double* chat, double l2,
                                                           double floor, double* psum,
                                                           long long* pcnt) {
  double s = 0.0;
  long long cnt = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double ch = chat[i];
    double x = nrow[i];
    // one rounding per numpy ufunc, as in the reference (no contraction)
    x = __dsub_rn(x, __dmul_rn(2.0, __dmul_rn(__dsub_rn(g[i], v[i]), ch)));
    x = __dadd_rn(x, __dmul_rn(l2, __dmul_rn(ch, ch)));
    if (x < -floor) ++cnt;
    x = x > 0.0 ? x : 0.0;
    nrow[i] = x;
    s += x;
  }
  s = warp_sum(s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  __shared__ double ws[8];
  __shared__ long long wc[8];
  if ((threadIdx.x & 31) == 0) { ws[threadIdx.x >> 5] = s; wc[threadIdx.x >> 5] = cnt; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    long long c = 0;
    for (int w = 0; w < 8; ++w) { t += ws[w]; c += wc[w]; }
    psum[blockIdx.x] = t;
    pcnt[blockIdx.x] = c;
  }
}

// ---------------------------------------------------------------------------
// host launchers

// Column splits of K7: at least ~4 CTAs per SM in total, at least 512
// columns per split, and -- since every CTA of one launch runs about equally
// long -- a CTA count that fills its last wave: among the admissible split
// counts take the one with the smallest wave-quantisation loss
// ceil(ctas / slots) / (ctas / slots) (C5: 1954 row blocks on 740 resident
// slots is 2.64 waves with 1 split, 7.92 with 3 splits).
static int gemv_splits(long long n, long long m, int rows_per_cta, int sms, int per_sm) {
  const long long rb = (n + rows_per_cta - 1) / rows_per_cta;
  const long long max_s = std::max(1LL, std::min((m + 511) / 512, 1024LL));
  long long s0 = std::max(1LL, std::min((4LL * sms + rb - 1) / rb, max_s));
  const double slots = (double)sms * std::max(per_sm, 1);
  long long best = s0;
  double best_eff = 0.0;
  for (long long s = s0; s <= std::min(max_s, s0 + 8); ++s) {
    const double waves = (double)(rb * s) / slots;
    const double eff = waves / std::ceil(waves);
    if (eff > best_eff + 0.01) { best_eff = eff; best = s; }
  }
  return (int)best;
}

template <int RPT>
static void gemv_launch(const GaussOp& op, const double* v, double* part, int splits, bool square,
                        cudaStream_t s) {
  constexpr int TJ = 256;
  dim3 grid((unsigned)((op.n + 256 * RPT - 1) / (256 * RPT)), (unsigned)splits);
  if (square) gauss_gemv_kernel<RPT, TJ, true><<<grid, 256, 0, s>>>(op, v, part, splits);
  else gauss_gemv_kernel<RPT, TJ, false><<<grid, 256, 0, s>>>(op, v, part, splits);
}

// rows per thread of K7 (RPLU_GEMV_RPT experiment override: 1, 2 or 4)
static int gemv_rpt() {
  static int v = [] {
    const char* e = getenv("RPLU_GEMV_RPT");
    int r = e ? atoi(e) : 4;   // measured at n = m = 1e6: 1 -> 1417 ms, 2 -> 1347, 4 -> 1336
    return (r == 1 || r == 2) ? r : 4;
  }();
  return v;
}

int gauss_gemv_impl(rplu_ctx* ctx, const GaussOp& op, const double* v, double* out, bool square,
                    cudaStream_t s, float* ms) {
  const int rpt = gemv_rpt();
  static int per_sm[3] = {0, 0, 0};   // resident CTAs per SM of each RPT instantiation
  const int slot = rpt == 1 ? 0 : (rpt == 2 ? 1 : 2);
  if (!per_sm[slot]) {
    int b = 0;
    if (rpt == 1)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, gauss_gemv_kernel<1, 256, false>, 256, 0);
    else if (rpt == 2)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, gauss_gemv_kernel<2, 256, false>, 256, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, gauss_gemv_kernel<4, 256, false>, 256, 0);
    per_sm[slot] = b > 0 ? b : 1;
  }
  const int splits = gemv_splits(op.n, op.m, 256 * rpt, ctx->sm_count, per_sm[slot]);
  int rc;
  if ((rc = ctx->scratch[4].ensure(sizeof(double) * (size_t)splits * op.n))) return rc;
  double* part = reinterpret_cast<double*>(ctx->scratch[4].ptr);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ms) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  count_launches(1);
  if (rpt == 1) gemv_launch<1>(op, v, part, splits, square, s);
  else if (rpt == 2) gemv_launch<2>(op, v, part, splits, square, s);
  else gemv_launch<4>(op, v, part, splits, square, s);
  if (ms) cudaEventRecord(e1, s);
  count_launches(1);
  reduce_splits_kernel<<<(unsigned)((op.n + 255) / 256), 256, 0, s>>>(part, splits, op.n, out);
  RPLU_CUDA(cudaGetLastError());
  if (ms) {
    RPLU_CUDA(cudaEventSynchronize(e1));
    cudaEventElapsedTime(ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return RPLU_OK;
}

int gauss_line_impl(const double* pts, long long count, const double* base, double c, double* out,
                    cudaStream_t s) {
  const int blocks = (int)std::min<long long>((count + 255) / 256, 4096);
  count_launches(1);
  gauss_line_kernel<<<blocks, 256, 0, s>>>(pts, count, base, c, out);
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

int gauss_restricted_impl(rplu_ctx* ctx, const double* targets, long long count,
                          const double* selpts, const long long* sel, const double* w,
                          long long k, double c, double* out, cudaStream_t s) {
  if (k == 0) {
    RPLU_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * count, s));
    return RPLU_OK;
  }
  const size_t smem = sizeof(double) * 4 * (size_t)k;
  if (smem > 48 * 1024) {
    RPLU_CUDA(cudaFuncSetAttribute(gauss_restricted_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  const int blocks = (int)std::min<long long>((count + 255) / 256, 16LL * ctx->sm_count);
  count_launches(1);
  gauss_restricted_kernel<<<blocks, 256, smem, s>>>(targets, count, selpts, sel, w, k, c, out);
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

int cur_downdate_impl(rplu_ctx* ctx, long long n, double* nrow, const double* g, const double* v,
                      const double* chat, double l2, double floor, long long* clamped,
                      double* total, cudaStream_t s) {
  const int blocks = (int)std::min<long long>((n + 255) / 256, 4LL * ctx->sm_count);
  int rc;
  if ((rc = ctx->scratch[5].ensure((sizeof(double) + sizeof(long long)) * (size_t)blocks)))
    return rc;
  double* ps = reinterpret_cast<double*>(ctx->scratch[5].ptr);
  long long* pc = reinterpret_cast<long long*>(ps + blocks);
  count_launches(1);
  cur_downdate_kernel<<<blocks, 256, 0, s>>>(n, nrow, g, v, chat, l2, floor, ps, pc);
  RPLU_CUDA(cudaGetLastError());
  std::vector<double> hs(blocks);
  std::vector<long long> hc(blocks);
  RPLU_CUDA(cudaMemcpyAsync(hs.data(), ps, sizeof(double) * blocks, cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaMemcpyAsync(hc.data(), pc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaStreamSynchronize(s));
  double t = 0.0;
  long long c = 0;
  for (int b = 0; b < blocks; ++b) { t += hs[b]; c += hc[b]; }
  *total = t;
  *clamped = c;
  return RPLU_OK;
}

}  // namespace rplu
