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
//
// Two forms of the exponent, chosen on the device from the points' bounding
// box (gauss_geo_kernel; no host round trip -- both kernels are launched and
// the one that does not apply exits at once):
//  * difference form (gauss_gemv_kernel): -|p'-q'|^2 from three differences,
//    16 FP64-pipe operations per entry, entries to ~1.5 ulp + d2 2^-53;
//  * dot-product form (gauss_gemv_dot_kernel): with the points centred on the
//    middle c0 of Q's bounding box and y the exponent in table units
//    (K = 32/ln2),  y = a_i + b_j + p~_i . q~~_j,  a_i = -K |p~_i|^2,
//    b_j = -K |q~_j|^2,  q~~_j = 2K q~_j  -- three DFMA and one DADD, then
//    exp_tab_units: 14 FP64-pipe operations per entry and no compare/select.
//    y carries an absolute rounding error of a few eps K r2 (r2 = the largest
//    squared scaled distance of a point from c0), i.e. a relative entry error
//    <= ~10 eps K r2 ln2/32; the form is taken only while K r2 < 8000 (then
//    also y > -32000: no underflow cut), so entries agree with the difference
//    form to <= 2e-13 relative in the worst case (C5: K r2 ~ 5600, typical
//    error ~3e-14, below the sqrt(m) eps of the row sum itself).  The centre
//    depends on Q only, so a row-sharded apply produces the same bits as the
//    unsharded one.  Pivot rows / columns and the core (K8) always use the
//    difference form.
constexpr double kExpK = 46.16624130844683;   // 32 / ln 2
constexpr double kDotRange = 8000.0;

// per-CTA bounding boxes: part[b][0..5] = lo/hi of Q, part[b][6..11] = lo/hi of P u Q
__global__ void __launch_bounds__(256) gauss_bbox_kernel(GaussOp op, double* __restrict__ part) {
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double ql[3] = {inf, inf, inf}, qh[3] = {-inf, -inf, -inf};
  double al[3] = {inf, inf, inf}, ah[3] = {-inf, -inf, -inf};
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < op.m; k += stride) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double x = op.Q[k * 3 + c];
      ql[c] = fmin(ql[c], x);
      qh[c] = fmax(qh[c], x);
    }
  }
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < op.n; k += stride) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double x = op.P[k * 3 + c];
      al[c] = fmin(al[c], x);
      ah[c] = fmax(ah[c], x);
    }
  }
  __shared__ double red[8][12];
  double vals[12];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    vals[c] = ql[c];
    vals[3 + c] = -qh[c];
    vals[6 + c] = fmin(al[c], ql[c]);
    vals[9 + c] = -fmax(ah[c], qh[c]);
  }
#pragma unroll
  for (int e = 0; e < 12; ++e) {   // every slot is a minimum (upper bounds negated)
    double x = vals[e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmin(x, __shfl_xor_sync(0xffffffffu, x, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][e] = x;
  }
  __syncthreads();
  if (threadIdx.x < 12) {
    double x = red[0][threadIdx.x];
    for (int w = 1; w < 8; ++w) x = fmin(x, red[w][threadIdx.x]);
    part[blockIdx.x * 12 + threadIdx.x] = x;
  }
}

// geo = [c0x, c0y, c0z, K c^2 r2]: c0 the middle of Q's box, r2 the largest
// squared distance of a corner of the (P u Q) box from c0.  Non-finite
// coordinates give a non-finite range, which selects the difference form.
__global__ void gauss_geo_kernel(const double* __restrict__ part, int nparts, double c,
                                 double* __restrict__ geo) {
  __shared__ double mn[12];
  if (threadIdx.x < 12) {
    double x = part[threadIdx.x];
    for (int b = 1; b < nparts; ++b) x = fmin(x, part[b * 12 + threadIdx.x]);
    mn[threadIdx.x] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double r2 = 0.0;
    for (int k = 0; k < 3; ++k) {
      const double c0 = 0.5 * (mn[k] - mn[3 + k]);
      const double d = fmax(fabs(mn[6 + k] - c0), fabs(-mn[9 + k] - c0)) * c;
      geo[k] = c0;
      r2 += d * d;
    }
    const double range = kExpK * r2;
    geo[3] = range == range ? range : __longlong_as_double(0x7ff0000000000000LL);
  }
}

// FACT (GEMV only): the per-point parts of the exponent are factored out of
// the entry, e_ij = A_i B_j E(t_ij) with A_i = exp(-|p~_i|^2), B_j =
// exp(-|q~_j|^2) and t_ij = p~_i . q~~_j, so that g_i = A_i sum_j (B_j v_j)
// E(t_ij): the column weight w_j = B_j v_j is formed once per tile column and
// A_i once per row, and the entry needs a bare 3-term dot product (DMUL + 2
// DFMA) -- one FP64-pipe instruction less per entry and 4 doubles per column
// in shared memory instead of 5.  Every term of a row carries the same factor
// 1/A_i, so the relative sizes of the summands (and the rounding of the sum)
// are unchanged; K r2 < 8000 keeps A_i, B_j >= 2^-250 and E <= 2^500 inside
// the double range.
template <int RPT, int TJ, bool SQUARE, int CU = 2, bool FACT = false>
__global__ void __launch_bounds__(256) gauss_gemv_dot_kernel(GaussOp op,
                                                             const double* __restrict__ v,
                                                             double* __restrict__ partial,
                                                             int splits,
                                                             const double* __restrict__ geo) {
  constexpr int NT = 256;
  if (!(geo[3] < kDotRange)) return;
  static_assert(!(FACT && SQUARE), "the factored form is for the GEMV");
  constexpr int SQ = FACT ? 4 : 6;   // doubles per tile column
  __shared__ __align__(16) double sq[TJ * SQ];
  const double c0x = geo[0], c0y = geo[1], c0z = geo[2];
  const long long row_base = (long long)blockIdx.x * NT * RPT;
  const long long cols_per = (op.m + splits - 1) / splits;
  const long long j0 = (long long)blockIdx.y * cols_per;
  const long long j1 = min(op.m, j0 + cols_per);
  const ExpTab tl = exp2tab_lane_comp();
  const ExpTab tp = exp2tab_lane();   // plain table for the per-point factors (FACT)
  double px[RPT], py[RPT], pz[RPT], pa[RPT], acc[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    long long i = row_base + threadIdx.x + (long long)r * NT;
    long long ii = i < op.n ? i : 0;
    px[r] = op.c * (op.P[ii * 3 + 0] - c0x);
    py[r] = op.c * (op.P[ii * 3 + 1] - c0y);
    pz[r] = op.c * (op.P[ii * 3 + 2] - c0z);
    const double p2 = fma(pz[r], pz[r], fma(py[r], py[r], px[r] * px[r]));
    pa[r] = FACT ? exp_neg(p2, tp) : -kExpK * p2;   // A_i, or a_i in table units
    acc[r] = 0.0;
  }
  for (long long jt = j0; jt < j1; jt += TJ) {
    const int cnt = (int)min((long long)TJ, j1 - jt);
    __syncthreads();
    // (warp-uniform trip count: the factored form's exp shuffles need every lane)
    for (int cb = 0; cb < TJ; cb += NT) {
      const int cc = cb + (int)threadIdx.x;
      const long long j = min(jt + cc, j1 - 1);
      const double qx = op.c * (op.Q[j * 3 + 0] - c0x);
      const double qy = op.c * (op.Q[j * 3 + 1] - c0y);
      const double qz = op.c * (op.Q[j * 3 + 2] - c0z);
      const double q2 = fma(qz, qz, fma(qy, qy, qx * qx));
      double last;
      if constexpr (FACT) last = exp_neg(q2, tp) * v[j];   // w_j = B_j v_j
      else last = -kExpK * q2;                             // b_j in table units
      if (cc < cnt) {
        sq[cc * SQ + 0] = (2.0 * kExpK) * qx;
        sq[cc * SQ + 1] = (2.0 * kExpK) * qy;
        sq[cc * SQ + 2] = (2.0 * kExpK) * qz;
        sq[cc * SQ + 3] = last;
        if constexpr (!FACT) sq[cc * SQ + 4] = SQUARE ? 1.0 : v[j];
      }
    }
    __syncthreads();
    // CU columns x RPT rows = E independent entries per trip, every stage
    // issued for all E before the next (interleaved dependency chains)
    constexpr int E = CU * RPT;
    int cc = 0;
    for (; cc + CU <= cnt; cc += CU) {
      double y[E], e[E], vj[CU];
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const double qz = sq[(cc + u) * SQ + 2], qb = sq[(cc + u) * SQ + 3];
#pragma unroll
        for (int r = 0; r < RPT; ++r) y[u * RPT + r] = FACT ? pz[r] * qz : fma(pz[r], qz, qb);
        if constexpr (FACT) vj[u] = qb;   // the column weight w_j
      }
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const double qy = sq[(cc + u) * SQ + 1];
#pragma unroll
        for (int r = 0; r < RPT; ++r) y[u * RPT + r] = fma(py[r], qy, y[u * RPT + r]);
      }
#pragma unroll
      for (int u = 0; u < CU; ++u) {
        const double qx = sq[(cc + u) * SQ + 0];
        if constexpr (!FACT) vj[u] = sq[(cc + u) * SQ + 4];
#pragma unroll
        for (int r = 0; r < RPT; ++r) y[u * RPT + r] = fma(px[r], qx, y[u * RPT + r]);
      }
      if constexpr (!FACT) {
#pragma unroll
        for (int u = 0; u < CU; ++u)
#pragma unroll
          for (int r = 0; r < RPT; ++r) y[u * RPT + r] += pa[r];
      }
      exp_tab_units_v<E>(y, e, tl);
#pragma unroll
      for (int u = 0; u < CU; ++u)
#pragma unroll
        for (int r = 0; r < RPT; ++r)
          acc[r] = SQUARE ? fma(e[u * RPT + r], e[u * RPT + r], acc[r])
                          : fma(e[u * RPT + r], vj[u], acc[r]);
    }
    for (; cc < cnt; ++cc) {   // tile tail (cnt % CU columns)
      const double qx = sq[cc * SQ + 0], qy = sq[cc * SQ + 1], qz = sq[cc * SQ + 2];
      const double qb = sq[cc * SQ + 3], vj = FACT ? qb : sq[cc * SQ + (FACT ? 3 : 4)];
      double y[RPT], e[RPT];
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        y[r] = FACT ? fma(px[r], qx, fma(py[r], qy, pz[r] * qz))
                    : fma(px[r], qx, fma(py[r], qy, fma(pz[r], qz, qb))) + pa[r];
      exp_tab_units_v<RPT>(y, e, tl);
#pragma unroll
      for (int r = 0; r < RPT; ++r) acc[r] = SQUARE ? fma(e[r], e[r], acc[r]) : fma(e[r], vj, acc[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    long long i = row_base + threadIdx.x + (long long)r * NT;
    if (i < op.n) partial[(long long)blockIdx.y * op.n + i] = FACT ? acc[r] * pa[r] : acc[r];
  }
}

template <int RPT, int TJ, bool SQUARE>
__global__ void __launch_bounds__(256) gauss_gemv_kernel(GaussOp op, const double* __restrict__ v,
                                                         double* __restrict__ partial, int splits,
                                                         const double* __restrict__ geo) {
  constexpr int NT = 256;
  if (geo[3] < kDotRange) return;   // the dot-product form below runs instead
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

// RPLU_GEMV_CU: columns per interleaved group of the dot kernel (1, 2 or 4)
static int gemv_cu() {
  static const int cu = [] {
    const char* e = getenv("RPLU_GEMV_CU");
    const int c = e ? atoi(e) : 4;   // measured at 1e6: 1 -> 1099 ms, 2 -> 1049, 4 -> 1021
    return (c == 1 || c == 2) ? c : 4;
  }();
  return cu;
}

template <int RPT>
static void gemv_launch(const GaussOp& op, const double* v, double* part, int splits, bool square,
                        const double* geo, cudaStream_t s) {
  constexpr int TJ = 256;
  dim3 grid((unsigned)((op.n + 256 * RPT - 1) / (256 * RPT)), (unsigned)splits);
  const int cu = gemv_cu();
  if (square) {
    if (cu == 1) gauss_gemv_dot_kernel<RPT, TJ, true, 1><<<grid, 256, 0, s>>>(op, v, part, splits, geo);
    else if (cu == 2) gauss_gemv_dot_kernel<RPT, TJ, true, 2><<<grid, 256, 0, s>>>(op, v, part, splits, geo);
    else gauss_gemv_dot_kernel<RPT, TJ, true, 4><<<grid, 256, 0, s>>>(op, v, part, splits, geo);
    gauss_gemv_kernel<RPT, TJ, true><<<grid, 256, 0, s>>>(op, v, part, splits, geo);
  } else {
    static const bool fact = [] {   // RPLU_GEMV_FACT=0: unfactored exponent (14 FP64 per entry)
      const char* e = getenv("RPLU_GEMV_FACT");
      return !(e && atoi(e) == 0);
    }();
    if (fact) {
      if (cu == 1) gauss_gemv_dot_kernel<RPT, TJ, false, 1, true><<<grid, 256, 0, s>>>(op, v, part, splits, geo);
      else if (cu == 2) gauss_gemv_dot_kernel<RPT, TJ, false, 2, true><<<grid, 256, 0, s>>>(op, v, part, splits, geo);
      else gauss_gemv_dot_kernel<RPT, TJ, false, 4, true><<<grid, 256, 0, s>>>(op, v, part, splits, geo);
    } else {
      if (cu == 1) gauss_gemv_dot_kernel<RPT, TJ, false, 1><<<grid, 256, 0, s>>>(op, v, part, splits, geo);
      else if (cu == 2) gauss_gemv_dot_kernel<RPT, TJ, false, 2><<<grid, 256, 0, s>>>(op, v, part, splits, geo);
      else gauss_gemv_dot_kernel<RPT, TJ, false, 4><<<grid, 256, 0, s>>>(op, v, part, splits, geo);
    }
    gauss_gemv_kernel<RPT, TJ, false><<<grid, 256, 0, s>>>(op, v, part, splits, geo);
  }
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

// RPLU_GEMV_DOT=0 forces the difference form (experiment / comparison knob)
static bool gemv_dot_enabled() {
  static bool v = [] {
    const char* e = getenv("RPLU_GEMV_DOT");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

__global__ void gauss_geo_off_kernel(double* geo) {
  if (threadIdx.x == 0) geo[3] = __longlong_as_double(0x7ff0000000000000LL);
}

int gauss_gemv_impl(rplu_ctx* ctx, const GaussOp& op, const double* v, double* out, bool square,
                    cudaStream_t s, float* ms) {
  const int rpt = gemv_rpt();
  // resident CTAs per SM of the kernel that normally runs (the dot-product
  // form; the split count balances its last wave)
  static int per_sm[3] = {0, 0, 0};
  const int slot = rpt == 1 ? 0 : (rpt == 2 ? 1 : 2);
  if (!per_sm[slot]) {
    int b = 0;
    const bool dot = gemv_dot_enabled();
    const int cu = gemv_cu();
#define RPLU_OCC(R)                                                                              \
  (dot ? (cu == 1 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(                               \
                        &b, gauss_gemv_dot_kernel<R, 256, false, 1>, 256, 0)                     \
                  : cu == 2 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(                     \
                                  &b, gauss_gemv_dot_kernel<R, 256, false, 2>, 256, 0)           \
                            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(                     \
                                  &b, gauss_gemv_dot_kernel<R, 256, false, 4>, 256, 0))          \
       : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, gauss_gemv_kernel<R, 256, false>,     \
                                                       256, 0))
    if (rpt == 1) RPLU_OCC(1);
    else if (rpt == 2) RPLU_OCC(2);
    else RPLU_OCC(4);
#undef RPLU_OCC
    per_sm[slot] = b > 0 ? b : 1;
  }
  const int splits = gemv_splits(op.n, op.m, 256 * rpt, ctx->sm_count, per_sm[slot]);
  int rc;
  // scratch: [bounding-box partials | geo | split partials]
  const int nbox = (int)std::min<long long>((std::max(op.n, op.m) + 255) / 256, ctx->sm_count);
  constexpr size_t kGeoDoubles = 4096;   // >= 12 * SMs + 4
  if ((rc = ctx->scratch[4].ensure(sizeof(double) * (kGeoDoubles + (size_t)splits * op.n))))
    return rc;
  double* boxes = reinterpret_cast<double*>(ctx->scratch[4].ptr);
  double* geo = boxes + kGeoDoubles - 8;
  double* part = boxes + kGeoDoubles;
  count_launches(2);
  if (gemv_dot_enabled()) {
    gauss_bbox_kernel<<<nbox, 256, 0, s>>>(op, boxes);
    gauss_geo_kernel<<<1, 32, 0, s>>>(boxes, nbox, op.c, geo);
  } else {
    gauss_geo_off_kernel<<<1, 32, 0, s>>>(geo);
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ms) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  count_launches(2);
  if (rpt == 1) gemv_launch<1>(op, v, part, splits, square, geo, s);
  else if (rpt == 2) gemv_launch<2>(op, v, part, splits, square, geo, s);
  else gemv_launch<4>(op, v, part, splits, square, geo, s);
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
