// Cauchy-like structured RPLU (Alg 3, exact row norms) — K5 generated-entry
// row masses, K6 pivot row / column generation and generator update.
//
// Reference: rplu.cauchy.structured_eliminate, plan=None branch
// (pkg/src/rplu/cauchy.py:177-256):
//   u = exact_row_norms(cur) (:209-210, :129-137), bound_maxes/sums (:211-214),
//   degenerate / tol stops (:217-222), i = sample_index(u, u1) (:228),
//   r = row(i) (:82-83), j = sample_index(|r|^2, u2) (:236), relative zero-pivot
//   guard with one resample (:237-245), c = column(j) (:85-86),
//   G -= outer(c/a, G_i), B -= outer(B_:,j, r/a) (:247-250).
//
// Device layout (complex128 = double2): x[n], y[m]; G row-major n x P (the
// reference's C-order G); Bt row-major m x P, i.e. column j of B contiguous
// (the reference's F-order B).  No matrix is ever stored: K5 regenerates
// every entry (G_i . B_j) / (x_i - y_j) from registers (row side) and a shared
// memory tile of (y_j, B_j) (column side), so a step is FP64-pipe bound.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <string.h>

#include <algorithm>
#include <vector>

#include "rplu_common.cuh"
#include "rplu_internal.h"

namespace rplu {

constexpr double kPivotRelTol = 1e-14;  // cauchy.py:33

struct CauchyParams {
  long long n, m, rank;
  int p;
  const double2* x;
  const double2* y;
  double2* G;
  double2* Bt;
  double* partial;   // [splits][n] partial row masses
  double* masses;    // n row masses (== partial when splits == 1)
  int splits;
  double2* rbuf;     // row r of the current step (m)
  double* wbuf;      // |r|^2 (m)
  double2* Cout;     // keep_steps: rank x n (or null)
  double2* Rout;     // keep_steps: rank x m (or null)
  double2* Aout;     // keep_steps: rank (or null)
  DevState* st;
  long long t;
  const double* uniforms;
  long long n_uniforms;
  long long* rows;
  long long* cols;
  double* bmax;
  double* bsum;
  double stop_tol;
  int rule;
  // sharded path: the pivot message [(i_global, 0), x_i, G_i[0..P)] the row
  // and snapshot kernels read instead of G / x (null on one GPU)
  const double2* psrc;
  // per-row-block arrival counters: the last split CTA of a row block sums
  // the split partials into masses (fixed split order) -- no separate launch
  unsigned* blk_count;
  // max_j |r_j| of the step's pivot row as the bits of a non-negative double
  // (atomicMax in the row kernel; read and cleared by the column select)
  unsigned long long* rmax_bits;
  double2* gsnap;    // G_i, B_j before the update (written by the column select)
};

// ---------------------------------------------------------------------------
// K5: partial[s][i] = sum_{j in split s} |G_i . B_j|^2 / |x_i - y_j|^2
template <int P, int RPT, int TJ, int NT>
__global__ void __launch_bounds__(NT) cauchy_mass_kernel(CauchyParams q) {
  if (q.st && !q.st->active) return;
  __shared__ double2 sy[TJ];
  __shared__ double2 sb[TJ * P];
  const long long row_base = (long long)blockIdx.x * NT * RPT;
  // this CTA's column range
  const long long cols_per = (q.m + q.splits - 1) / q.splits;
  const long long j0 = (long long)blockIdx.y * cols_per;
  const long long j1 = min(q.m, j0 + cols_per);

  double2 g[RPT][P];
  double2 xr[RPT];
  double acc[RPT];
  bool valid[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    long long i = row_base + threadIdx.x + (long long)r * NT;
    valid[r] = i < q.n;
    long long ii = valid[r] ? i : 0;
    xr[r] = q.x[ii];
#pragma unroll
    for (int l = 0; l < P; ++l) g[r][l] = q.G[ii * P + l];
    acc[r] = 0.0;
  }
  for (long long jt = j0; jt < j1; jt += TJ) {
    const int cnt = (int)min((long long)TJ, j1 - jt);
    __syncthreads();
    for (int c = threadIdx.x; c < TJ; c += NT) {
      if (c < cnt) {
        sy[c] = q.y[jt + c];
        if constexpr (P == 1) {
          const double2 bj = q.Bt[jt + c];
          sb[c] = make_double2(fma(bj.x, bj.x, bj.y * bj.y), 0.0);
        } else {
#pragma unroll
          for (int l = 0; l < P; ++l) sb[c * P + l] = q.Bt[(jt + c) * P + l];
        }
      }
    }
    __syncthreads();
#pragma unroll 2
    for (int c = 0; c < cnt; ++c) {
      const double2 yj = sy[c];
      double2 b[P];
#pragma unroll
      for (int l = 0; l < P; ++l) b[l] = sb[c * P + l];
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const double dr = xr[r].x - yj.x, di = xr[r].y - yj.y;
        const double den = fma(dr, dr, di * di);
        if constexpr (P == 1) {
          // displacement rank 1: |g_i b_j|^2 = |g_i|^2 |b_j|^2, so the
          // column weight |b_j|^2 (staged in sb[c].x) is accumulated here
          // and |g_i|^2 applied once per row: 9 FP64 ops per entry, not 15
          acc[r] = fma(b[0].x, rcp_nr(den), acc[r]);
        } else {
          double re = 0.0, im = 0.0;
#pragma unroll
          for (int l = 0; l < P; ++l) {
            re = fma(g[r][l].x, b[l].x, re);
            re = fma(-g[r][l].y, b[l].y, re);
            im = fma(g[r][l].x, b[l].y, im);
            im = fma(g[r][l].y, b[l].x, im);
          }
          const double num = fma(re, re, im * im);
          acc[r] = fma(num, rcp_nr(den), acc[r]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    long long i = row_base + threadIdx.x + (long long)r * NT;
    if constexpr (P == 1) acc[r] *= fma(g[r][0].x, g[r][0].x, g[r][0].y * g[r][0].y);
    if (valid[r]) q.partial[(long long)blockIdx.y * q.n + i] = acc[r];
  }
  if (q.splits > 1 && q.blk_count) {
    // the last of the row block's split CTAs to finish forms the masses
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0)
      s_last = atomicAdd(&q.blk_count[blockIdx.x], 1u) == (unsigned)(q.splits - 1);
    __syncthreads();
    if (s_last) {
      __threadfence();
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const long long i = row_base + threadIdx.x + (long long)r * NT;
        if (valid[r]) {
          double sv = 0.0;
          for (int k = 0; k < q.splits; ++k) sv += __ldcg(q.partial + (long long)k * q.n + i);
          q.masses[i] = sv;
        }
      }
      if (threadIdx.x == 0) q.blk_count[blockIdx.x] = 0u;
    }
  }
}

// Sum the split partials into masses (used by exact_row_norms).
__global__ void sum_partials_kernel(const double* partial, int splits, long long n, double* out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int k = 0; k < splits; ++k) s += partial[(long long)k * n + i];
  out[i] = s;
}

// ---------------------------------------------------------------------------
// K2a: row selection + stop rules (block-uniform result: the row, or -1
// when the loop stops here).
__device__ __forceinline__ long long cauchy_select_row_dev(const CauchyParams& q) {
  constexpr int B = 1024;
  DevState* st = q.st;
  __shared__ CdfSmem<B> sm;
  __shared__ int s_stop;
  __shared__ double s_max[B / 32];
  const long long n = q.n, t = q.t;
  const double* masses = q.masses;
  auto wrow = [&](long long k) { return masses[k]; };
  Cdf<B> cr = cdf_build<B>(wrow, n, sm);
  // umax over rows
  double mx = 0.0;
  for (long long k = threadIdx.x; k < n; k += B) mx = fmax(mx, wrow(k));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double umax = 0.0;
    for (int w = 0; w < B / 32; ++w) umax = fmax(umax, s_max[w]);
    q.bmax[t] = umax;
    q.bsum[t] = cr.total;
    if (t == 0) st->fro0 = umax;
    const double u0 = (t == 0) ? umax : st->fro0;
    int stop = 0;
    if (umax <= 0.0) {
      st->status = kDegenerate;
      stop = 1;
    } else if (q.stop_tol > 0.0 && umax <= q.stop_tol * q.stop_tol * u0) {
      st->status = kTolStop;
      stop = 1;
    }
    if (stop) st->active = 0;
    s_stop = stop;
  }
  __syncthreads();
  if (s_stop) return -1;
  long long i;
  long long uc = st->ucount;
  if (q.rule == RPLU_RULE_RPLU) {
    if (uc + 1 > q.n_uniforms) {
      if (threadIdx.x == 0) { st->status = kUniformsExhausted; st->active = 0; }
      return -1;
    }
    const double u1 = q.uniforms[uc];
    i = cdf_find<B>(wrow, n, cr, u1, sm);
    if (threadIdx.x == 0) {
      const double tol = kNearBoundaryRel * cr.total, tg = u1 * cr.total;
      if (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) st->near_boundary++;
      st->ucount = uc + 1;
    }
  } else {
    i = block_argmax<B>(wrow, n, nullptr);
  }
  if (threadIdx.x == 0) st->pi = i;
  return i;
}

__global__ void __launch_bounds__(1024) cauchy_select_row_kernel(CauchyParams q) {
  if (!q.st->active) return;
  cauchy_select_row_dev(q);
}

// ---------------------------------------------------------------------------
// K6a: pivot row r_j = (G_i . B_j) / (x_i - y_j) for all j, weights |r_j|^2.
// numpy order: matmul then complex division (Smith).
template <int P>
__device__ __forceinline__ void cauchy_row_dev(const CauchyParams& q, long long j0, long long js) {
  double2 gi[P];
  double2 xi;
  if (q.psrc) {
#pragma unroll
    for (int l = 0; l < P; ++l) gi[l] = q.psrc[2 + l];
    xi = q.psrc[1];
    if (blockIdx.x == 0 && threadIdx.x == 0) q.st->pi = (long long)q.psrc[0].x;
  } else {
    const long long i = q.st->pi;
#pragma unroll
    for (int l = 0; l < P; ++l) gi[l] = q.G[i * P + l];
    xi = q.x[i];
  }
  double amax = 0.0;
  for (long long j = j0; j < q.m; j += js) {
    double re = 0.0, im = 0.0;
#pragma unroll
    for (int l = 0; l < P; ++l) {
      const double2 b = q.Bt[j * P + l];
      re = fma(gi[l].x, b.x, fma(-gi[l].y, b.y, re));
      im = fma(gi[l].x, b.y, fma(gi[l].y, b.x, im));
    }
    const double2 yj = q.y[j];
    const double2 d = make_double2(xi.x - yj.x, xi.y - yj.y);
    const double2 r = cdiv_np(make_double2(re, im), d);
    q.rbuf[j] = r;
    const double a = cabs_np(r);
    q.wbuf[j] = a * a;
    amax = fmax(amax, a);
  }
  if (q.rmax_bits) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0 && amax > 0.0)
      atomicMax(q.rmax_bits, (unsigned long long)__double_as_longlong(amax));
  }
}

template <int P>
__global__ void cauchy_row_kernel(CauchyParams q) {
  if (!q.st->active) return;
  cauchy_row_dev<P>(q, (long long)blockIdx.x * blockDim.x + threadIdx.x,
                    (long long)gridDim.x * blockDim.x);
}

// ---------------------------------------------------------------------------
// K2b: column selection with the relative zero-pivot guard; captures G_i and
// B_j (pre-update) and 1/a coefficients into the state for the update.
__device__ __forceinline__ void cauchy_select_col_dev(const CauchyParams& q) {
  constexpr int B = 1024;
  DevState* st = q.st;
  __shared__ CdfSmem<B> sm;
  __shared__ double s_max[B / 32];
  const long long m = q.m, t = q.t;
  const double* w = q.wbuf;
  auto wcol = [&](long long k) { return w[k]; };
  auto wabs = [&](long long k) { return cabs_np(q.rbuf[k]); };
  // max |r| for the relative threshold (from the row kernel's atomic max,
  // else scanned here)
  double rmax = 0.0;
  if (q.rmax_bits) {
    rmax = __longlong_as_double((long long)__ldcg(q.rmax_bits));
  } else {
    double mx = 0.0;
    for (long long k = threadIdx.x; k < m; k += B) mx = fmax(mx, wabs(k));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mx;
    __syncthreads();
    for (int k = 0; k < B / 32; ++k) rmax = fmax(rmax, s_max[k]);
  }
  const double thr = kPivotRelTol * rmax;
  long long j;
  long long uc = st->ucount;
  long long near = 0;
  if (q.rule == RPLU_RULE_RPLU) {
    Cdf<B> cc = cdf_build<B>(wcol, m, sm);
    int attempt = 0;
    for (;;) {
      if (uc + 1 > q.n_uniforms) {
        if (threadIdx.x == 0) { st->status = kUniformsExhausted; st->active = 0; }
        return;
      }
      const double u2 = q.uniforms[uc];
      uc += 1;
      j = cdf_find<B>(wcol, m, cc, u2, sm);
      if (threadIdx.x == 0) {
        const double tol = kNearBoundaryRel * cc.total, tg = u2 * cc.total;
        if (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) near++;
      }
      __syncthreads();
      if (wabs(j) > thr) break;
      if (attempt++ == 1) {
        if (threadIdx.x == 0) {
          st->status = kZeroPivot;
          st->active = 0;
          st->err_i = st->pi;
          st->err_j = j;
          st->ucount = uc;
          st->near_boundary += near;
        }
        return;
      }
    }
  } else {
    j = block_argmax<B>(wabs, m, nullptr);
    if (!(wabs(j) > thr)) {
      if (threadIdx.x == 0) {
        st->status = kZeroPivot;
        st->active = 0;
        st->err_i = st->pi;
        st->err_j = j;
      }
      return;
    }
  }
  if (threadIdx.x == 0) {
    const long long i = st->pi;
    const double2 a = q.rbuf[j];
    st->pj = j;
    st->ucount = uc;
    st->near_boundary += near;
    st->a_re = a.x;
    st->a_im = a.y;
    const CDivCoef cf = cdiv_coef(a);
    st->rat = cf.rat;
    st->scl = cf.scl;
    st->branch = cf.branch;
    // pre-update generator row G_i and column B_j (P <= 8 -> 16 doubles in aux)
    // are captured by the update kernel itself from its own registers; record
    // the step here.
    q.rows[t] = i;
    q.cols[t] = j;
    if (q.Aout) q.Aout[t] = a;
    st->done = t + 1;
    if (q.rmax_bits) *q.rmax_bits = 0ull;  // for the next step's row kernel
  }
  if (q.gsnap && threadIdx.x < q.p) {  // G_i and B_j before the update
    const int l = threadIdx.x;
    q.gsnap[l] = q.psrc ? q.psrc[2 + l] : q.G[st->pi * q.p + l];
    q.gsnap[q.p + l] = q.Bt[j * q.p + l];
  }
}

__global__ void __launch_bounds__(1024) cauchy_select_col_kernel(CauchyParams q) {
  if (!q.st->active) return;
  cauchy_select_col_dev(q);
}

// K2a + K6a + K2b in one CTA (single-GPU loop): the row draw, the pivot row
// generated by the same 1024 threads (m entries, O(mp) work: microseconds even
// at m = 2^20 against a multi-second step at that size), and the column draw
// -- two launches and two L2 round trips fewer per step than the separate
// kernels the sharded path uses.
template <int P>
__global__ void __launch_bounds__(1024) cauchy_select_kernel(CauchyParams q) {
  if (!q.st->active) return;
  if (cauchy_select_row_dev(q) < 0) return;
  __syncthreads();  // st->pi written by thread 0
  cauchy_row_dev<P>(q, threadIdx.x, blockDim.x);
  __syncthreads();  // r, |r|^2 and the row max are in place
  cauchy_select_col_dev(q);
}

// ---------------------------------------------------------------------------
// K6b: c_k = (G_k . B_j)/(x_k - y_j); G_k -= (c_k/a) G_i  (k < n)
//      B_l -= B_j (r_l/a)                                 (l < m)
// G_i and B_j are read from a snapshot taken before any CTA writes (gsnap).
template <int P>
__global__ void cauchy_update_kernel(CauchyParams q, const double2* __restrict__ gsnap) {
  if (!q.st->active) return;
  const long long j = q.st->pj;
  CDivCoef cf;
  cf.rat = q.st->rat;
  cf.scl = q.st->scl;
  cf.branch = q.st->branch;
  double2 gi[P], bj[P];
#pragma unroll
  for (int l = 0; l < P; ++l) {
    gi[l] = gsnap[l];
    bj[l] = gsnap[P + l];
  }
  const double2 yj = q.y[j];
  const long long total = q.n + q.m;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (long long)gridDim.x * blockDim.x) {
    if (k < q.n) {
      double2 g[P];
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int l = 0; l < P; ++l) {
        g[l] = q.G[k * P + l];
        re = fma(g[l].x, bj[l].x, fma(-g[l].y, bj[l].y, re));
        im = fma(g[l].x, bj[l].y, fma(g[l].y, bj[l].x, im));
      }
      const double2 xk = q.x[k];
      const double2 c = cdiv_np(make_double2(re, im), make_double2(xk.x - yj.x, xk.y - yj.y));
      if (q.Cout) q.Cout[q.t * q.n + k] = c;
      const double2 ca = cdiv_apply(c, cf);
#pragma unroll
      for (int l = 0; l < P; ++l) {
        const double2 pr = cmul_np(ca, gi[l]);
        q.G[k * P + l] = make_double2(__dsub_rn(g[l].x, pr.x), __dsub_rn(g[l].y, pr.y));
      }
    } else {
      const long long l2 = k - q.n;
      const double2 r = q.rbuf[l2];
      if (q.Rout) q.Rout[q.t * q.m + l2] = r;
      const double2 ra = cdiv_apply(r, cf);
#pragma unroll
      for (int l = 0; l < P; ++l) {
        const double2 b = q.Bt[l2 * P + l];
        const double2 pr = cmul_np(bj[l], ra);
        q.Bt[l2 * P + l] = make_double2(__dsub_rn(b.x, pr.x), __dsub_rn(b.y, pr.y));
      }
    }
  }
}

// snapshot G_i and B_j (2P complex) before the update kernel overwrites them
__global__ void cauchy_snapshot_kernel(CauchyParams q, double2* gsnap) {
  if (!q.st->active) return;
  const int l = threadIdx.x;
  if (l < q.p) {
    gsnap[l] = q.psrc ? q.psrc[2 + l] : q.G[q.st->pi * q.p + l];
    gsnap[q.p + l] = q.Bt[q.st->pj * q.p + l];
  }
}

// ---------------------------------------------------------------------------
// launch helpers

static int choose_splits(long long n, long long m, int rows_per_cta, int sm_count) {
  // latency-bound sizes: about two CTAs per SM (a whole number of CTAs per
  // SM, so no SM runs a lone extra CTA), each with >= 64 columns
  static const int per_sm = [] {  // RPLU_CAUCHY_CTAS_PER_SM experiment override
    const char* e = getenv("RPLU_CAUCHY_CTAS_PER_SM");
    const int v = e ? atoi(e) : 2;
    return v >= 1 && v <= 8 ? v : 2;
  }();
  static const int min_cols = [] {
    const char* e = getenv("RPLU_CAUCHY_MIN_COLS");
    const int v = e ? atoi(e) : 64;
    return v >= 8 && v <= 4096 ? v : 64;
  }();
  long long row_blocks = (n + rows_per_cta - 1) / rows_per_cta;
  long long want = (long long)per_sm * sm_count;
  long long s = (want + row_blocks - 1) / row_blocks;
  long long max_s = (m + min_cols - 1) / min_cols;
  if (s > max_s) s = max_s;
  if (s < 1) s = 1;
  if (s > 1024) s = 1024;
  return (int)s;
}

// K5 CTA shape: rows_per_cta(p) rows per CTA either as 256 threads x 2 rows
// (ILP: compute-bound sizes, C4 1956 ms vs 2022 ms) or 512 threads x 1 row
// (TLP: latency-bound sizes, C2 22.4 us vs 26.0 us per launch).  The per-row
// summation order is the same in both (bit-identical masses).
// RPLU_CAUCHY_MASS_TLP=0/1 forces either.
static bool mass_tlp(long long n, long long m) {
  static const int v = [] {
    const char* e = getenv("RPLU_CAUCHY_MASS_TLP");
    return e ? atoi(e) : -1;
  }();
  if (v == 0 || v == 1) return v == 1;
  return (double)n * (double)m <= 268435456.0;  // 2^28 entries
}

// threads (= rows) per CTA of the TLP shape (RPLU_CAUCHY_TLP_NT: 512 / 768 / 1024)
static int tlp_nt() {
  static const int v = [] {
    const char* e = getenv("RPLU_CAUCHY_TLP_NT");
    const int x = e ? atoi(e) : 512;
    return (x == 768 || x == 1024) ? x : 512;
  }();
  return v;
}

template <int P>
static void launch_mass(CauchyParams& q, cudaStream_t s) {
  constexpr int TJ = 128;
  if (P <= 4 && mass_tlp(q.n, q.m)) {
    const int nt = tlp_nt();
    dim3 grid((unsigned)((q.n + nt - 1) / nt), (unsigned)q.splits);
    if (nt == 1024) cauchy_mass_kernel<P, 1, TJ, 1024><<<grid, 1024, 0, s>>>(q);
    else if (nt == 768) cauchy_mass_kernel<P, 1, TJ, 768><<<grid, 768, 0, s>>>(q);
    else cauchy_mass_kernel<P, 1, TJ, 512><<<grid, 512, 0, s>>>(q);
    return;
  }
  constexpr int RPT = (P <= 4) ? 2 : 1;
  dim3 grid((unsigned)((q.n + 256 * RPT - 1) / (256 * RPT)), (unsigned)q.splits);
  cauchy_mass_kernel<P, RPT, TJ, 256><<<grid, 256, 0, s>>>(q);
}

#define RPLU_P_SWITCH(p, CALL)      \
  switch (p) {                      \
    case 1: { constexpr int PP = 1; CALL; } break; \
    case 2: { constexpr int PP = 2; CALL; } break; \
    case 3: { constexpr int PP = 3; CALL; } break; \
    case 4: { constexpr int PP = 4; CALL; } break; \
    case 5: { constexpr int PP = 5; CALL; } break; \
    case 6: { constexpr int PP = 6; CALL; } break; \
    case 7: { constexpr int PP = 7; CALL; } break; \
    case 8: { constexpr int PP = 8; CALL; } break; \
    default: break;                 \
  }

static int rows_per_cta(int p, long long n, long long m) {
  if (p <= 4 && mass_tlp(n, m)) return tlp_nt();
  return 256 * ((p <= 4) ? 2 : 1);
}

// ---------------------------------------------------------------------------
// Plan-path step primitives (structured_eliminate with certified bounds,
// cauchy.py:207-277): the proposal's pivot row and the generator update run
// in the exact-norm loop's K6 kernels (numpy-exact Smith division and
// complex products), driven by the host rejection loop.

// st <- (pi, pj, Smith coefficients of a = r_j), snapshot G_i, B_j
__global__ void cauchy_plan_pivot_kernel(CauchyParams q, long long i, long long j,
                                         double2* gsnap) {
  DevState* st = q.st;
  if (threadIdx.x == 0) {
    st->active = 1;
    st->status = kRunning;
    st->pi = i;
    st->pj = j;
    const double2 a = q.rbuf[j];
    st->a_re = a.x;
    st->a_im = a.y;
    const CDivCoef cf = cdiv_coef(a);
    st->rat = cf.rat;
    st->scl = cf.scl;
    st->branch = cf.branch;
  }
  const int l = threadIdx.x;
  if (l < q.p) {
    gsnap[l] = q.G[i * q.p + l];
    gsnap[q.p + l] = q.Bt[j * q.p + l];
  }
}

__global__ void cauchy_plan_init_kernel(DevState* st, long long i, unsigned long long* rmax_bits) {
  st->active = 1;
  st->status = kRunning;
  st->pi = i;
  *rmax_bits = 0ull;
}

static int plan_params(rplu_ctx* ctx, int p, long long n, long long m, const void* x,
                       const void* y, void* G, void* Bt, void* rbuf, double* wbuf,
                       CauchyParams& q, double2*& gsnap) {
  q = CauchyParams{};
  q.n = n;
  q.m = m;
  q.p = p;
  q.x = reinterpret_cast<const double2*>(x);
  q.y = reinterpret_cast<const double2*>(y);
  q.G = reinterpret_cast<double2*>(G);
  q.Bt = reinterpret_cast<double2*>(Bt);
  q.rbuf = reinterpret_cast<double2*>(rbuf);
  q.wbuf = wbuf;
  int rc;
  if ((rc = ctx->state.ensure(sizeof(DevState)))) return rc;
  q.st = reinterpret_cast<DevState*>(ctx->state.ptr);
  // layout: [0,8) row-max bits | [16, 16 + 32 p) G_i / B_j snapshot | [512, 544) read-back slots
  if ((rc = ctx->csync.ensure(1024))) return rc;
  q.rmax_bits = reinterpret_cast<unsigned long long*>(ctx->csync.ptr);
  gsnap = reinterpret_cast<double2*>(reinterpret_cast<char*>(ctx->csync.ptr) + 16);
  return RPLU_OK;
}

int cauchy_plan_row_impl(rplu_ctx* ctx, int p, long long n, long long m, const void* x,
                         const void* y, void* G, void* Bt, long long i, void* rbuf, double* wbuf,
                         const double* bounds, double* host3, cudaStream_t s) {
  CauchyParams q;
  double2* gsnap;
  int rc;
  if ((rc = plan_params(ctx, p, n, m, x, y, G, Bt, rbuf, wbuf, q, gsnap))) return rc;
  cauchy_plan_init_kernel<<<1, 1, 0, s>>>(q.st, i, q.rmax_bits);
  const int row_blocks = (int)std::min<long long>((m + 255) / 256, 8LL * ctx->sm_count);
  count_launches(2);
  RPLU_P_SWITCH(p, (cauchy_row_kernel<PP><<<row_blocks, 256, 0, s>>>(q)));
  RPLU_CUDA(cudaGetLastError());
  unsigned long long rbits = 0;
  double bi = 0.0;
  RPLU_CUDA(cudaMemcpyAsync(&rbits, q.rmax_bits, sizeof(rbits), cudaMemcpyDeviceToHost, s));
  if (bounds) RPLU_CUDA(cudaMemcpyAsync(&bi, bounds + i, sizeof(double), cudaMemcpyDeviceToHost, s));
  double rho = 0.0;  // sum of |r_j|^2 in the draw code's (deterministic) order
  if ((rc = sample_index_impl(ctx, wbuf, m, 0.0, 2, nullptr, nullptr, &rho, s))) return rc;
  host3[0] = rho;
  double rmax = 0.0;
  memcpy(&rmax, &rbits, sizeof(rmax));
  host3[1] = rmax;
  host3[2] = bi;
  return RPLU_OK;
}

// the proposal's row index from a device-side draw (first 8 bytes of its
// SampleOut): st->pi <- idx, *bi <- bounds[idx], row-max slot cleared
__global__ void cauchy_plan_init_dev_kernel(DevState* st, const long long* didx, long long n,
                                            const double* bounds, double* bi,
                                            unsigned long long* rmax_bits) {
  long long i = *didx;
  if (i < 0 || i >= n) i = 0;   // a failed draw: the host raises after the read-back
  st->active = 1;
  st->status = kRunning;
  st->pi = i;
  *bi = bounds[i];
  *rmax_bits = 0ull;
}

// Proposal of the plan path in ONE host synchronisation: i ~ bounds (uniform
// u), pivot row i into rbuf / wbuf, host5 = {i, near-boundary flag, sum |r|^2,
// max |r|, bounds[i]} (sample_index + rplu_cauchy_plan_row took two).
int cauchy_plan_propose_impl(rplu_ctx* ctx, int p, long long n, long long m, const void* x,
                             const void* y, void* G, void* Bt, const double* bounds, double u,
                             void* rbuf, double* wbuf, double* host5, cudaStream_t s) {
  CauchyParams q;
  double2* gsnap;
  int rc;
  if ((rc = plan_params(ctx, p, n, m, x, y, G, Bt, rbuf, wbuf, q, gsnap))) return rc;
  double* bi_slot = reinterpret_cast<double*>(reinterpret_cast<char*>(ctx->csync.ptr) + 528);
  const int row_blocks = (int)std::min<long long>((m + 255) / 256, 8LL * ctx->sm_count);
  const void* d0 = nullptr;
  const void* d1 = nullptr;
  auto after_draw = [&](const void* d) -> int {
    count_launches(2);
    cauchy_plan_init_dev_kernel<<<1, 1, 0, s>>>(q.st, reinterpret_cast<const long long*>(d), n,
                                                bounds, bi_slot, q.rmax_bits);
    RPLU_P_SWITCH(p, (cauchy_row_kernel<PP><<<row_blocks, 256, 0, s>>>(q)));
    RPLU_CUDA(cudaGetLastError());
    return RPLU_OK;
  };
  if ((rc = sample_two_launch(ctx, bounds, n, u, after_draw, wbuf, m, s, &d0, &d1))) return rc;
  unsigned char h0[kSampleOutBytes], h1[kSampleOutBytes];
  unsigned long long rbits = 0;
  double bi = 0.0;
  RPLU_CUDA(cudaMemcpyAsync(h0, d0, kSampleOutBytes, cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaMemcpyAsync(h1, d1, kSampleOutBytes, cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaMemcpyAsync(&rbits, q.rmax_bits, sizeof(rbits), cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaMemcpyAsync(&bi, bi_slot, sizeof(bi), cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaStreamSynchronize(s));
  long long idx = -1;
  int near = 0;
  double rho = 0.0;
  if ((rc = sample_out_unpack(h0, &idx, &near, nullptr))) return rc;   // bad bounds: raises as sample_index does
  if ((rc = sample_out_unpack(h1, nullptr, nullptr, &rho))) {
    // an all-zero row is not an error here: rho = 0 (the caller's acceptance test handles it)
    rho = 0.0;
  }
  double rmax = 0.0;
  memcpy(&rmax, &rbits, sizeof(rmax));
  host5[0] = (double)idx;
  host5[1] = (double)near;
  host5[2] = rho;
  host5[3] = rmax;
  host5[4] = bi;
  return RPLU_OK;
}

int cauchy_plan_update_impl(rplu_ctx* ctx, int p, long long n, long long m, const void* x,
                            const void* y, void* G, void* Bt, long long i, long long j, void* rbuf,
                            void* Cout, void* Rout, cudaStream_t s) {
  CauchyParams q;
  double2* gsnap;
  int rc;
  if ((rc = plan_params(ctx, p, n, m, x, y, G, Bt, rbuf, nullptr, q, gsnap))) return rc;
  q.Cout = reinterpret_cast<double2*>(Cout);
  q.Rout = reinterpret_cast<double2*>(Rout);
  q.t = 0;
  const int upd_blocks = (int)std::min<long long>((n + m + 255) / 256, 8LL * ctx->sm_count);
  count_launches(2);
  cauchy_plan_pivot_kernel<<<1, 32, 0, s>>>(q, i, j, gsnap);
  RPLU_P_SWITCH(p, (cauchy_update_kernel<PP><<<upd_blocks, 256, 0, s>>>(q, gsnap)));
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

int cauchy_norms_impl(rplu_ctx* ctx, int p, long long n, long long m, const void* x, const void* y,
                      const void* G, const void* Bt, double* out, cudaStream_t s) {
  CauchyParams q{};
  q.n = n;
  q.m = m;
  q.p = p;
  q.x = reinterpret_cast<const double2*>(x);
  q.y = reinterpret_cast<const double2*>(y);
  q.G = reinterpret_cast<double2*>(const_cast<void*>(G));
  q.Bt = reinterpret_cast<double2*>(const_cast<void*>(Bt));
  q.splits = choose_splits(n, m, rows_per_cta(p, n, m), ctx->sm_count);
  int rc;
  if ((rc = ctx->scratch[0].ensure(sizeof(double) * (size_t)q.splits * n))) return rc;
  q.partial = reinterpret_cast<double*>(ctx->scratch[0].ptr);
  q.st = nullptr;
  RPLU_P_SWITCH(p, launch_mass<PP>(q, s));
  sum_partials_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(q.partial, q.splits, n, out);
  RPLU_CUDA(cudaGetLastError());
  RPLU_CUDA(cudaStreamSynchronize(s));
  return RPLU_OK;
}

// ---------------------------------------------------------------------------
// Resident Cauchy-like loop for small problems (BASELINE configs[1], C2):
// ONE cooperative launch for the whole pivot loop and ONE grid barrier per
// pivot step (the per-step launches above spend ~41 us per step at C2 on
// three dependent kernels: masses 22, single-CTA select 13, update 4.5).
//
// Every CTA (one per SM, 512 threads) owns a contiguous row block of the
// generators and keeps, for the whole run, in shared memory: its rows of G
// and x, and a full private copy of B (plus |B_j|^2 for displacement rank 1)
// that it updates itself every step.  Per step:
//   1. masses of the CTA's rows from its shared-memory state (4 rows per
//      thread x strided columns, per-row sums in a fixed order) -> global,
//      double-buffered by step parity;
//   2. the grid barrier;
//   3. every CTA makes the SAME draws redundantly from the same data with the
//      same code (stop rules, row CDF over the n masses, the pivot row
//      generated from the global copy of G_i and the CTA's own B, column CDF
//      in shared memory, relative zero-pivot guard with one resample) -- so
//      nothing has to be broadcast and no second barrier is needed;
//   4. every CTA updates its own G rows (and publishes them in the other of
//      two global G buffers for the next steps' pivot-row lookups) and ALL of
//      its private B copy.
// CTA 0 records the outputs.  The arithmetic of every entry, row, column and
// update is the per-step kernels' (numpy Smith division / products); the
// summation order of the masses and the CDF width (512 instead of 1024
// threads) differ, which moves draws only within rounding of a CDF boundary
// (counted as near-boundary draws, as everywhere).
namespace {

constexpr int kResNT = 512;   // threads per CTA
constexpr int kResRPT = 4;    // rows per thread in the mass phase

struct CauchyResArgs {
  CauchyParams q;
  double* mbuf;       // [2][n] row masses (step parity)
  double2* gbuf;      // [n * P] second global copy of G (ping-pong with q.G)
  unsigned* sync;     // grid-barrier counter
  double2* rglob;     // [m] the step's pivot row (each CTA generates a slice)
  double* wglob;      // [m] its weights |r_j|^2
  double* amaxg;      // [ctas] per-CTA max |r_j| of the slice
  int rows_cta;       // rows per CTA (multiple of kResRPT)
  long long* trace;   // optional CTA-0 phase timestamps [1024][8]
};

// dynamic shared memory: B | |B|^2 (P == 1) | weights / mass partials / row
// masses | G rows | x rows | y (when it fits: YS)
__host__ __device__ inline long long cauchy_res_wlen(long long n, long long m, int rows_cta) {
  const int rg = rows_cta / kResRPT, cg = kResNT / (rg > 0 ? rg : 1);
  long long w = (long long)rows_cta * cg;
  if (m > w) w = m;
  if (n > w) w = n;
  return (w + 1) & ~1LL;
}
__host__ __device__ inline size_t cauchy_res_smem(long long n, long long m, int p, int rows_cta,
                                                  bool ys) {
  const long long me = (m + 1) & ~1LL;
  return (size_t)m * p * 16 + (p == 1 ? (size_t)me * 8 : 0) +
         (size_t)cauchy_res_wlen(n, m, rows_cta) * 8 + (size_t)rows_cta * (p + 1) * 16 +
         (ys ? (size_t)m * 16 : 0);
}

__device__ __forceinline__ long long res_clock() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int P, bool YS>
__global__ void __launch_bounds__(kResNT, 1) cauchy_resident_kernel(CauchyResArgs a) {
  constexpr int B = kResNT;
  const CauchyParams& q = a.q;
  extern __shared__ __align__(16) unsigned char res_smem[];
  const long long n = q.n, m = q.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rows_cta = a.rows_cta, RG = rows_cta / kResRPT, CG = B / RG;
  double2* sB = reinterpret_cast<double2*>(res_smem);
  double* sbb = reinterpret_cast<double*>(sB + m * P);
  double* sw = sbb + (P == 1 ? ((m + 1) & ~1LL) : 0);
  double2* sg = reinterpret_cast<double2*>(sw + cauchy_res_wlen(n, m, rows_cta));
  double2* sx = sg + (long long)rows_cta * P;
  double2* sy = sx + rows_cta;   // YS: the column points, read in every phase
  auto ycol = [&](long long j) -> double2 { return YS ? sy[j] : __ldg(q.y + j); };
  __shared__ CdfSmem<B> sm;
  __shared__ double s_red[B / 32];
  __shared__ double s_val;

  const long long row0 = (long long)blockIdx.x * rows_cta;
  const int nrows = (int)max(0LL, min((long long)rows_cta, n - row0));
  const bool lead = blockIdx.x == 0;
  const bool tracing = a.trace != nullptr && lead && tid == 0;

  // resident state
  for (long long k = tid; k < m * P; k += B) sB[k] = q.Bt[k];
  if constexpr (YS) {
    for (long long j = tid; j < m; j += B) sy[j] = q.y[j];
  }
  if constexpr (P == 1) {
    for (long long j = tid; j < m; j += B) {
      const double2 bj = q.Bt[j];
      sbb[j] = fma(bj.x, bj.x, bj.y * bj.y);
    }
  }
  for (int k = tid; k < rows_cta; k += B) {
    const long long i = (k < nrows) ? row0 + k : 0;   // padding rows repeat row 0 (never stored)
    sx[k] = q.x[i];
#pragma unroll
    for (int l = 0; l < P; ++l) sg[k * P + l] = q.G[i * P + l];
  }
  __syncthreads();

  auto block_max = [&](double v) -> double {   // block-uniform maximum
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    double r = s_red[0];
#pragma unroll
    for (int w = 1; w < B / 32; ++w) r = fmax(r, s_red[w]);
    return r;
  };

  // loop state, identical in every thread of every CTA
  long long ucount = 0, near = 0, done = 0, err_i = -1, err_j = -1, pi = -1, pj = -1;
  int status = kRunning;
  double u0 = 0.0;
  unsigned nbar = 0;
  const double2* Gcur = q.G;
  double2* Gnext = a.gbuf;

  for (long long t = 0; t < q.rank; ++t) {
    double* M = a.mbuf + (size_t)(t & 1) * n;
    if (tracing && t < 1024) a.trace[8 * t + 0] = res_clock();
    // the step's uniforms, fetched ahead of the draws that consume them
    const bool pre = q.rule == RPLU_RULE_RPLU && ucount + 2 <= q.n_uniforms;
    const double u1p = pre ? q.uniforms[ucount] : 0.0, u2p = pre ? q.uniforms[ucount + 1] : 0.0;
    // ---- 1. masses of this CTA's rows -------------------------------------
    {
      const int rg = tid / CG, cg = tid - rg * CG;
      if (rg < RG) {
        double2 xr[kResRPT], g[kResRPT][P];
        double acc[kResRPT];
#pragma unroll
        for (int r = 0; r < kResRPT; ++r) {
          xr[r] = sx[rg * kResRPT + r];
#pragma unroll
          for (int l = 0; l < P; ++l) g[r][l] = sg[(rg * kResRPT + r) * P + l];
          acc[r] = 0.0;
        }
        const int mi = (int)m;   // resident sizes: m fits an int (cheap address math)
#pragma unroll 4
        for (int j = cg; j < mi; j += CG) {
          const double2 yj = ycol(j);
          if constexpr (P == 1) {
            const double bbj = sbb[j];
            double den[kResRPT];
#pragma unroll
            for (int r = 0; r < kResRPT; ++r) {
              const double dr = xr[r].x - yj.x, di = xr[r].y - yj.y;
              den[r] = fma(dr, dr, di * di);
            }
#pragma unroll
            for (int r = 0; r < kResRPT; ++r) acc[r] = fma(bbj, rcp_nr(den[r]), acc[r]);
          } else {
            double2 b[P];
#pragma unroll
            for (int l = 0; l < P; ++l) b[l] = sB[j * P + l];
#pragma unroll
            for (int r = 0; r < kResRPT; ++r) {
              const double dr = xr[r].x - yj.x, di = xr[r].y - yj.y;
              const double den = fma(dr, dr, di * di);
              double re = 0.0, im = 0.0;
#pragma unroll
              for (int l = 0; l < P; ++l) {
                re = fma(g[r][l].x, b[l].x, re);
                re = fma(-g[r][l].y, b[l].y, re);
                im = fma(g[r][l].x, b[l].y, im);
                im = fma(g[r][l].y, b[l].x, im);
              }
              const double num = fma(re, re, im * im);
              acc[r] = fma(num, rcp_nr(den), acc[r]);
            }
          }
        }
#pragma unroll
        for (int r = 0; r < kResRPT; ++r) {
          if constexpr (P == 1) acc[r] *= fma(g[r][0].x, g[r][0].x, g[r][0].y * g[r][0].y);
          sw[(rg * kResRPT + r) * CG + cg] = acc[r];
        }
      }
      __syncthreads();
      // per-row sum over the CG column groups: lane-strided partial sums, then
      // a fixed shuffle tree (deterministic)
      for (int lr = warp; lr < nrows; lr += B / 32) {
        double v = 0.0;
        for (int c = lane; c < CG; c += 32) v += sw[lr * CG + c];
        v = warp_sum(v);
        if (lane == 0) M[row0 + lr] = v;
      }
    }
    if (tracing && t < 1024) a.trace[8 * t + 1] = res_clock();
    // ---- 2. the step's one grid barrier ------------------------------------
    grid_barrier(a.sync, gridDim.x * (++nbar));
    if (tracing && t < 1024) a.trace[8 * t + 2] = res_clock();
    // ---- 3a. stop rules and the row draw (cauchy_select_row_dev) ------------
    // the n masses once from L2 into shared memory (the mass partials there
    // were consumed before the barrier), then CDF / maximum / search from it
    double mx = 0.0;
    for (long long k = tid; k < n; k += B) {
      const double v = __ldcg(M + k);
      sw[k] = v;
      mx = fmax(mx, v);
    }
    const double umax = block_max(mx);   // (its barriers publish sw)
    auto wrow = [&](long long k) { return sw[k]; };
    Cdf<B> cr = cdf_build<B>(wrow, n, sm);
    if (lead && tid == 0) {
      q.bmax[t] = umax;
      q.bsum[t] = cr.total;
    }
    if (t == 0) u0 = umax;
    if (umax <= 0.0) { status = kDegenerate; break; }
    if (q.stop_tol > 0.0 && umax <= q.stop_tol * q.stop_tol * u0) { status = kTolStop; break; }
    long long i;
    if (q.rule == RPLU_RULE_RPLU) {
      if (ucount + 1 > q.n_uniforms) { status = kUniformsExhausted; break; }
      const double u1 = pre ? u1p : q.uniforms[ucount];
      i = cdf_find<B>(wrow, n, cr, u1, sm);
      const double tol = kNearBoundaryRel * cr.total, tg = u1 * cr.total;
      if (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) near++;
      ucount += 1;
    } else {
      i = block_argmax<B>(wrow, n, nullptr);
    }
    pi = i;
    if (tracing && t < 1024) a.trace[8 * t + 3] = res_clock();
    // ---- 3b. pivot row r_j = (G_i . B_j) / (x_i - y_j), weights |r_j|^2 -----
    // Generated ONCE per step, a slice per CTA (two Smith divisions, one more
    // division and a square root per entry: generating all m entries in every
    // CTA cost 5.8 us of FP64-pipe time per step at C2), exchanged through
    // global memory behind the step's second grid barrier.
    double2 gi[P];
#pragma unroll
    for (int l = 0; l < P; ++l) {
      const double* gp = reinterpret_cast<const double*>(Gcur + i * P + l);
      gi[l] = make_double2(__ldcg(gp), __ldcg(gp + 1));
    }
    const double2 xi = q.x[i];
    auto rgen = [&](long long j) -> double2 {
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int l = 0; l < P; ++l) {
        const double2 b = sB[j * P + l];
        re = fma(gi[l].x, b.x, fma(-gi[l].y, b.y, re));
        im = fma(gi[l].x, b.y, fma(gi[l].y, b.x, im));
      }
      const double2 yj = ycol(j);
      return cdiv_np(make_double2(re, im), make_double2(xi.x - yj.x, xi.y - yj.y));
    };
    {
      const long long per = (m + gridDim.x - 1) / gridDim.x;
      const long long j0 = (long long)blockIdx.x * per, j1 = min(m, j0 + per);
      double amax = 0.0;
      for (long long j = j0 + tid; j < j1; j += B) {
        const double2 r = rgen(j);
        a.rglob[j] = r;
        if (q.Rout) q.Rout[t * m + j] = r;
        const double ab = cabs_np(r);
        a.wglob[j] = ab * ab;
        amax = fmax(amax, ab);
      }
      if (per <= 32) {   // the slice sits in warp 0: no CTA barrier
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        if (tid == 0) a.amaxg[blockIdx.x] = amax;
      } else {
        const double cmax = block_max(amax);
        if (tid == 0) a.amaxg[blockIdx.x] = cmax;
      }
    }
    grid_barrier(a.sync, gridDim.x * (++nbar));
    double amax = 0.0;
    for (long long j = tid; j < m; j += B) sw[j] = __ldcg(a.wglob + j);   // row masses consumed
    for (int c = tid; c < (int)gridDim.x; c += B) amax = fmax(amax, __ldcg(a.amaxg + c));
    const double rmax = block_max(amax);   // (its barriers also publish sw)
    auto rget = [&](long long j) -> double2 {
      const double* rp = reinterpret_cast<const double*>(a.rglob + j);
      return make_double2(__ldcg(rp), __ldcg(rp + 1));
    };
    if (tracing && t < 1024) a.trace[8 * t + 4] = res_clock();
    // ---- 3c. column draw with the relative zero-pivot guard ------------------
    const double thr = kPivotRelTol * rmax;
    auto wcol = [&](long long k) { return sw[k]; };
    auto wabs = [&](long long k) { return cabs_np(rget(k)); };
    long long j;
    bool zero = false;
    double2 apiv = make_double2(0.0, 0.0);   // r_j of the accepted column
    if (q.rule == RPLU_RULE_RPLU) {
      Cdf<B> cc = cdf_build<B>(wcol, m, sm);
      int attempt = 0;
      bool exhausted = false;
      for (;;) {
        if (ucount + 1 > q.n_uniforms) { exhausted = true; break; }
        const double u2 = (pre && attempt == 0) ? u2p : q.uniforms[ucount];
        ucount += 1;
        j = cdf_find<B>(wcol, m, cc, u2, sm);
        const double tol = kNearBoundaryRel * cc.total, tg = u2 * cc.total;
        if (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) near++;
        __syncthreads();
        apiv = rget(j);
        if (cabs_np(apiv) > thr) break;
        if (attempt++ == 1) { zero = true; break; }
      }
      if (exhausted) { status = kUniformsExhausted; break; }
    } else {
      j = block_argmax<B>(wabs, m, nullptr);
      apiv = rget(j);
      if (!(cabs_np(apiv) > thr)) zero = true;
    }
    if (zero) {
      status = kZeroPivot;
      err_i = i;
      err_j = j;
      break;
    }
    pj = j;
    const CDivCoef cf = cdiv_coef(apiv);
    if (lead && tid == 0) {
      q.rows[t] = i;
      q.cols[t] = j;
      if (q.Aout) q.Aout[t] = apiv;
    }
    done = t + 1;
    if (tracing && t < 1024) a.trace[8 * t + 5] = res_clock();
    // ---- 4. generator update (cauchy_update_kernel's arithmetic) -------------
    double2 bj[P];
#pragma unroll
    for (int l = 0; l < P; ++l) bj[l] = sB[j * P + l];
    const double2 yj = ycol(j);
    __syncthreads();   // every thread holds B_j before any column changes
    if (tid < rows_cta) {
      double2 g[P];
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int l = 0; l < P; ++l) {
        g[l] = sg[tid * P + l];
        re = fma(g[l].x, bj[l].x, fma(-g[l].y, bj[l].y, re));
        im = fma(g[l].x, bj[l].y, fma(g[l].y, bj[l].x, im));
      }
      const double2 xk = sx[tid];
      const double2 c = cdiv_np(make_double2(re, im), make_double2(xk.x - yj.x, xk.y - yj.y));
      const bool valid = tid < nrows;
      if (valid && q.Cout) q.Cout[t * n + row0 + tid] = c;
      const double2 ca = cdiv_apply(c, cf);
#pragma unroll
      for (int l = 0; l < P; ++l) {
        const double2 pr = cmul_np(ca, gi[l]);
        g[l] = make_double2(__dsub_rn(g[l].x, pr.x), __dsub_rn(g[l].y, pr.y));
        sg[tid * P + l] = g[l];
        if (valid) Gnext[(row0 + tid) * P + l] = g[l];
      }
    }
#pragma unroll 4
    for (long long l2 = tid; l2 < m; l2 += B) {
      const double2 ra = cdiv_apply(rget(l2), cf);
#pragma unroll
      for (int l = 0; l < P; ++l) {
        const double2 b = sB[l2 * P + l];
        const double2 pr = cmul_np(bj[l], ra);
        const double2 nb = make_double2(__dsub_rn(b.x, pr.x), __dsub_rn(b.y, pr.y));
        sB[l2 * P + l] = nb;
        if constexpr (P == 1) sbb[l2] = fma(nb.x, nb.x, nb.y * nb.y);
      }
    }
    __syncthreads();
    {  // the other global G buffer takes over
      const double2* tmp = Gcur;
      Gcur = Gnext;
      Gnext = const_cast<double2*>(tmp);
    }
    if (tracing && t < 1024) a.trace[8 * t + 6] = res_clock();
  }

  // every CTA leaves the loop at the same step; after one more barrier nobody
  // reads the global generators any more and the final state goes back
  grid_barrier(a.sync, gridDim.x * (++nbar));
  for (int k = tid; k < nrows * P; k += B) q.G[row0 * P + k] = sg[k];
  if (lead) {
    for (long long k = tid; k < m * P; k += B) q.Bt[k] = sB[k];
    if (tid == 0) {
      DevState* st = q.st;
      st->ucount = ucount;
      st->near_boundary = near;
      st->pi = pi;
      st->pj = pj;
      st->err_i = err_i;
      st->err_j = err_j;
      st->done = done;
      st->active = 0;
      st->status = status;
      st->fro0 = u0;
    }
  }
}

}  // namespace

// Resident-loop geometry for (n, m, p): CTAs, rows per CTA, shared memory
// (0 CTAs: the problem does not fit).
static int cauchy_resident_plan(int p, long long n, long long m, int sm_count, int* rows_cta,
                                size_t* smem, bool* ys) {
  if (p < 1 || p > 2 || n < 1 || m < 1) return 0;   // p > 2: 4 rows of G per thread spill
  long long ctas = std::min<long long>(sm_count, (n + kResRPT - 1) / kResRPT);
  const long long rows = (n + ctas * kResRPT - 1) / (ctas * kResRPT) * kResRPT;
  if (rows > kResNT) return 0;   // one thread per own row in the update
  ctas = (n + rows - 1) / rows;
  *rows_cta = (int)rows;
  static const size_t cap = [] {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return (size_t)(optin > 8192 ? optin - 8192 : 0);   // static shared + reserve
  }();
  *ys = cauchy_res_smem(n, m, p, (int)rows, true) <= cap;   // y resident too when it fits
  *smem = cauchy_res_smem(n, m, p, (int)rows, *ys);
  return *smem <= cap ? (int)ctas : 0;
}

template <int P, bool YS>
static int cauchy_resident_launch(rplu_ctx* ctx, const CauchyResArgs& a, int ctas, size_t smem,
                                  cudaStream_t s) {
  auto kern = cauchy_resident_kernel<P, YS>;
  static size_t attr = 0;
  if (smem > attr) {
    RPLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  int per_sm = 0;
  RPLU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kResNT, smem));
  if (per_sm < 1 || (long long)per_sm * ctx->sm_count < ctas) {
    set_error("resident Cauchy loop does not fit on the device");
    return RPLU_ERR_CUDA;
  }
  CauchyResArgs arg = a;
  void* args[] = {&arg};
  RPLU_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)ctas), dim3(kResNT), args,
                                        smem, s));
  return RPLU_OK;
}

__global__ void cauchy_init_state(DevState* st) {
  st->ucount = 0;
  st->near_boundary = 0;
  st->pi = st->pj = -1;
  st->err_i = st->err_j = -1;
  st->active = 1;
  st->status = kRunning;
  st->fro0 = 0.0;
  st->done = 0;
}

int cauchy_run_impl(rplu_ctx* ctx, const rplu_cauchy_args* a, rplu_cauchy_out* out) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(a->stream);
  const long long n = a->n, m = a->m, K = a->rank;
  const int p = a->p;
  int rc;
  CauchyParams q{};
  q.n = n;
  q.m = m;
  q.rank = K;
  q.p = p;
  q.x = reinterpret_cast<const double2*>(a->x);
  q.y = reinterpret_cast<const double2*>(a->y);
  q.G = reinterpret_cast<double2*>(a->G);
  q.Bt = reinterpret_cast<double2*>(a->Bt);
  q.splits = choose_splits(n, m, rows_per_cta(p, n, m), ctx->sm_count);
  q.stop_tol = a->stop_tol;
  q.rule = a->rule;
  if ((rc = ctx->scratch[0].ensure(sizeof(double) * (size_t)q.splits * n))) return rc;
  if ((rc = ctx->scratch[1].ensure(sizeof(double2) * (size_t)m))) return rc;
  if ((rc = ctx->scratch[2].ensure(sizeof(double) * (size_t)m))) return rc;
  if ((rc = ctx->scratch[3].ensure(sizeof(double2) * 16))) return rc;
  if ((rc = ctx->state.ensure(sizeof(DevState)))) return rc;
  if ((rc = ctx->pivots.ensure(sizeof(long long) * (size_t)(2 * K + 2)))) return rc;
  if ((rc = ctx->resid.ensure(sizeof(double) * (size_t)(2 * K + 2)))) return rc;
  long long nu = (a->rule == RPLU_RULE_RPLU) ? a->n_uniforms : 0;
  if ((rc = ctx->uniforms.ensure(sizeof(double) * (size_t)(nu > 0 ? nu : 1)))) return rc;
  if (nu > 0)
    RPLU_CUDA(cudaMemcpyAsync(ctx->uniforms.ptr, a->uniforms, sizeof(double) * nu,
                              cudaMemcpyHostToDevice, s));
  q.partial = reinterpret_cast<double*>(ctx->scratch[0].ptr);
  if ((rc = ctx->masses.ensure(sizeof(double) * (size_t)n))) return rc;
  q.masses = q.splits > 1 ? reinterpret_cast<double*>(ctx->masses.ptr) : q.partial;
  q.rbuf = reinterpret_cast<double2*>(ctx->scratch[1].ptr);
  q.wbuf = reinterpret_cast<double*>(ctx->scratch[2].ptr);
  double2* gsnap = reinterpret_cast<double2*>(ctx->scratch[3].ptr);
  q.Cout = reinterpret_cast<double2*>(a->C);
  q.Rout = reinterpret_cast<double2*>(a->Rrow);
  q.Aout = reinterpret_cast<double2*>(a->a);
  q.st = reinterpret_cast<DevState*>(ctx->state.ptr);
  q.uniforms = reinterpret_cast<const double*>(ctx->uniforms.ptr);
  q.n_uniforms = nu;
  // fused per-step bookkeeping: split sums in K5, row max in K6a, snapshot
  // in the column select (no sum / snapshot launches)
  const long long mass_blocks = (n + rows_per_cta(p, n, m) - 1) / rows_per_cta(p, n, m);
  const size_t sync_bytes = sizeof(unsigned long long) * (size_t)(mass_blocks + 1);
  if ((rc = ctx->csync.ensure(sync_bytes))) return rc;
  q.rmax_bits = reinterpret_cast<unsigned long long*>(ctx->csync.ptr);
  q.blk_count = reinterpret_cast<unsigned*>(q.rmax_bits + 1);
  q.gsnap = gsnap;
  long long* piv = reinterpret_cast<long long*>(ctx->pivots.ptr);
  q.rows = piv;
  q.cols = piv + K + 1;
  double* bb = reinterpret_cast<double*>(ctx->resid.ptr);
  q.bmax = bb;
  q.bsum = bb + K + 1;
  const bool timing = (a->flags & RPLU_FLAG_TIME_KERNELS) != 0;
  std::vector<cudaEvent_t> ev;
  long long launches = 1;
  const int upd_blocks = (int)std::min<long long>((n + m + 255) / 256, 8LL * ctx->sm_count);
  // per-step GPU time of tens of microseconds: capture the loop as one graph
  const bool graph = (a->flags & (RPLU_FLAG_NO_GRAPH | RPLU_FLAG_TIME_KERNELS)) == 0 &&
                     (double)n * (double)m * p <= 256.0 * 1024 * 1024 && K >= 4;
  // small problems: the whole loop in one cooperative launch (resident
  // generators, one grid barrier per step) unless per-kernel timing or
  // per-step launches were asked for (RPLU_CAUCHY_RESIDENT=0 disables)
  int res_rows = 0;
  size_t res_smem = 0;
  bool res_ys = false;
  static const bool res_env = [] {
    const char* e = getenv("RPLU_CAUCHY_RESIDENT");
    return !(e && e[0] == '0');
  }();
  const int res_ctas =
      (res_env && (a->flags & (RPLU_FLAG_TIME_KERNELS | RPLU_FLAG_STEPWISE)) == 0 && K >= 1 &&
       (double)n * (double)m * p <= 256.0 * 1024 * 1024)
          ? cauchy_resident_plan(p, n, m, ctx->sm_count, &res_rows, &res_smem, &res_ys)
          : 0;
  if (res_ctas > 0) {
    CauchyResArgs ra{};
    ra.q = q;
    ra.rows_cta = res_rows;
    if ((rc = ctx->masses2.ensure(sizeof(double) * 2 * (size_t)n))) return rc;
    if ((rc = ctx->scratch[3].ensure(sizeof(double2) * std::max<size_t>((size_t)n * p, 16)))) return rc;
    if ((rc = ctx->gbar.ensure(2 * sizeof(unsigned)))) return rc;
    ra.q.gsnap = nullptr;
    ra.mbuf = reinterpret_cast<double*>(ctx->masses2.ptr);
    ra.gbuf = reinterpret_cast<double2*>(ctx->scratch[3].ptr);
    ra.sync = reinterpret_cast<unsigned*>(ctx->gbar.ptr);
    ra.rglob = q.rbuf;                                   // scratch[1]: m double2
    ra.wglob = q.wbuf;                                   // scratch[2]: m doubles
    if ((rc = ctx->csync.ensure(std::max(sync_bytes, sizeof(double) * (size_t)res_ctas)))) return rc;
    ra.amaxg = reinterpret_cast<double*>(ctx->csync.ptr);
    RPLU_CUDA(cudaMemsetAsync(ctx->gbar.ptr, 0, 2 * sizeof(unsigned), s));
    static const bool tracing = getenv("RPLU_PERSIST_TRACE") != nullptr;
    if (tracing) {
      RPLU_CUDA(cudaMalloc(&ra.trace, sizeof(long long) * 8 * 1024));
      RPLU_CUDA(cudaMemsetAsync(ra.trace, 0, sizeof(long long) * 8 * 1024, s));
    }
    cauchy_init_state<<<1, 1, 0, s>>>(q.st);
    if (p == 1)
      rc = res_ys ? cauchy_resident_launch<1, true>(ctx, ra, res_ctas, res_smem, s)
                  : cauchy_resident_launch<1, false>(ctx, ra, res_ctas, res_smem, s);
    else
      rc = res_ys ? cauchy_resident_launch<2, true>(ctx, ra, res_ctas, res_smem, s)
                  : cauchy_resident_launch<2, false>(ctx, ra, res_ctas, res_smem, s);
    if (rc) return rc;
    launches = 2;
    if (tracing) {
      std::vector<long long> h(8 * 1024);
      RPLU_CUDA(cudaMemcpyAsync(h.data(), ra.trace, sizeof(long long) * h.size(),
                                cudaMemcpyDeviceToHost, s));
      RPLU_CUDA(cudaStreamSynchronize(s));
      cudaFree(ra.trace);
      const char* names[6] = {"masses", "barrier", "row draw", "pivot row", "col draw", "update"};
      double acc[6] = {0, 0, 0, 0, 0, 0};
      long long k = 0;
      for (; k < 1024 && k < K && h[8 * k + 6] != 0; ++k)
        for (int ph = 0; ph < 6; ++ph) acc[ph] += (double)(h[8 * k + ph + 1] - h[8 * k + ph]);
      if (k > 0) {
        fprintf(stderr, "[rplu] resident cauchy loop, CTA 0, %lld steps (us/step):", k);
        for (int ph = 0; ph < 6; ++ph) fprintf(stderr, " %s %.2f", names[ph], acc[ph] / k / 1e3);
        fprintf(stderr, "\n");
      }
    }
  } else
  rc = run_maybe_graph(ctx, s, graph, 1, [&](cudaStream_t qs) -> int {
    RPLU_CUDA(cudaMemsetAsync(ctx->csync.ptr, 0, sync_bytes, qs));
    cauchy_init_state<<<1, 1, 0, qs>>>(q.st);
    for (long long t = 0; t < K; ++t) {
      q.t = t;
      if (timing) {
        cudaEvent_t e0;
        cudaEventCreate(&e0);
        cudaEventRecord(e0, qs);
        ev.push_back(e0);
      }
      RPLU_P_SWITCH(p, launch_mass<PP>(q, qs));
      if (timing) {
        cudaEvent_t e1;
        cudaEventCreate(&e1);
        cudaEventRecord(e1, qs);
        ev.push_back(e1);
      }
      RPLU_P_SWITCH(p, (cauchy_select_kernel<PP><<<1, 1024, 0, qs>>>(q)));
      RPLU_P_SWITCH(p, (cauchy_update_kernel<PP><<<upd_blocks, 256, 0, qs>>>(q, gsnap)));
      launches += 3;
    }
    RPLU_CUDA(cudaGetLastError());
    return RPLU_OK;
  });
  if (rc) return rc;
  RPLU_CUDA(cudaGetLastError());
  DevState hs;
  RPLU_CUDA(cudaMemcpyAsync(&hs, q.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaStreamSynchronize(s));
  const long long done = hs.done;
  // bounds are recorded for every step that started (done, plus the stopping one)
  long long nb = done + ((hs.status == kTolStop || hs.status == kDegenerate ||
                          hs.status == kZeroPivot) ? 1 : 0);
  if (nb > K) nb = K;
  if (done > 0) {
    RPLU_CUDA(cudaMemcpy(out->rows, q.rows, sizeof(long long) * done, cudaMemcpyDeviceToHost));
    RPLU_CUDA(cudaMemcpy(out->cols, q.cols, sizeof(long long) * done, cudaMemcpyDeviceToHost));
  }
  if (nb > 0) {
    RPLU_CUDA(cudaMemcpy(out->bound_maxes, q.bmax, sizeof(double) * nb, cudaMemcpyDeviceToHost));
    RPLU_CUDA(cudaMemcpy(out->bound_sums, q.bsum, sizeof(double) * nb, cudaMemcpyDeviceToHost));
  }
  out->steps_done = done;
  out->bounds_recorded = nb;
  out->uniforms_consumed = hs.ucount;
  out->near_boundary_draws = hs.near_boundary;
  out->tol_stop = hs.status == kTolStop;
  out->degenerate_stop = hs.status == kDegenerate;
  out->zero_pivot_i = hs.err_i;
  out->zero_pivot_j = hs.err_j;
  out->kernel_launches = launches;
  out->masses_ms = 0.0;
  out->masses_launches = 0;
  if (timing) {
    for (size_t k = 0; k + 1 < ev.size(); k += 2) {
      if ((long long)(k / 2) >= nb) break;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
      out->masses_ms += ms;
      out->masses_launches++;
    }
    for (auto e : ev) cudaEventDestroy(e);
  }
  return hs.status;
}

// ---------------------------------------------------------------------------
// Row-block sharded Cauchy-like RPLU.  Rank s owns rows
// [row_offset, row_offset + n_local) of x / G; y / Bt are replicated.
namespace {

struct CauchyShard {
  CauchyParams q;
  double2* gsnap;
  int world, rank;
  long long row_offset;
  long long steps;
};

// Local [sum u_i (the CDF code's association), max u_i] of the local rows.
__global__ void __launch_bounds__(1024) cauchy_shard_stats_kernel(const double* masses, long long n,
                                                                 double* out) {
  constexpr int B = 1024;
  __shared__ CdfSmem<B> sm;
  __shared__ double s_max[B / 32];
  double mx = 0.0;
  for (long long k = threadIdx.x; k < n; k += B) mx = fmax(mx, masses[k]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mx;
  double total = 0.0;
  if (n > 0) {
    auto w = [&](long long k) { return masses[k]; };
    Cdf<B> c = cdf_build<B>(w, n, sm);
    total = c.total;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m2 = 0.0;
    for (int k = 0; k < B / 32; ++k) m2 = fmax(m2, s_max[k]);
    out[0] = total;
    out[1] = m2;
  }
}

__device__ __forceinline__ void cauchy_msg_neg_zero(double* msg) {
  if (threadIdx.x < RPLU_CAUCHY_MSG_DOUBLES) msg[threadIdx.x] = -0.0;
}

// Global stats + stop rules + owner (every rank identically), owner's local
// row draw, pivot message.
__global__ void __launch_bounds__(1024) cauchy_shard_select_kernel(CauchyParams q, int world,
                                                                  int rank, long long row_offset,
                                                                  const double* totals,
                                                                  double* msg) {
  constexpr int B = 1024;
  DevState* st = q.st;
  __shared__ CdfSmem<B> sm;
  __shared__ int s_owner, s_stop;
  __shared__ double s_target;
  if (!st->active) {
    cauchy_msg_neg_zero(msg);
    return;
  }
  const long long t = q.t;
  if (threadIdx.x == 0) {
    double T_all = 0.0, umax = 0.0;
    for (int s = 0; s < world; ++s) {
      T_all += totals[2 * s];
      umax = fmax(umax, totals[2 * s + 1]);
    }
    q.bmax[t] = umax;
    q.bsum[t] = T_all;
    if (t == 0) st->fro0 = umax;
    const double u0 = (t == 0) ? umax : st->fro0;
    int stop = 0;
    if (umax <= 0.0) {
      st->status = kDegenerate;
      stop = 1;
    } else if (q.stop_tol > 0.0 && umax <= q.stop_tol * q.stop_tol * u0) {
      st->status = kTolStop;
      stop = 1;
    } else if (q.rule == RPLU_RULE_RPLU && st->ucount + 1 > q.n_uniforms) {
      st->status = kUniformsExhausted;
      stop = 1;
    }
    int owner = -1;
    double target = 0.0;
    if (!stop) {
      if (q.rule == RPLU_RULE_RPLU) {
        const double tg = q.uniforms[st->ucount] * T_all;
        double c = 0.0;
        int last_pos = -1;
        for (int s = 0; s < world; ++s) {
          if (totals[2 * s] > 0.0) last_pos = s;
          const double c2 = c + totals[2 * s];
          if (owner < 0 && c2 > tg && totals[2 * s] > 0.0) {
            owner = s;
            target = tg - c;
          }
          c = c2;
        }
        if (owner < 0) {
          owner = last_pos;
          target = totals[2 * owner];
        }
        const double tol = kNearBoundaryRel * T_all;
        double cb = 0.0;
        for (int s = 0; s <= owner; ++s) {
          if (fabs(cb - tg) <= tol) st->near_boundary++;
          cb += totals[2 * s];
        }
        st->ucount += 1;
      } else {
        // greedy: the first shard holding the global maximum (np.argmax)
        for (int s = 0; s < world && owner < 0; ++s)
          if (totals[2 * s + 1] == umax) owner = s;
      }
    }
    if (stop) st->active = 0;
    s_stop = stop;
    s_owner = owner;
    s_target = target;
  }
  __syncthreads();
  if (s_stop || s_owner != rank) {
    cauchy_msg_neg_zero(msg);
    return;
  }
  const double* masses = q.masses;
  auto wrow = [&](long long k) { return masses[k]; };
  long long i;
  if (q.rule == RPLU_RULE_RPLU) {
    Cdf<B> cr = cdf_build<B>(wrow, q.n, sm);
    i = cdf_find_target<B>(wrow, q.n, cr, s_target, sm);
  } else {
    i = block_argmax<B>(wrow, q.n, nullptr);
  }
  if (threadIdx.x == 0) {
    msg[0] = (double)(row_offset + i);
    msg[1] = 0.0;
    msg[2] = q.x[i].x;
    msg[3] = q.x[i].y;
  }
  if (threadIdx.x < 8) {
    const int l = threadIdx.x;
    const double2 g = l < q.p ? q.G[i * q.p + l] : make_double2(-0.0, -0.0);
    msg[4 + 2 * l] = g.x;
    msg[5 + 2 * l] = g.y;
  }
}

__global__ void cauchy_shard_init_state(DevState* st) {
  st->ucount = 0;
  st->near_boundary = 0;
  st->pi = st->pj = -1;
  st->err_i = st->err_j = -1;
  st->active = 1;
  st->status = kRunning;
  st->fro0 = 0.0;
  st->done = 0;
  st->step = 0;
}

int cauchy_shard_setup(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, CauchyShard& sh,
                       bool alloc) {
  const long long n = a->n_local, m = a->m, K = a->steps;
  CauchyParams& q = sh.q;
  q = CauchyParams{};
  q.n = n;
  q.m = m;
  q.rank = K;
  q.p = a->p;
  q.x = reinterpret_cast<const double2*>(a->x);
  q.y = reinterpret_cast<const double2*>(a->y);
  q.G = reinterpret_cast<double2*>(a->G);
  q.Bt = reinterpret_cast<double2*>(a->Bt);
  q.splits = n > 0 ? choose_splits(n, m, rows_per_cta(a->p, n, m), ctx->sm_count) : 1;
  q.stop_tol = a->stop_tol;
  q.rule = a->rule;
  int rc;
  if (alloc) {
    const size_t nn = (size_t)(n > 0 ? n : 1);
    if ((rc = ctx->scratch[0].ensure(sizeof(double) * (size_t)q.splits * nn))) return rc;
    if ((rc = ctx->scratch[1].ensure(sizeof(double2) * (size_t)m))) return rc;
    if ((rc = ctx->scratch[2].ensure(sizeof(double) * (size_t)m))) return rc;
    if ((rc = ctx->scratch[3].ensure(sizeof(double2) * 16))) return rc;
    if ((rc = ctx->state.ensure(sizeof(DevState)))) return rc;
    if ((rc = ctx->pivots.ensure(sizeof(long long) * (size_t)(2 * K + 2)))) return rc;
    if ((rc = ctx->resid.ensure(sizeof(double) * (size_t)(2 * K + 2)))) return rc;
    if ((rc = ctx->masses.ensure(sizeof(double) * nn))) return rc;
    const long long nu = a->rule == RPLU_RULE_RPLU ? a->n_uniforms : 0;
    if ((rc = ctx->uniforms.ensure(sizeof(double) * (size_t)(nu > 0 ? nu : 1)))) return rc;
  }
  q.partial = reinterpret_cast<double*>(ctx->scratch[0].ptr);
  q.masses = q.splits > 1 ? reinterpret_cast<double*>(ctx->masses.ptr) : q.partial;
  q.rbuf = reinterpret_cast<double2*>(ctx->scratch[1].ptr);
  q.wbuf = reinterpret_cast<double*>(ctx->scratch[2].ptr);
  sh.gsnap = reinterpret_cast<double2*>(ctx->scratch[3].ptr);
  q.Cout = reinterpret_cast<double2*>(a->C);
  q.Rout = reinterpret_cast<double2*>(a->Rrow);
  q.Aout = reinterpret_cast<double2*>(a->a);
  q.st = reinterpret_cast<DevState*>(ctx->state.ptr);
  q.uniforms = reinterpret_cast<const double*>(ctx->uniforms.ptr);
  q.n_uniforms = a->rule == RPLU_RULE_RPLU ? a->n_uniforms : 0;
  long long* piv = reinterpret_cast<long long*>(ctx->pivots.ptr);
  q.rows = piv;
  q.cols = piv + K + 1;
  double* bb = reinterpret_cast<double*>(ctx->resid.ptr);
  q.bmax = bb;
  q.bsum = bb + K + 1;
  sh.world = a->world;
  sh.rank = a->rank;
  sh.row_offset = a->row_offset;
  sh.steps = K;
  return RPLU_OK;
}

// K5 masses of the local rows (+ split sum) and the local stats.
int cauchy_shard_masses(CauchyShard& sh, double* stats, cudaStream_t s) {
  CauchyParams& q = sh.q;
  if (q.n > 0) {
    RPLU_P_SWITCH(q.p, launch_mass<PP>(q, s));
    if (q.splits > 1)
      sum_partials_kernel<<<(unsigned)((q.n + 255) / 256), 256, 0, s>>>(q.partial, q.splits, q.n,
                                                                        q.masses);
  }
  cauchy_shard_stats_kernel<<<1, 1024, 0, s>>>(q.masses, q.n, stats);
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

}  // namespace

int cauchy_shard_begin_impl(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, double* stats) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(a->stream);
  CauchyShard sh;
  int rc;
  if ((rc = cauchy_shard_setup(ctx, a, sh, true))) return rc;
  if (sh.q.n_uniforms > 0)
    RPLU_CUDA(cudaMemcpyAsync(ctx->uniforms.ptr, a->uniforms, sizeof(double) * sh.q.n_uniforms,
                              cudaMemcpyHostToDevice, s));
  cauchy_shard_init_state<<<1, 1, 0, s>>>(sh.q.st);
  // K5 reads q.st->active (set by the init kernel, stream-ordered)
  return cauchy_shard_masses(sh, stats, s);
}

int cauchy_shard_select_impl(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, long long t,
                             const double* totals, void* msg) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(a->stream);
  CauchyShard sh;
  int rc;
  if ((rc = cauchy_shard_setup(ctx, a, sh, false))) return rc;
  sh.q.t = t;
  cauchy_shard_select_kernel<<<1, 1024, 0, s>>>(sh.q, sh.world, sh.rank, sh.row_offset, totals,
                                                reinterpret_cast<double*>(msg));
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

int cauchy_shard_update_impl(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, long long t,
                             const void* msg, double* stats) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(a->stream);
  CauchyShard sh;
  int rc;
  if ((rc = cauchy_shard_setup(ctx, a, sh, false))) return rc;
  CauchyParams& q = sh.q;
  q.t = t;
  q.psrc = reinterpret_cast<const double2*>(msg);
  const int sm = ctx->sm_count;
  const int upd_blocks = (int)std::min<long long>((q.n + q.m + 255) / 256, 8LL * sm);
  const int row_blocks = (int)std::min<long long>((q.m + 255) / 256, 8LL * sm);
  RPLU_P_SWITCH(q.p, (cauchy_row_kernel<PP><<<row_blocks, 256, 0, s>>>(q)));
  cauchy_select_col_kernel<<<1, 1024, 0, s>>>(q);
  cauchy_snapshot_kernel<<<1, 32, 0, s>>>(q, sh.gsnap);
  RPLU_P_SWITCH(q.p, (cauchy_update_kernel<PP><<<upd_blocks, 256, 0, s>>>(q, sh.gsnap)));
  RPLU_CUDA(cudaGetLastError());
  if (t + 1 < sh.steps) return cauchy_shard_masses(sh, stats, s);
  return RPLU_OK;
}

int cauchy_shard_finish_impl(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, rplu_cauchy_out* out) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(a->stream);
  CauchyShard sh;
  int rc;
  if ((rc = cauchy_shard_setup(ctx, a, sh, false))) return rc;
  const CauchyParams& q = sh.q;
  DevState hs;
  RPLU_CUDA(cudaMemcpyAsync(&hs, q.st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaStreamSynchronize(s));
  const long long K = a->steps, done = hs.done;
  long long nb = done + ((hs.status == kTolStop || hs.status == kDegenerate ||
                          hs.status == kZeroPivot) ? 1 : 0);
  if (nb > K) nb = K;
  if (done > 0) {
    RPLU_CUDA(cudaMemcpy(out->rows, q.rows, sizeof(long long) * done, cudaMemcpyDeviceToHost));
    RPLU_CUDA(cudaMemcpy(out->cols, q.cols, sizeof(long long) * done, cudaMemcpyDeviceToHost));
  }
  if (nb > 0) {
    RPLU_CUDA(cudaMemcpy(out->bound_maxes, q.bmax, sizeof(double) * nb, cudaMemcpyDeviceToHost));
    RPLU_CUDA(cudaMemcpy(out->bound_sums, q.bsum, sizeof(double) * nb, cudaMemcpyDeviceToHost));
  }
  out->steps_done = done;
  out->bounds_recorded = nb;
  out->uniforms_consumed = hs.ucount;
  out->near_boundary_draws = hs.near_boundary;
  out->tol_stop = hs.status == kTolStop;
  out->degenerate_stop = hs.status == kDegenerate;
  out->zero_pivot_i = hs.err_i;
  out->zero_pivot_j = hs.err_j;
  out->masses_ms = 0.0;
  out->masses_launches = 0;
  out->kernel_launches = 0;
  return hs.status;
}

int cauchy_shard_active_impl(rplu_ctx* ctx, const rplu_cauchy_shard_args* a, int* active) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(a->stream);
  DevState hs;
  RPLU_CUDA(cudaMemcpyAsync(&hs, ctx->state.ptr, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaStreamSynchronize(s));
  *active = hs.active;
  return RPLU_OK;
}

}  // namespace rplu
