// Dense RPLU pivot loop (Alg 1) — K1 row masses, K2 two-stage pivot
// selection, K3 fused rank-1 Schur update + next-step row masses.
//
// Reference: rplu.dense_pivots.eliminate (pkg/src/rplu/dense_pivots.py:129-209)
//   per step: norms = einsum(R*conj R) (:115), i = sample_index(norms, u1),
//   j = sample_index(|R[i]|^2, u2) (:116-117), zero-pivot resample (:178-184),
//   col = R[:,j]/a, row = R[i].copy(), R -= outer(col,row) (:185-187),
//   L[:,t] = col, U[t] = row (:188-189), resid_fro = ||R||_F (:192),
//   clean stop on zero residual (:162-164), tol stop (:195-197).
//
// B200 layout: R is row-major n x ld in HBM and is streamed exactly once per
// step by K3 (read + write = 2*n*m*sizeof(T) bytes, the algorithmic traffic);
// the pivot row U[t,:] (<= 512 KB) stays L2-resident while every CTA re-reads
// it; row masses for step t+1 fall out of the same pass, so there is no
// separate reduction pass over R.  K2 is a single CTA (1024 threads) that
// scans the n masses and the m pivot-row weights; it never leaves the device,
// so the whole loop runs without a host round trip.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <type_traits>
#include <stdint.h>

#include <stdlib.h>

#include <vector>

#include "rplu_common.cuh"
#include "rplu_internal.h"

namespace rplu {

struct DenseParams {
  void* R;
  long long ld, n, m;
  void* Lt;
  void* U;
  long long ldu;
  double* masses;
  double* rowmax;
  long long* rowarg;
  DevState* st;
  long long t, steps;
  const double* uniforms;
  long long n_uniforms;
  double* resid;
  long long* pivots;
  double stop_tol;
  int rule;
  // delayed-update (lazy) mode: R holds the residual R^(t0) of the last
  // flush; steps t0..t-1 are applied on the fly from Lt / U
  long long t0;
  int lazy;
  int force;  // run the pass even after a stop (final flush)
  int fused;  // delayed updates: one FMA per pending term instead of the
              // reference's multiply-then-subtract (bit-identical to eager)
  // Gram-mass delayed updates (fp64): masses of R^(t+1) from R^(t0) without
  // applying the pending terms -- m0 - 2 lin + quad per row (see below)
  int gram;
  long long gram_t0;   // first pending step (t0) of the Gram masses
  double* m0;          // [n] exact masses at the last flush
  double* lin;         // [n] sum_s L_is (r0_i . U_s)
  double* quad;        // [n] sum_{s,s'} L_is L_is' (U_s . U_s')
  double* gmat;        // [16 x 16] U_s . U_s' of the pending steps
  // Block-relative steps (captured shard blocks): the kernels take the
  // absolute step from the device counter st->step; t, t0 and gram_t0 then
  // only carry their differences (t - t0 = pending terms before this step).
  int rel;
  long long u_rows;    // rows of U the tensor map may cover (rel mode)
  // TMA pass: residual rows per work item (<= 32; 0 = 32).  Fewer rows per
  // item let the item count fill whole waves of the 148 persistent CTAs on
  // short row blocks (4096 shard rows: 147 items of 28 rows instead of 128
  // of 32 on 148 CTAs).
  int pass_rows;
};

__device__ __forceinline__ long long lz_t(const DenseParams& p) {
  return p.rel ? p.st->step : p.t;
}
__device__ __forceinline__ long long lz_t0(const DenseParams& p) {
  return p.rel ? p.st->step - (p.t - p.t0) : p.t0;
}
__device__ __forceinline__ long long lz_g0(const DenseParams& p) {
  return p.rel ? p.st->step - (p.t - p.gram_t0) : p.gram_t0;
}

// One pending term of the delayed-update loop, R -= L_s U_s at one element:
// fused, one rounding per term (the FP64 pipe does half the work of the
// reference's multiply + subtract, so more terms fit under the HBM time);
// complex128 as numpy's product components, each with fused accumulations.
template <typename T> __device__ __forceinline__ T pend_fused(T x, T l, T u);
template <> __device__ __forceinline__ double pend_fused<double>(double x, double l, double u) {
  return fma(-l, u, x);
}
template <> __device__ __forceinline__ float pend_fused<float>(float x, float l, float u) {
  return fmaf(-l, u, x);
}
template <> __device__ __forceinline__ double2 pend_fused<double2>(double2 x, double2 l, double2 u) {
  return make_double2(fma(-l.x, u.x, fma(l.y, u.y, x.x)), fma(-l.x, u.y, fma(-l.y, u.x, x.y)));
}
template <typename T>
__device__ __forceinline__ T pend_sub(bool fused, T x, T l, T u) {
  return fused ? pend_fused<T>(x, l, u) : Scalar<T>::sub_outer(x, l, u);
}

template <typename T, int VEC>
struct alignas(sizeof(T) * VEC) VecT {
  T v[VEC];
};

template <typename T> __device__ __forceinline__ typename Scalar<T>::coef_t load_coef(const DevState* st);
template <> __device__ __forceinline__ double load_coef<double>(const DevState* st) { return st->inv_d; }
template <> __device__ __forceinline__ float load_coef<float>(const DevState* st) { return st->inv_f; }
template <> __device__ __forceinline__ CDivCoef load_coef<double2>(const DevState* st) {
  CDivCoef c;
  c.rat = st->rat;
  c.scl = st->scl;
  c.branch = st->branch;
  return c;
}

template <typename T> __device__ __forceinline__ void store_coef(DevState* st, T a);
template <> __device__ __forceinline__ void store_coef<double>(DevState* st, double a) {
  st->inv_d = Scalar<double>::make_coef(a);
  st->a_re = a;
  st->a_im = 0.0;
}
template <> __device__ __forceinline__ void store_coef<float>(DevState* st, float a) {
  st->inv_f = Scalar<float>::make_coef(a);
  st->a_re = a;
  st->a_im = 0.0;
}
template <> __device__ __forceinline__ void store_coef<double2>(DevState* st, double2 a) {
  CDivCoef c = cdiv_coef(a);
  st->rat = c.rat;
  st->scl = c.scl;
  st->branch = c.branch;
  st->a_re = a.x;
  st->a_im = a.y;
}

// ---------------------------------------------------------------------------
// K1 / K3: one CTA owns RB consecutive rows and streams them in 16-byte
// vectors.  UPDATE=false: masses only (step 0).  UPDATE=true: in-place
// R[k,:] -= (R[k,j]/a) * U[t,:] fused with the masses of the updated rows.
// The pivot-column entries R[k,j] are captured before any write of the row
// (WAR hazard), L[:,t] is written transposed (Lt[t,k]) so the
// store is coalesced.
// 16-byte vector load/store, optionally with the streaming (evict-first)
// cache hint so the once-per-step residual stream does not push the pivot row
// and the masses out of L2.
template <bool STREAM, typename V>
__device__ __forceinline__ V vload(const V* ptr) {
  if constexpr (STREAM && sizeof(V) == 16) {
    uint4 u = __ldcs(reinterpret_cast<const uint4*>(ptr));
    return *reinterpret_cast<V*>(&u);
  } else {
    return *ptr;
  }
}
template <bool STREAM, typename V>
__device__ __forceinline__ void vstore(V* ptr, const V& v) {
  if constexpr (STREAM && sizeof(V) == 16) {
    __stcs(reinterpret_cast<uint4*>(ptr), *reinterpret_cast<const uint4*>(&v));
  } else {
    *ptr = v;
  }
}

template <typename T, int VEC, int RB, bool UPDATE, bool TRACK_MAX, bool STREAM = false>
__global__ void __launch_bounds__(256) dense_sweep_kernel(DenseParams p) {
  using S = Scalar<T>;
  constexpr int NT = 256;
  if (UPDATE && !p.st->active) return;
  const long long row0 = (long long)blockIdx.x * RB;
  const long long n = p.n, m = p.m, ld = p.ld;
  // step index: the launch argument, or the device counter (t < 0, sharded
  // graph replay)
  const long long t = (UPDATE && p.t < 0) ? p.st->step : p.t;
  T* R = reinterpret_cast<T*>(p.R);
  __shared__ T lval[RB];
  if (UPDATE) {
    if (threadIdx.x < RB) {
      long long k = row0 + threadIdx.x;
      T lv = S::zero();
      if (k < n) {
        typename S::coef_t cf = load_coef<T>(p.st);
        lv = S::scale(R[k * ld + p.st->pj], cf);
        reinterpret_cast<T*>(p.Lt)[t * n + k] = lv;
      }
      lval[threadIdx.x] = lv;
    }
    __syncthreads();
  }
  T lv[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) lv[r] = UPDATE ? lval[r] : S::zero();
  const T* prow = UPDATE ? reinterpret_cast<const T*>(p.U) + t * p.ldu : nullptr;

  double acc[RB];
  double mx[RB];
  long long mi[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) { acc[r] = 0.0; mx[r] = -1.0; mi[r] = m; }

  const long long mv = (m / VEC) * VEC;  // vectorised part
  for (long long l = (long long)threadIdx.x * VEC; l < mv; l += (long long)NT * VEC) {
    VecT<T, VEC> pv;
    if (UPDATE) pv = *reinterpret_cast<const VecT<T, VEC>*>(prow + l);
    VecT<T, VEC> rv[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r)
      if (row0 + r < n)
        rv[r] = vload<STREAM>(reinterpret_cast<const VecT<T, VEC>*>(R + (row0 + r) * ld + l));
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      if (row0 + r < n) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          T x = rv[r].v[e];
          if (UPDATE) x = S::sub_outer(x, lv[r], pv.v[e]);
          rv[r].v[e] = x;
          acc[r] += S::mass(x);
          if (TRACK_MAX) argmax_merge(mx[r], mi[r], S::absval(x), l + e);
        }
        if (UPDATE) vstore<STREAM>(reinterpret_cast<VecT<T, VEC>*>(R + (row0 + r) * ld + l), rv[r]);
      }
    }
  }
  // scalar tail (m % VEC columns)
  for (long long l = mv + threadIdx.x; l < m; l += NT) {
    T pvs = UPDATE ? prow[l] : S::zero();
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      if (row0 + r < n) {
        T x = R[(row0 + r) * ld + l];
        if (UPDATE) {
          x = S::sub_outer(x, lv[r], pvs);
          R[(row0 + r) * ld + l] = x;
        }
        acc[r] += S::mass(x);
        if (TRACK_MAX) argmax_merge(mx[r], mi[r], S::absval(x), l);
      }
    }
  }
  // block reduction of the RB row masses (and maxima)
  __shared__ double red[NT / 32][RB];
  __shared__ double redm[TRACK_MAX ? NT / 32 : 1][RB];
  __shared__ long long redi[TRACK_MAX ? NT / 32 : 1][RB];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < RB; ++r) {
    double s = warp_sum(acc[r]);
    if (lane == 0) red[w][r] = s;
    if (TRACK_MAX) {
      double v = mx[r];
      long long i = mi[r];
      warp_argmax(v, i);
      if (lane == 0) { redm[w][r] = v; redi[w][r] = i; }
    }
  }
  __syncthreads();
  if (threadIdx.x < RB) {
    const int r = threadIdx.x;
    const long long k = row0 + r;
    if (k < n) {
      double s = 0.0;
#pragma unroll
      for (int ww = 0; ww < NT / 32; ++ww) s += red[ww][r];
      p.masses[k] = s;
      if (TRACK_MAX) {
        double v = -1.0;
        long long i = m;
        for (int ww = 0; ww < NT / 32; ++ww) argmax_merge(v, i, redm[ww][r], redi[ww][r]);
        p.rowmax[k] = v;
        p.rowarg[k] = i;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K2: pivot selection for step t (t == steps: final residual norm only).
template <typename T>
__global__ void __launch_bounds__(1024) dense_select_kernel(DenseParams p) {
  using S = Scalar<T>;
  constexpr int B = 1024;
  DevState* st = p.st;
  if (!st->active) return;
  __shared__ CdfSmem<B> sm;
  __shared__ long long s_i, s_j;
  __shared__ int s_stop;
  const long long n = p.n, m = p.m, ld = p.ld, t = p.t;
  const T* R = reinterpret_cast<const T*>(p.R);
  const double* masses = p.masses;
  auto wrow = [&](long long k) { return masses[k]; };
  // the step's two uniforms, loaded before the CDF build (latency overlap)
  const long long uc0 = st->ucount;
  const bool pre = p.rule == RPLU_RULE_RPLU && uc0 + 2 <= p.n_uniforms;
  const double u1p = pre ? p.uniforms[uc0] : 0.0, u2p = pre ? p.uniforms[uc0 + 1] : 0.0;

  Cdf<B> cr = cdf_build<B>(wrow, n, sm);
  const double total = cr.total;
  const double resid = sqrt(total);
  if (threadIdx.x == 0) {
    p.resid[t] = resid;
    if (t == 0) st->fro0 = resid;
    double fro0 = (t == 0) ? resid : st->fro0;
    int stop = 0;
    if (t > 0 && p.stop_tol > 0.0 && resid <= p.stop_tol * fro0) {
      st->status = kTolStop;
      stop = 1;
    } else if (t >= p.steps) {
      stop = 1;
    } else if (resid == 0.0) {
      st->status = kCleanStop;
      stop = 1;
    }
    if (stop) st->active = 0;
    s_stop = stop;
  }
  __syncthreads();
  if (s_stop) return;

  long long uc = uc0;
  long long near = 0;
  long long i = 0, j = 0;
  T a = S::zero();
  T* urow = reinterpret_cast<T*>(p.U) + t * p.ldu;
  // (eager loop: the residual in R is current; the lazy loop uses
  // lazy_select_row / lazy_row / lazy_select_col instead)
  auto pivot_row = [&](long long ii) -> const T* { return R + ii * ld; };
  const T* row = nullptr;
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (p.rule == RPLU_RULE_RPLU) {
      if (uc + 2 > p.n_uniforms) {
        if (threadIdx.x == 0) { st->status = kUniformsExhausted; st->active = 0; }
        return;
      }
      const double u1 = attempt == 0 ? u1p : p.uniforms[uc];
      const double u2 = attempt == 0 ? u2p : p.uniforms[uc + 1];
      uc += 2;
      i = cdf_find<B>(wrow, n, cr, u1, sm);
      // near-boundary accounting for the row draw
      if (threadIdx.x == 0) {
        double tol = kNearBoundaryRel * total, tg = u1 * total;
        if (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) near++;
      }
      __syncthreads();
      row = pivot_row(i);
      auto wcol = [&](long long k) { return S::weight(row[k]); };
      Cdf<B> cc = cdf_build<B>(wcol, m, sm);
      j = cdf_find<B>(wcol, m, cc, u2, sm);
      if (threadIdx.x == 0) {
        double tol = kNearBoundaryRel * cc.total, tg = u2 * cc.total;
        if (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) near++;
      }
    } else if (p.rule == RPLU_RULE_C2PLU) {
      i = block_argmax<B>(wrow, n, nullptr);
      row = pivot_row(i);
      auto wabs = [&](long long k) { return S::absval(row[k]); };
      j = block_argmax<B>(wabs, m, nullptr);
    } else {  // CPLU (eager only): flat argmax of |R| from the per-row maxima
      const double* rm = p.rowmax;
      auto wmax = [&](long long k) { return rm[k]; };
      i = block_argmax<B>(wmax, n, nullptr);
      j = p.rowarg[i];
      row = R + i * ld;
    }
    a = row[j];
    if (!S::is_zero(a)) break;
    if (attempt == 1 || p.rule != RPLU_RULE_RPLU) {
      if (threadIdx.x == 0) {
        st->status = kZeroPivot;
        st->active = 0;
        st->err_i = i;
        st->err_j = j;
        st->ucount = uc;
        st->near_boundary += near;
      }
      return;
    }
    __syncthreads();
  }
  // U[t,:] = R[i,:] (the pre-update pivot row; K3 reads it from here)
  for (long long k = threadIdx.x; k < m; k += B) urow[k] = row[k];
  if (threadIdx.x == 0) {
    st->ucount = uc;
    st->near_boundary += near;
    st->pi = i;
    st->pj = j;
    store_coef<T>(st, a);
    p.pivots[2 * t] = i;
    p.pivots[2 * t + 1] = j;
    st->done = t + 1;
  }
}

// ---------------------------------------------------------------------------
// Lazy-mode select, split in three launches so the pivot-row reconstruction
// (m elements x q pending terms) runs on the whole GPU instead of one CTA:
//   row select (1 CTA): residual norm, stop rules, row draw (u1)
//   row rebuild (grid): U[t,:] = R^(t0)[i,:] - pending terms
//   column select (1 CTA): column draw (u2) over U[t,:], zero-pivot resample

template <typename T>
__global__ void __launch_bounds__(1024) lazy_select_row_kernel(DenseParams p) {
  constexpr int B = 1024;
  DevState* st = p.st;
  if (!st->active) return;
  __shared__ CdfSmem<B> sm;
  __shared__ int s_stop;
  const long long n = p.n, t = p.t;
  const double* masses = p.masses;
  auto wrow = [&](long long k) { return masses[k]; };
  Cdf<B> cr = cdf_build<B>(wrow, n, sm);
  const double total = cr.total;
  const double resid = sqrt(total);
  if (threadIdx.x == 0) {
    p.resid[t] = resid;
    if (t == 0) st->fro0 = resid;
    const double fro0 = (t == 0) ? resid : st->fro0;
    int stop = 0;
    if (t > 0 && p.stop_tol > 0.0 && resid <= p.stop_tol * fro0) {
      st->status = kTolStop;
      stop = 1;
    } else if (t >= p.steps) {
      stop = 1;
    } else if (resid == 0.0) {
      st->status = kCleanStop;
      stop = 1;
    } else if (p.rule == RPLU_RULE_RPLU && st->ucount + 2 > p.n_uniforms) {
      st->status = kUniformsExhausted;
      stop = 1;
    }
    if (stop) st->active = 0;
    s_stop = stop;
  }
  __syncthreads();
  if (s_stop) return;
  long long i;
  if (p.rule == RPLU_RULE_RPLU) {
    const double u1 = p.uniforms[st->ucount];
    i = cdf_find<B>(wrow, n, cr, u1, sm);
    if (threadIdx.x == 0) {
      const double tol = kNearBoundaryRel * total, tg = u1 * total;
      if (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) st->near_boundary++;
      st->ucount += 1;
    }
  } else {
    i = block_argmax<B>(wrow, n, nullptr);
  }
  if (threadIdx.x == 0) st->pi = i;
}

template <typename T>
__global__ void __launch_bounds__(256) lazy_row_kernel(DenseParams p) {
  using S = Scalar<T>;
  if (!p.st->active) return;
  const long long i = p.st->pi, t = p.t, n = p.n;
  const int q = (int)(t - p.t0);
  const T* R = reinterpret_cast<const T*>(p.R);
  const T* Lt = reinterpret_cast<const T*>(p.Lt);
  const T* U = reinterpret_cast<const T*>(p.U) + p.t0 * p.ldu;
  T* urow = reinterpret_cast<T*>(p.U) + t * p.ldu;
  __shared__ T s_l[kLazyMaxBlock];
  if ((int)threadIdx.x < q) s_l[threadIdx.x] = Lt[(p.t0 + threadIdx.x) * n + i];
  __syncthreads();
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < p.m;
       k += (long long)gridDim.x * blockDim.x) {
    T x = R[i * p.ld + k];
    for (int s = 0; s < q; ++s) x = pend_sub<T>(p.fused, x, s_l[s], U[s * p.ldu + k]);
    urow[k] = x;
  }
}

template <typename T>
__global__ void __launch_bounds__(1024) lazy_select_col_kernel(DenseParams p) {
  using S = Scalar<T>;
  constexpr int B = 1024;
  DevState* st = p.st;
  if (!st->active) return;
  __shared__ CdfSmem<B> sm;
  const long long n = p.n, m = p.m, t = p.t;
  T* urow = reinterpret_cast<T*>(p.U) + t * p.ldu;
  const T* R = reinterpret_cast<const T*>(p.R);
  long long uc = st->ucount;
  long long near = 0;
  long long i = st->pi, j = 0;
  T a = S::zero();
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (attempt == 1) {
      // zero pivot (probability-zero event): resample the row with the next
      // uniform and rebuild its residual row inside this CTA
      const double* masses = p.masses;
      auto wrow = [&](long long k) { return masses[k]; };
      __syncthreads();
      Cdf<B> cr = cdf_build<B>(wrow, n, sm);
      if (uc + 2 > p.n_uniforms) {
        if (threadIdx.x == 0) { st->status = kUniformsExhausted; st->active = 0; }
        return;
      }
      const double u1 = p.uniforms[uc];
      uc += 1;
      i = cdf_find<B>(wrow, n, cr, u1, sm);
      const T* Lt = reinterpret_cast<const T*>(p.Lt);
      const T* U = reinterpret_cast<const T*>(p.U);
      for (long long k = threadIdx.x; k < m; k += B) {
        T x = R[i * p.ld + k];
        for (long long s = p.t0; s < t; ++s)
          x = pend_sub<T>(p.fused, x, Lt[s * n + i], U[s * p.ldu + k]);
        urow[k] = x;
      }
      __syncthreads();
    }
    if (p.rule == RPLU_RULE_RPLU) {
      const double u2 = p.uniforms[uc];
      uc += 1;
      auto wcol = [&](long long k) { return S::weight(urow[k]); };
      Cdf<B> cc = cdf_build<B>(wcol, m, sm);
      j = cdf_find<B>(wcol, m, cc, u2, sm);
      if (threadIdx.x == 0) {
        const double tol = kNearBoundaryRel * cc.total, tg = u2 * cc.total;
        if (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) near++;
      }
    } else {
      auto wabs = [&](long long k) { return S::absval(urow[k]); };
      j = block_argmax<B>(wabs, m, nullptr);
    }
    a = urow[j];
    if (!S::is_zero(a)) break;
    if (attempt == 1 || p.rule != RPLU_RULE_RPLU) {
      if (threadIdx.x == 0) {
        st->status = kZeroPivot;
        st->active = 0;
        st->err_i = i;
        st->err_j = j;
        st->ucount = uc;
        st->near_boundary += near;
      }
      return;
    }
  }
  if (threadIdx.x == 0) {
    st->ucount = uc;
    st->near_boundary += near;
    st->pi = i;
    st->pj = j;
    store_coef<T>(st, a);
    p.pivots[2 * t] = i;
    p.pivots[2 * t + 1] = j;
    st->done = t + 1;
  }
}

// ---------------------------------------------------------------------------
// Delayed-update (lazy) dense loop.  Between flushes R keeps R^(t0); each
// step reads R once (no write) and applies the pending rank-1 terms
// s = t0..t on the fly, in step order with the eager kernel's rounding, to
// get the masses of R^(t+1); every `block` steps the same pass writes
// R^(t+1) back (flush).  HBM traffic per step: n*m*s read (+ n*m*s write
// every block steps) instead of 2*n*m*s, at the cost of 2q FP ops per
// element (q = pending terms); the residual, L and U stay bit-identical to
// the eager path.

// L[:,t] = R^(t)[:,j] / a, the pivot column reconstructed on the fly.
template <typename T>
__global__ void __launch_bounds__(256) lazy_pivcol_kernel(DenseParams p) {
  using S = Scalar<T>;
  if (!p.st->active) return;
  const long long n = p.n, j = p.st->pj, t = lz_t(p), t0 = lz_t0(p);
  const T* R = reinterpret_cast<const T*>(p.R);
  T* Lt = reinterpret_cast<T*>(p.Lt);
  const T* U = reinterpret_cast<const T*>(p.U);
  const typename S::coef_t cf = load_coef<T>(p.st);
  const int q = (int)(t - t0);
  __shared__ T s_upiv[kLazyMaxBlock];  // U[s][j] of the pending steps
  if ((int)threadIdx.x < q) s_upiv[threadIdx.x] = U[(t0 + threadIdx.x) * p.ldu + j];
  __syncthreads();
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    T x = R[k * p.ld + j];
    T ll[kLazyMaxBlock];
#pragma unroll
    for (int s = 0; s < kLazyMaxBlock; ++s)
      if (s < q) ll[s] = Lt[(t0 + s) * n + k];
#pragma unroll
    for (int s = 0; s < kLazyMaxBlock; ++s)
      if (s < q) x = pend_sub<T>(p.fused, x, ll[s], s_upiv[s]);
    Lt[t * n + k] = S::scale(x, cf);
  }
}

// ---------------------------------------------------------------------------
// Delayed-update pass, TMA-fed (default): masses of
// R^(t+1) = R^(t0) - sum_{s=t0..t} L_s U_s and, FLUSH, the write of R^(t+1).
//
// Persistent, warp-specialised CTA (one per SM): warp 8 is the producer, one
// lane per residual row, and streams (32 rows x 1 KB) of R plus the matching
// 1 KB of each pending U row into a ring of STAGES shared-memory stages with
// 1-D bulk copies (cp.async.bulk, completion counted in bytes on the stage's
// "full" mbarrier; R with an L2 evict-first hint, U evict-last).  Warps 0..7
// consume: 64 threads across the 1 KB column chunk x 4 groups of 8 rows, each
// thread applies the QC pending terms in step order with the reference's
// rounding (one multiply, one subtract per term) to its 8 x 16 bytes and
// releases the stage with one arrive per warp on its "empty" mbarrier.  No
// CTA-wide barrier sits in the stream, so the copy engine stays up to
// STAGES x 33..48 KB ahead of the FP64 work; the only named barrier is at a
// row-block switch (pending L values, mass write-out).  A CTA owns row blocks
// b, b+grid, ...; each block's masses are summed by that CTA alone in a
// fixed order (per-thread chunks, warp tree, two warps), so the result is
// deterministic.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  unsigned ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void consumer_bar() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src,
                                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint"
      " [%0, {%1, %2}], [%3], %4;\n" ::"l"(map),
      "r"(c0), "r"(c1), "r"(smem_u32(src)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

template <typename T, int QC, int TXW = 64>
struct LazyTma {
  // TXW threads across a (TXW x 16)-byte column chunk x (256 / TXW) groups of
  // RPT rows: 32 rows x 1 KB (TXW = 64) or 16 rows x 2 KB (TXW = 128)
  static constexpr int TX = TXW, RPT = 8, ROWS = (256 / TXW) * RPT, NCW = 8;  // NCW consumer warps
  static constexpr int WPG = TX / 32;                         // warps per row group
  static constexpr int LINE = TX * 16;                        // bytes of one row per stage
  static constexpr int STAGE = (ROWS + QC) * LINE;
  static constexpr int STAGES = (196 * 1024) / STAGE > 8 ? 8 : (196 * 1024) / STAGE;
  static constexpr size_t OFF_L = (size_t)STAGES * STAGE;
  static constexpr size_t OFF_RED = OFF_L + 2 * sizeof(T) * QC * ROWS;
  static constexpr size_t OFF_BAR = (OFF_RED + 2 * NCW * RPT * sizeof(double) + 7) & ~size_t(7);
  static constexpr size_t SMEM = OFF_BAR + 2 * STAGES * sizeof(uint64_t) + 1024;  // + alignment
};

// Gram-mass delayed updates (fp64).  With r0_i the row of R^(t0) (the last
// flush) and the pending rank-1 terms s = t0..t,
//   |r_i^(t+1)|^2 = |r0_i|^2 - 2 sum_s L_is (r0_i . U_s)
//                   + sum_{s,s'} L_is L_is' (U_s . U_s'),
// so a step needs one dot product per row with the newest U row (one read of
// R at one FMA per element, whatever the number of pending terms) plus O(q)
// per row: lin_i += L_it g_it, quad_i += L_it (2 sum_{s<t} L_is G_ts +
// L_it G_tt).  The pass therefore stays HBM-bound for every q and the flush
// interval can grow to 16.  Only the sampling masses come from this formula
// (they differ from the applied-update masses by a few ulps of |r0_i|^2:
// draws change only within rounding of a CDF boundary, counted as
// near-boundary draws); L, U and the residual still come from the exact
// pending-term arithmetic (pivot row / column, flush), bit-identical to the
// eager loop.  Negative rounding residue of eliminated rows is clamped to 0.
__device__ __forceinline__ void gram_mass_update(const DenseParams& p, long long i, double g) {
  const long long t = lz_t(p), t0 = lz_g0(p), n = p.n;
  const double* Lt = reinterpret_cast<const double*>(p.Lt);
  const double* G = p.gmat + (t - t0) * kLazyMaxBlock;
  const double lt = Lt[t * n + i];
  double cross = 0.0;
  for (long long s = t0; s < t; ++s) cross = fma(Lt[s * n + i], G[s - t0], cross);
  const double lin = fma(lt, g, p.lin[i]);
  const double quad = fma(lt, fma(2.0, cross, lt * G[t - t0]), p.quad[i]);
  p.lin[i] = lin;
  p.quad[i] = quad;
  const double mass = fma(-2.0, lin, p.m0[i]) + quad;
  p.masses[i] = mass > 0.0 ? mass : 0.0;
}

// G[t - t0][s - t0] = U_t . U_s for the pending s (one CTA of 1024 threads
// per s; 8 independent loads in flight per thread -- with 256 threads and a
// serial load-FMA loop the kernel was L2-latency bound at 23 us per step at
// m = 32768 -- then a fixed-order reduction: deterministic)
__global__ void __launch_bounds__(1024) lazy_gram_kernel(DenseParams p) {
  if (!p.st->active) return;
  const long long t = lz_t(p), g0 = lz_g0(p), s = g0 + blockIdx.x, m = p.m;
  const double* U = reinterpret_cast<const double*>(p.U);
  const double* ut = U + t * p.ldu;
  const double* us = U + s * p.ldu;
  constexpr int NT = 1024, UN = 8;
  double acc[UN];
#pragma unroll
  for (int u = 0; u < UN; ++u) acc[u] = 0.0;
  for (long long k0 = threadIdx.x; k0 < m; k0 += (long long)NT * UN) {
    double a[UN], b[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const long long k = k0 + (long long)u * NT;
      a[u] = k < m ? ut[k] : 0.0;
      b[u] = k < m ? us[k] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) acc[u] = fma(a[u], b[u], acc[u]);
  }
  double v = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  v = warp_sum(v);
  __shared__ double red[NT / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < NT / 32; ++w) r += red[w];
    p.gmat[(t - g0) * kLazyMaxBlock + blockIdx.x] = r;
  }
}

// start of a pending block: m0 = the exact masses, lin = quad = 0
__global__ void gram_reset_kernel(DenseParams p) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
       i += (long long)gridDim.x * blockDim.x) {
    p.m0[i] = p.masses[i];
    p.lin[i] = 0.0;
    p.quad[i] = 0.0;
  }
}

// tmR: R as a 2-D tensor (columns x rows, in 8-byte words for fp64 and
// complex128, 4-byte for fp32), box = 1 KB x 32 rows; tmU: the pending rows
// U[t0 .. t0+QC) with box 1 KB x QC rows.  Out-of-range rows and columns are
// zero-filled by the TMA unit, so every stage carries (32 + QC) KB.
template <typename T, int VEC, bool FLUSH, int QC, int TXW = 64, bool FUSED = false,
          bool DOT = false>
__global__ void __launch_bounds__(288, 1)
    lazy_pass4_kernel(DenseParams p, const __grid_constant__ CUtensorMap tmR,
                      const __grid_constant__ CUtensorMap tmU) {
  using S = Scalar<T>;
  using C = LazyTma<T, QC, TXW>;
  using V = VecT<T, VEC>;
  constexpr int TX = C::TX, RPT = C::RPT, ROWS = C::ROWS, STAGES = C::STAGES, CW = TX * VEC;
  constexpr int WORDS = C::LINE / (sizeof(T) == 4 ? 4 : 8);  // box inner extent in map words
  static_assert(WORDS <= 256, "TMA box extent");
  static_assert(sizeof(V) == 16, "16-byte vectors");
  if (!p.force && !p.st->active) return;
  extern __shared__ __align__(1024) unsigned char smem_dyn[];
  unsigned char* smem_raw =
      smem_dyn + ((1024 - (smem_u32(smem_dyn) & 1023)) & 1023);  // 1 KB-aligned stages
  V* tiles = reinterpret_cast<V*>(smem_raw);
  T* Ls = reinterpret_cast<T*>(smem_raw + C::OFF_L);  // [2][QC][ROWS]
  double* red = reinterpret_cast<double*>(smem_raw + C::OFF_RED);  // [2][NCW][RPT]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + C::OFF_BAR);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const long long n = p.n, m = p.m, ld = p.ld;
  const long long nchunks = (m + CW - 1) / CW;
  // rows per work item: the stage layout stays ROWS rows, an item fills RB
  const int RB = (p.pass_rows > 0 && p.pass_rows < ROWS) ? p.pass_rows : ROWS;
  const long long nblocks = (n + RB - 1) / RB;
  const T* Lt = reinterpret_cast<const T*>(p.Lt);
  const long long l_row0 = lz_t0(p);

  if (warp == C::NCW) {  // producer warp: one elected lane issues two TMA loads per stage
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmR) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmU) : "memory");
      const uint64_t pol_r = policy_evict_first(), pol_u = policy_evict_last();
      const int u_row0 = (int)lz_t0(p);
      int stage = 0;
      unsigned phase = 0;
      long long i = 0;  // items (row block, column chunk) issued by this CTA
      // FLUSH: the consumers write the updated tile back into its stage; the
      // stage's previous occupant (item i - STAGES) is stored with one TMA
      // store before the stage is refilled (rows / columns outside R are
      // clipped by the tensor map).
      auto store_item = [&](long long j) {
        const long long rbj = blockIdx.x + (j / nchunks) * gridDim.x, cj = j % nchunks;
        const V* sj = tiles + (size_t)(j % STAGES) * (ROWS + QC) * TX;
        tma_store_2d(&tmR, (int)(cj * WORDS), (int)(rbj * RB), sj, pol_r);
        bulk_commit();
      };
      for (long long rb = blockIdx.x; rb < nblocks; rb += gridDim.x) {
        for (long long c = 0; c < nchunks; ++c, ++i) {
          mbar_wait(&empty[stage], phase ^ 1);
          V* st = tiles + (size_t)stage * (ROWS + QC) * TX;
          if constexpr (FLUSH) {
            if (i >= STAGES) {
              store_item(i - STAGES);
              bulk_wait_read_all();  // the store has read the stage
            }
          }
          mbar_expect_tx(&full[stage], (unsigned)((RB + QC) * C::LINE));
          tma_load_2d(st, &tmR, (int)(c * WORDS), (int)(rb * RB), &full[stage], pol_r);
          tma_load_2d(st + ROWS * TX, &tmU, (int)(c * WORDS), u_row0, &full[stage], pol_u);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if constexpr (FLUSH) {
        for (long long j = i > STAGES ? i - STAGES : 0; j < i; ++j) {
          mbar_wait(&empty[j % STAGES], (unsigned)((j / STAGES) & 1));
          store_item(j);
        }
        bulk_wait_all();
      }
    }
    return;
  }

  // consumers
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  int stage = 0;
  unsigned phase = 0;
  int k = 0;  // row blocks done by this CTA
  long long prev_row0 = -1;
  for (long long rb = blockIdx.x; rb < nblocks; rb += gridDim.x, ++k) {
    const long long row0 = rb * RB;
    const int buf = k & 1;
    T* L = Ls + buf * QC * ROWS;
    for (int idx = threadIdx.x; idx < QC * ROWS; idx += C::NCW * 32) {
      const int s = idx / ROWS, r = idx % ROWS;
      L[idx] = (r < RB && row0 + r < n) ? Lt[(l_row0 + s) * n + row0 + r] : S::zero();
    }
    consumer_bar();  // L visible; red[buf^1] of the previous block complete
    if (prev_row0 >= 0 && threadIdx.x < RB) {
      const double* rd = red + (buf ^ 1) * C::NCW * RPT;
      const int g = threadIdx.x / RPT, r = threadIdx.x % RPT;
      if (prev_row0 + threadIdx.x < n) {
        double sv = rd[(C::WPG * g) * RPT + r];
#pragma unroll
        for (int q = 1; q < C::WPG; ++q) sv += rd[(C::WPG * g + q) * RPT + r];
        if constexpr (DOT) gram_mass_update(p, prev_row0 + threadIdx.x, sv);
        else p.masses[prev_row0 + threadIdx.x] = sv;
      }
    }
    const long long myrow0 = row0 + ty * RPT;
    const int nr = (int)max(0LL, min(min((long long)RPT, (long long)(RB - ty * RPT)), n - myrow0));
    double acc[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) acc[r] = 0.0;
    for (long long c = 0; c < nchunks; ++c) {
      mbar_wait(&full[stage], phase);
      V* st = tiles + (size_t)stage * (ROWS + QC) * TX;
      const long long l = c * CW + (long long)tx * VEC;
      if (DOT && l < m) {
        // Gram-mass step: g_i = r0_i . U_t (the stage's one U row is U_t)
        if constexpr (!std::is_same<T, double2>::value) {   // real types only
          const V u = st[ROWS * TX + tx];
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const V x = st[(ty * RPT + r) * TX + tx];
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              if (VEC == 1 || l + e < m) acc[r] = fma((double)x.v[e], (double)u.v[e], acc[r]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
      } else if (l < m) {
        V rv[RPT];
#pragma unroll
        for (int r = 0; r < RPT; ++r) rv[r] = st[(ty * RPT + r) * TX + tx];
#pragma unroll
        for (int s = 0; s < QC; ++s) {
          const V u = st[(ROWS + s) * TX + tx];
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const T lv = L[s * ROWS + ty * RPT + r];
#pragma unroll
            for (int e = 0; e < VEC; ++e)
              rv[r].v[e] = FUSED ? pend_fused<T>(rv[r].v[e], lv, u.v[e])
                                 : S::sub_outer(rv[r].v[e], lv, u.v[e]);
          }
        }
        if constexpr (FLUSH) {
#pragma unroll
          for (int r = 0; r < RPT; ++r) st[(ty * RPT + r) * TX + tx] = rv[r];
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // visible to the TMA store
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (VEC == 1 || l + VEC <= m) {
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            if (r < nr) {
#pragma unroll
              for (int e = 0; e < VEC; ++e) acc[r] += S::mass(rv[r].v[e]);
            }
          }
        } else {  // last, partial vector of a row (m % VEC columns)
          for (int r = 0; r < RPT; ++r) {
            if (r < nr) {
              for (int e = 0; e < VEC && l + e < m; ++e) acc[r] += S::mass(rv[r].v[e]);
            }
          }
        }
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
      }
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
    double* rd = red + buf * C::NCW * RPT;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const double sv = warp_sum(acc[r]);
      if (lane == 0) rd[warp * RPT + r] = sv;
    }
    prev_row0 = row0;
  }
  consumer_bar();
  if (prev_row0 >= 0 && threadIdx.x < RB) {
    const double* rd = red + ((k - 1) & 1) * C::NCW * RPT;
    const int g = threadIdx.x / RPT, r = threadIdx.x % RPT;
    if (prev_row0 + threadIdx.x < n) {
      double sv = rd[(C::WPG * g) * RPT + r];
#pragma unroll
      for (int q = 1; q < C::WPG; ++q) sv += rd[(C::WPG * g + q) * RPT + r];
      if constexpr (DOT) gram_mass_update(p, prev_row0 + threadIdx.x, sv);
      else p.masses[prev_row0 + threadIdx.x] = sv;
    }
  }
}

// Pipelined version: the next column chunk of the CTA's residual rows and of
// the pending U rows is copied global->shared with cp.async (LDGSTS) while
// the current chunk is computed, so the HBM stream and the 2q FP operations
// per element overlap.  Each thread reads back only the residual elements it
// copied itself; the U chunk is shared by the CTA's rows.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <typename T, int VEC, int RPT>
struct LazyPipeSmem {
  static constexpr int TX = 64, TY = 4, ROWS = TY * RPT;
  VecT<T, VEC> Rs[2][ROWS][TX];
  VecT<T, VEC> Us[2][kLazyMaxBlock][TX];
  T Ls[kLazyMaxBlock][ROWS];
  double red[8][RPT];
};

// QC > 0: the number of pending terms is a compile-time constant (one
// instantiation per q), so the term loop is fully unrolled with immediate
// shared-memory offsets and the FP64 pipe is not starved by address math.
template <typename T, int VEC, int RPT, bool FLUSH, int QC = 0>
__global__ void __launch_bounds__(256) lazy_pass3_kernel(DenseParams p) {
  using S = Scalar<T>;
  using SM = LazyPipeSmem<T, VEC, RPT>;
  constexpr int NT = 256, TX = SM::TX, ROWS = SM::ROWS, CW = TX * VEC;
  static_assert(sizeof(VecT<T, VEC>) == 16, "16-byte vectors");
  if (!p.force && !p.st->active) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const long long row0 = (long long)blockIdx.x * ROWS;
  const long long n = p.n, m = p.m, ld = p.ld;
  const int q = QC > 0 ? QC : (int)(p.t - p.t0 + 1);
  T* R = reinterpret_cast<T*>(p.R);
  const T* Lt = reinterpret_cast<const T*>(p.Lt);
  const T* U = reinterpret_cast<const T*>(p.U) + p.t0 * p.ldu;
  for (int idx = threadIdx.x; idx < q * ROWS; idx += NT) {
    const int s = idx / ROWS, r = idx % ROWS;
    sm.Ls[s][r] = (row0 + r < n) ? Lt[(p.t0 + s) * n + row0 + r] : S::zero();
  }
  const long long myrow0 = row0 + ty * RPT;
  const int nr = (int)max(0LL, min((long long)RPT, n - myrow0));
  const long long mv = (m / VEC) * VEC;
  const long long nchunks = (mv + CW - 1) / CW;

  auto issue = [&](long long c, int buf) {
    const long long l = c * CW + (long long)tx * VEC;
    if (l < mv) {
#pragma unroll
      for (int r = 0; r < RPT; ++r)
        if (r < nr) cp_async16(&sm.Rs[buf][ty * RPT + r][tx], R + (myrow0 + r) * ld + l);
    }
    for (int idx = threadIdx.x; idx < q * TX; idx += NT) {
      const int s = idx / TX, v = idx % TX;
      const long long lc = c * CW + (long long)v * VEC;
      if (lc < mv) cp_async16(&sm.Us[buf][s][v], U + s * p.ldu + lc);
    }
    cp_async_commit();
  };

  double acc[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) acc[r] = 0.0;
  if (nchunks > 0) issue(0, 0);
  for (long long c = 0; c < nchunks; ++c) {
    const int buf = (int)(c & 1);
    __syncthreads();  // every thread is done reading buffer buf^1 (chunk c-1)
    if (c + 1 < nchunks) {
      issue(c + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // chunk c (R rows and the shared U chunk) has landed
    const long long l = c * CW + (long long)tx * VEC;
    if (l < mv) {
      VecT<T, VEC> rv[RPT];
#pragma unroll
      for (int r = 0; r < RPT; ++r) rv[r] = sm.Rs[buf][ty * RPT + r][tx];
      auto term = [&](int s) {
        const VecT<T, VEC> u = sm.Us[buf][s][tx];
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const T lv = sm.Ls[s][ty * RPT + r];
#pragma unroll
          for (int e = 0; e < VEC; ++e) rv[r].v[e] = pend_sub<T>(p.fused, rv[r].v[e], lv, u.v[e]);
        }
      };
      if constexpr (QC > 0) {
#pragma unroll
        for (int s = 0; s < QC; ++s) term(s);
      } else {
        for (int s = 0; s < q; ++s) term(s);
      }
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        if (r < nr) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[r] += S::mass(rv[r].v[e]);
          if (FLUSH) *reinterpret_cast<VecT<T, VEC>*>(R + (myrow0 + r) * ld + l) = rv[r];
        }
      }
    }
  }
  for (long long l = mv + tx; l < m; l += TX) {  // scalar tail (m % VEC columns)
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      if (r < nr) {
        T x = R[(myrow0 + r) * ld + l];
        for (int s = 0; s < q; ++s) x = pend_sub<T>(p.fused, x, sm.Ls[s][ty * RPT + r], U[s * p.ldu + l]);
        acc[r] += S::mass(x);
        if (FLUSH) R[(myrow0 + r) * ld + l] = x;
      }
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const double sv = warp_sum(acc[r]);
    if (lane == 0) sm.red[w][r] = sv;
  }
  __syncthreads();
  if (threadIdx.x < ROWS) {
    const int g = threadIdx.x / RPT, r = threadIdx.x % RPT;
    if (row0 + threadIdx.x < n) p.masses[row0 + threadIdx.x] = sm.red[2 * g][r] + sm.red[2 * g + 1][r];
  }
}

// ---------------------------------------------------------------------------
// Shared-memory-resident loop for small residuals (C1: 2000^2 fp64 = 32 MB =
// 148 SMs x 216 KB): the whole elimination is ONE cooperative launch of one
// 1024-thread CTA per SM, and each CTA keeps its contiguous block of rows of
// R in shared memory for the whole run, so a pivot step moves no residual
// bytes through L2 or HBM at all.  Per step:
//   1. every CTA draws the row from the n masses (identical code and data:
//      identical draws everywhere; CTA 0 alone writes the outputs);
//   2. the CTA holding row i writes it to U[t,:] (an output anyway) and
//      publishes it with a release counter; the others acquire it;
//   3. every CTA draws the column from U[t,:] and updates its own rows in
//      shared memory (pivot-column entries captured first), leaving the
//      masses of R^(t+1) in a double-buffered global array;
//   4. one grid barrier.
// R is written back once, after the last step.  The CDF uses the same
// 1024-thread layout as dense_select_kernel; masses are summed in a fixed
// order (per-thread vector, warp tree, 32 warps in order).
struct ResidentLayout {
  int rows;     // rows per CTA (max)
  size_t off_l, off_red, bytes;
};
template <typename T>
__host__ __device__ inline ResidentLayout resident_layout(long long n, long long ld, int grid) {
  ResidentLayout L;
  L.rows = (int)((n + grid - 1) / grid);
  const size_t rbytes = (size_t)L.rows * (size_t)ld * sizeof(T);
  L.off_l = (rbytes + 15) & ~size_t(15);
  L.off_red = (L.off_l + sizeof(T) * L.rows + 15) & ~size_t(15);
  L.bytes = L.off_red + sizeof(double) * 32 * L.rows;
  return L;
}

template <typename T>
__global__ void __launch_bounds__(1024, 1)
    dense_resident_kernel(DenseParams p, double* masses2, unsigned* sync, long long* trace) {
  using S = Scalar<T>;
  constexpr int B = 1024, VEC = S::kVec, NW = B / 32;
  using V = VecT<T, VEC>;
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ CdfSmem<B> sm;
  __shared__ int s_stop;
  DevState* st = p.st;
  const bool lead = blockIdx.x == 0;
  const unsigned G = gridDim.x;
  const long long n = p.n, m = p.m, ld = p.ld;
  const ResidentLayout lay = resident_layout<T>(n, ld, (int)G);
  T* Rs = reinterpret_cast<T*>(dsm);  // [rows][ld]
  T* lvals = reinterpret_cast<T*>(dsm + lay.off_l);
  double* red = reinterpret_cast<double*>(dsm + lay.off_red);  // [NW][rows]
  T* R = reinterpret_cast<T*>(p.R);
  T* Lt = reinterpret_cast<T*>(p.Lt);
  const long long r0 = (long long)blockIdx.x * lay.rows;
  const int nr = (int)max(0LL, min((long long)lay.rows, n - r0));
  double* mbuf[2] = {p.masses, masses2};
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long ldv = ld / VEC;  // 16-byte vectors per row (ld is a multiple of VEC)
  const int tv = threadIdx.x;      // this thread's column vector (m <= 1024 * VEC)
  const bool has_v = (long long)tv * VEC < m;

  // load the block's rows (16-byte vectors)
  for (long long k = threadIdx.x; k < (long long)nr * ldv; k += B)
    reinterpret_cast<V*>(Rs)[k] = reinterpret_cast<const V*>(R + r0 * ld)[k];
  __syncthreads();

  // masses of the block's rows (with the update of step t when upd)
  // The 32 lanes' partial masses of 16 rows are reduced by recursive halving
  // (16 shuffles + 16 adds per lane instead of 16 separate warp trees); lane
  // 2q ends with the warp's sum for row q of the chunk.
  auto rows_pass = [&](bool upd, const V& pv, double* mout) {
    for (int c0 = 0; c0 < nr; c0 += 16) {
      double c[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        c[r] = 0.0;
        if (c0 + r < nr && has_v) {
          V x = reinterpret_cast<V*>(Rs + (long long)(c0 + r) * ld)[tv];
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            if ((long long)tv * VEC + e < m) {
              if (upd) x.v[e] = S::sub_outer(x.v[e], lvals[c0 + r], pv.v[e]);
              c[r] += S::mass(x.v[e]);
            }
          }
          if (upd) reinterpret_cast<V*>(Rs + (long long)(c0 + r) * ld)[tv] = x;
        }
      }
#pragma unroll
      for (int h = 8, o = 16; h >= 1; h >>= 1, o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < h; ++k) {
          const double send = up ? c[k] : c[k + h];
          const double keep = up ? c[k + h] : c[k];
          c[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      c[0] += __shfl_xor_sync(0xffffffffu, c[0], 1);
      const int q = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 +
                    ((lane >> 1) & 1);
      if ((lane & 1) == 0 && c0 + q < nr) red[w * lay.rows + c0 + q] = c[0];
    }
    __syncthreads();
    for (int r = w; r < nr; r += NW) {  // row r: the 32 warp sums, one per lane
      const double sv = warp_sum(red[lane * lay.rows + r]);
      if (lane == 0) mout[r0 + r] = sv;
    }
  };

  unsigned nbar = 0;
  rows_pass(false, V{}, mbuf[0]);
  grid_barrier(sync, G * (++nbar));

  long long uc = 0, near = 0;
  double fro0 = 0.0;
  auto mark = [&](long long t, int k) {  // phase timestamps (diagnostics only)
    if (trace && lead && threadIdx.x == 0 && t < 1024) {
      long long v;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
      trace[8 * t + k] = v;
    }
  };
  for (long long t = 0;; ++t) {
    mark(t, 0);
    const bool pre = p.rule == RPLU_RULE_RPLU && uc + 2 <= p.n_uniforms;
    const double u1p = pre ? p.uniforms[uc] : 0.0, u2p = pre ? p.uniforms[uc + 1] : 0.0;
    const double* masses = mbuf[t & 1];
    auto wrow = [&](long long k) { return __ldcg(masses + k); };
    Cdf<B> cr = cdf_build<B>(wrow, n, sm);
    mark(t, 4);
    const double total = cr.total;
    const double resid = sqrt(total);
    if (t == 0) fro0 = resid;
    if (threadIdx.x == 0) {
      int stop = 0, status = kRunning;
      if (t > 0 && p.stop_tol > 0.0 && resid <= p.stop_tol * fro0) {
        status = kTolStop;
        stop = 1;
      } else if (t >= p.steps) {
        stop = 1;
      } else if (resid == 0.0) {
        status = kCleanStop;
        stop = 1;
      }
      if (lead) {
        p.resid[t] = resid;
        if (t == 0) st->fro0 = resid;
        if (stop) {
          st->status = status;
          st->active = 0;
          st->ucount = uc;
          st->near_boundary = near;
        }
      }
      s_stop = stop;
    }
    __syncthreads();
    if (s_stop) break;

    T* urow = reinterpret_cast<T*>(p.U) + t * p.ldu;
    long long i = 0, j = 0;
    T a = S::zero();
    V pv{};
    bool fail = false;
    for (int attempt = 0; attempt < 2; ++attempt) {
      double u2 = 0.0;
      if (p.rule == RPLU_RULE_RPLU) {
        if (uc + 2 > p.n_uniforms) {
          if (lead && threadIdx.x == 0) {
            st->status = kUniformsExhausted;
            st->active = 0;
            st->ucount = uc;
            st->near_boundary = near;
          }
          fail = true;
          break;
        }
        const double u1 = attempt == 0 ? u1p : p.uniforms[uc];
        u2 = attempt == 0 ? u2p : p.uniforms[uc + 1];
        uc += 2;
        i = cdf_find<B>(wrow, n, cr, u1, sm);
        if (threadIdx.x == 0) {
          const double tol = kNearBoundaryRel * total, tg = u1 * total;
          if (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) near++;
        }
      } else {
        i = block_argmax<B>(wrow, n, nullptr);
      }
      mark(t, 5);
      // the holder of row i publishes it as U[t,:]; the others acquire it
      const unsigned seq = (unsigned)(2 * t + attempt + 1);
      if (i >= r0 && i < r0 + nr) {
        const T* src = Rs + (i - r0) * ld;
        for (long long k = threadIdx.x; k < m; k += B) urow[k] = src[k];
        __syncthreads();
        if (threadIdx.x == 0) {
          __threadfence();
          st_release_u32(sync + 1, seq);
        }
      } else {
        if (threadIdx.x == 0) wait_count(sync + 1, seq);
        __syncthreads();
      }
      mark(t, 6);
      if (has_v) {  // this thread's slice of the pivot row, for the update
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          pv.v[e] = ((long long)tv * VEC + e < m) ? __ldcg(urow + (long long)tv * VEC + e) : S::zero();
      }
      if (p.rule == RPLU_RULE_RPLU) {
        auto wcol = [&](long long k) { return S::weight(__ldcg(urow + k)); };
        Cdf<B> cc = cdf_build<B>(wcol, m, sm);
        mark(t, 7);
        j = cdf_find<B>(wcol, m, cc, u2, sm);
        if (threadIdx.x == 0) {
          const double tol = kNearBoundaryRel * cc.total, tg = u2 * cc.total;
          if (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) near++;
        }
      } else {
        auto wabs = [&](long long k) { return S::absval(__ldcg(urow + k)); };
        j = block_argmax<B>(wabs, m, nullptr);
      }
      a = __ldcg(urow + j);
      if (!S::is_zero(a)) break;
      if (attempt == 1 || p.rule != RPLU_RULE_RPLU) {
        if (lead && threadIdx.x == 0) {
          st->status = kZeroPivot;
          st->active = 0;
          st->err_i = i;
          st->err_j = j;
          st->ucount = uc;
          st->near_boundary = near;
        }
        fail = true;
        break;
      }
      __syncthreads();
    }
    if (fail) break;
    mark(t, 1);
    if (lead && threadIdx.x == 0) {
      st->pi = i;
      st->pj = j;
      store_coef<T>(st, a);
      p.pivots[2 * t] = i;
      p.pivots[2 * t + 1] = j;
      st->done = t + 1;
    }
    // pivot-column entries of the block's rows, before any row is written
    const typename S::coef_t cf = S::make_coef(a);
    if (threadIdx.x < nr) {
      const T lv = S::scale(Rs[(long long)threadIdx.x * ld + j], cf);
      lvals[threadIdx.x] = lv;
      Lt[t * n + r0 + threadIdx.x] = lv;
    }
    __syncthreads();
    rows_pass(true, pv, mbuf[(t + 1) & 1]);
    mark(t, 2);
    grid_barrier(sync, G * (++nbar));
    mark(t, 3);
  }
  // the residual R^(k) back to HBM
  __syncthreads();
  for (long long k = threadIdx.x; k < (long long)nr * ldv; k += B)
    reinterpret_cast<V*>(R + r0 * ld)[k] = reinterpret_cast<const V*>(Rs)[k];
}

// ---------------------------------------------------------------------------
// host-side launchers

__global__ void init_state_kernel(DevState* st) {
  st->ucount = 0;
  st->near_boundary = 0;
  st->pi = st->pj = -1;
  st->err_i = st->err_j = -1;
  st->active = 1;
  st->status = kRunning;
  st->fro0 = 0.0;
  st->done = 0;
}

template <typename T, int VEC, int RB>
static void launch_sweep(const DenseParams& p, bool update, bool track, cudaStream_t s) {
  dim3 grid((unsigned)((p.n + RB - 1) / RB));
  if (update) {
    if (track) dense_sweep_kernel<T, VEC, RB, true, true><<<grid, 256, 0, s>>>(p);
    else dense_sweep_kernel<T, VEC, RB, true, false><<<grid, 256, 0, s>>>(p);
  } else {
    if (track) dense_sweep_kernel<T, VEC, RB, false, true><<<grid, 256, 0, s>>>(p);
    else dense_sweep_kernel<T, VEC, RB, false, false><<<grid, 256, 0, s>>>(p);
  }
}

// K3 variant for experiments (RPLU_SWEEP_VARIANT, read once): 0 = 4 rows per
// CTA (default), 1 = 4 rows + streaming hints, 2 = 8 rows, 3 = 2 rows,
// 4 = 8 rows + streaming hints.  Only the vectorised update path varies.
static int sweep_variant() {
  static int v = [] {
    const char* e = getenv("RPLU_SWEEP_VARIANT");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <typename T, int VEC, int RB, bool STREAM>
static void launch_update_variant(const DenseParams& p, cudaStream_t s) {
  dim3 grid((unsigned)((p.n + RB - 1) / RB));
  dense_sweep_kernel<T, VEC, RB, true, false, STREAM><<<grid, 256, 0, s>>>(p);
}

template <typename T>
static void sweep(const DenseParams& p, bool update, bool track, cudaStream_t s) {
  constexpr int VEC = Scalar<T>::kVec;
  bool vec_ok = (p.ld % VEC == 0) && ((uintptr_t)p.R % 16 == 0) &&
                (!update || ((p.ldu % VEC == 0) && ((uintptr_t)p.U % 16 == 0)));
  if (vec_ok && update && !track) {
    switch (sweep_variant()) {
      case 1: launch_update_variant<T, VEC, 4, true>(p, s); return;
      case 2: launch_update_variant<T, VEC, 8, false>(p, s); return;
      case 3: launch_update_variant<T, VEC, 2, false>(p, s); return;
      case 4: launch_update_variant<T, VEC, 8, true>(p, s); return;
      default: break;
    }
  }
  if (vec_ok) launch_sweep<T, VEC, 4>(p, update, track, s);
  else launch_sweep<T, 1, 4>(p, update, track, s);
}

struct LoopTiming {
  bool on = false;
  std::vector<cudaEvent_t> ev;  // pairs (start, end) per timed launch
  std::vector<int> kind;        // 0 = select, 1 = sweep
  ~LoopTiming() {
    for (auto e : ev) cudaEventDestroy(e);
  }
  void mark(int k, cudaStream_t s, bool start) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back(e);
    if (start) kind.push_back(k);
  }
};

template <typename T>
static int dense_loop(const DenseParams& base, cudaStream_t s, LoopTiming& tm, long long* launches) {
  DenseParams p = base;
  const bool track = (p.rule == RPLU_RULE_CPLU);
  sweep<T>(p, false, track, s);  // K1: masses of A
  RPLU_CUDA(cudaGetLastError());
  long long nl = 1;
  for (long long t = 0; t <= p.steps; ++t) {
    p.t = t;
    tm.mark(0, s, true);
    dense_select_kernel<T><<<1, 1024, 0, s>>>(p);
    tm.mark(0, s, false);
    ++nl;
    if (t < p.steps) {
      tm.mark(1, s, true);
      sweep<T>(p, true, track, s);
      tm.mark(1, s, false);
      ++nl;
    }
  }
  RPLU_CUDA(cudaGetLastError());
  *launches = nl;
  return RPLU_OK;
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

static int sm_count() {
  static int c = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return c;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// libcuda link dependency).
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// 2-D map over a row-major (rows x cols) array of element size esize with a
// row pitch of ld elements; box = 1 KB of columns x box_rows rows.
static bool make_row_map(CUtensorMap* map, const void* base, int esize, long long rows,
                         long long cols, long long ld, int box_rows, int box_bytes = 1024) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const int w = esize == 4 ? 4 : 8;  // complex128 = pairs of fp64 words
  const int per = esize / w;
  const cuuint64_t dims[2] = {(cuuint64_t)(cols * per), (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)(ld * esize)};
  const cuuint32_t box[2] = {(cuuint32_t)(box_bytes / w), (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, w == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
             const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, bool FLUSH, int QC, int TXW, bool FUSED, bool DOT = false>
static int launch_lazy_pass4_w(const DenseParams& p, cudaStream_t s) {
  constexpr int VEC = Scalar<T>::kVec;
  using C = LazyTma<T, QC, TXW>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(lazy_pass4_kernel<T, VEC, FLUSH, QC, TXW, FUSED, DOT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    attr = true;
  }
  // rows per work item: the count that minimises waves x rows on the
  // persistent CTAs (ties keep the larger item); RPLU_PASS_ROWS overrides
  static const int rows_env = env_int("RPLU_PASS_ROWS", 0);
  int rb_rows = C::ROWS;
  if (rows_env >= 8 && rows_env <= C::ROWS) {
    rb_rows = rows_env;
  } else {
    long long best = -1;
    for (int r = C::ROWS; r >= C::ROWS - 8; --r) {
      const long long items = (p.n + r - 1) / r;
      const long long cost = ((items + sm_count() - 1) / sm_count()) * r;
      if (best < 0 || cost < best) { best = cost; rb_rows = r; }
    }
  }
  DenseParams pp = p;
  pp.pass_rows = rb_rows;
  const long long nblocks = (p.n + rb_rows - 1) / rb_rows;
  const long long g = nblocks < sm_count() ? nblocks : sm_count();
  if (g <= 0 || p.m <= 0) return RPLU_OK;
  CUtensorMap tmR, tmU;
  const long long urows = p.rel ? p.u_rows : p.t0 + QC;  // U rows 0 .. t0+QC-1 exist
  if (!make_row_map(&tmR, p.R, (int)sizeof(T), p.n, p.m, p.ld, rb_rows, C::LINE) ||
      !make_row_map(&tmU, p.U, (int)sizeof(T), urows, p.m, p.ldu, QC, C::LINE)) {
    set_error("cuTensorMapEncodeTiled failed for the delayed-update pass");
    return RPLU_ERR_CUDA;
  }
  lazy_pass4_kernel<T, VEC, FLUSH, QC, TXW, FUSED, DOT><<<(unsigned)g, 288, C::SMEM, s>>>(pp, tmR,
                                                                                       tmU);
  return RPLU_OK;
}

// (16 rows x 2 KB stages, TXW = 128, were measured no faster than 32 rows x
// 1 KB at C3 fp64: 623 vs 627 steps/s at b = 6)
template <typename T, bool FLUSH, int QC>
static int launch_lazy_pass4_q(const DenseParams& p, cudaStream_t s) {
  if (p.fused) return launch_lazy_pass4_w<T, FLUSH, QC, 64, true>(p, s);
  return launch_lazy_pass4_w<T, FLUSH, QC, 64, false>(p, s);
}

template <typename T, bool FLUSH>
static int launch_lazy_pass4_f(const DenseParams& p, cudaStream_t s) {
  static_assert(kLazyMaxBlock == 16, "one instantiation per pending-term count");
  switch ((int)(p.t - p.t0 + 1)) {
    case 1: return launch_lazy_pass4_q<T, FLUSH, 1>(p, s);
    case 2: return launch_lazy_pass4_q<T, FLUSH, 2>(p, s);
    case 3: return launch_lazy_pass4_q<T, FLUSH, 3>(p, s);
    case 4: return launch_lazy_pass4_q<T, FLUSH, 4>(p, s);
    case 5: return launch_lazy_pass4_q<T, FLUSH, 5>(p, s);
    case 6: return launch_lazy_pass4_q<T, FLUSH, 6>(p, s);
    case 7: return launch_lazy_pass4_q<T, FLUSH, 7>(p, s);
    case 8: return launch_lazy_pass4_q<T, FLUSH, 8>(p, s);
    case 9: return launch_lazy_pass4_q<T, FLUSH, 9>(p, s);
    case 10: return launch_lazy_pass4_q<T, FLUSH, 10>(p, s);
    case 11: return launch_lazy_pass4_q<T, FLUSH, 11>(p, s);
    case 12: return launch_lazy_pass4_q<T, FLUSH, 12>(p, s);
    case 13: return launch_lazy_pass4_q<T, FLUSH, 13>(p, s);
    case 14: return launch_lazy_pass4_q<T, FLUSH, 14>(p, s);
    case 15: return launch_lazy_pass4_q<T, FLUSH, 15>(p, s);
    default: return launch_lazy_pass4_q<T, FLUSH, 16>(p, s);
  }
}

template <typename T, int RPT, bool FLUSH, int QC>
static void launch_lazy_pass3_q(const DenseParams& p, cudaStream_t s) {
  constexpr int VEC = Scalar<T>::kVec;
  using SM = LazyPipeSmem<T, VEC, RPT>;
  const int smem = (int)sizeof(SM);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(lazy_pass3_kernel<T, VEC, RPT, FLUSH, QC>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((unsigned)((p.n + SM::ROWS - 1) / SM::ROWS));
  lazy_pass3_kernel<T, VEC, RPT, FLUSH, QC><<<grid, 256, smem, s>>>(p);
}

template <typename T>
static int lazy_pass(const DenseParams& p, bool flush, cudaStream_t s) {
  // RPLU_LAZY_KERNEL=3: the round-1 cp.async double-buffered pass (one
  // instantiation, runtime q; experiments only); default 4: TMA-fed pass
  static const int kernel = env_int("RPLU_LAZY_KERNEL", 4);
  constexpr int RPT3 = sizeof(T) == 16 ? 2 : 8;
  if (kernel == 3) {
    if (flush) launch_lazy_pass3_q<T, RPT3, true, 0>(p, s);
    else launch_lazy_pass3_q<T, RPT3, false, 0>(p, s);
    return RPLU_OK;
  }
  return flush ? launch_lazy_pass4_f<T, true>(p, s) : launch_lazy_pass4_f<T, false>(p, s);
}

// Default flush interval, from the measured per-q pass times of the TMA-fed
// pass at C3 (profiles/r01/pass4_q_launches_summary.txt): a read pass is
// HBM-bound at ~1.19 ms up to q ~ 5 pending terms, then FP64-bound at ~0.115
// ms per term (2 FP64 operations per element and term, 76% of the FP64
// pipe), while a flush costs ~2.9 ms; the per-step minimum is at b = 7..8
// for fp64 at full clocks (646 / 650 steps/s, 642 at 6) and at b = 6 on the
// boxes whose power cap held the SMs at ~1.45 GHz (624-627 vs 619-622 at 7-8):
// with b = 6 every read pass stays HBM-bound (q <= 5), so 6 is the default;
// 6 for fp32 and 5 for complex128 (profiles/r01/sweep_lazy_block_*.txt).
// RPLU_LAZY_BLOCK overrides.
// With fused pending terms (one FMA per term, the default) a read pass
// stays HBM-bound to about twice as many terms, so the flush interval is
// longer (RPLU_LAZY_BLOCK_FUSED overrides; profiles/r02/sweep_lazy_block_fused_*.txt).
template <typename T>
static int lazy_block(bool fused) {
  const int dflt = fused ? (sizeof(T) == 16 ? 8 : 12)
                         : (sizeof(T) == 16 ? 5 : (sizeof(T) == 4 ? 6 : 6));
  int b = fused ? env_int("RPLU_LAZY_BLOCK_FUSED", env_int("RPLU_LAZY_BLOCK", dflt))
                : env_int("RPLU_LAZY_BLOCK", dflt);
  return b < 1 ? 1 : (b > kLazyMaxBlock ? kLazyMaxBlock : b);
}

// One Gram-mass step (fp64): U_t . U_s for the pending s, then the read pass
// g_i = r0_i . U_t with the mass update (the TMA map loads U row t).
template <typename T>
static int gram_step(const DenseParams& p, long long t0, cudaStream_t s) {
  if constexpr (std::is_same<T, double>::value) {
    DenseParams q = p;
    q.gram_t0 = t0;
    lazy_gram_kernel<<<(unsigned)(p.t - t0 + 1), 1024, 0, s>>>(q);
    q.t0 = p.t;  // the pass's one "pending" U row is U_t
    return launch_lazy_pass4_w<double, false, 1, 64, false, true>(q, s);
  } else {
    set_error("Gram-mass delayed updates are fp64 only");
    return RPLU_ERR_ARG;
  }
}

// Flush interval of the Gram-mass loop: the read passes cost the same for
// every q, so the longest block (16) minimises the flushes
// (RPLU_LAZY_BLOCK_GRAM overrides).
static int gram_block() {
  const int b = env_int("RPLU_LAZY_BLOCK_GRAM", kLazyMaxBlock);
  return b < 1 ? 1 : (b > kLazyMaxBlock ? kLazyMaxBlock : b);
}

template <typename T>
static int dense_loop_lazy(const DenseParams& base, cudaStream_t s, LoopTiming& tm,
                           long long* launches) {
  DenseParams p = base;
  p.lazy = 1;
  const int block = p.gram ? gram_block() : lazy_block<T>(p.fused != 0);
  sweep<T>(p, false, false, s);  // K1: masses of A
  RPLU_CUDA(cudaGetLastError());
  const int reset_blocks = (int)std::min<long long>((p.n + 255) / 256, 1024);
  if (p.gram) gram_reset_kernel<<<reset_blocks, 256, 0, s>>>(p);
  long long nl = p.gram ? 2 : 1;
  long long t0 = 0;
  const int pc_blocks = (int)((p.n + 255) / 256 < 1024 ? (p.n + 255) / 256 : 1024);
  const int row_blocks = (int)((p.m + 255) / 256 < 1024 ? (p.m + 255) / 256 : 1024);
  for (long long t = 0; t <= p.steps; ++t) {
    p.t = t;
    p.t0 = t0;
    tm.mark(0, s, true);
    lazy_select_row_kernel<T><<<1, 1024, 0, s>>>(p);
    if (t < p.steps) {
      lazy_row_kernel<T><<<row_blocks, 256, 0, s>>>(p);
      lazy_select_col_kernel<T><<<1, 1024, 0, s>>>(p);
      nl += 2;
    }
    tm.mark(0, s, false);
    ++nl;
    if (t < p.steps) {
      lazy_pivcol_kernel<T><<<pc_blocks, 256, 0, s>>>(p);
      const bool flush = (t - t0 + 1 == block) || (t == p.steps - 1);
      tm.mark(flush ? 2 : 1, s, true);
      if (!flush && p.gram) {
        if (int rc = gram_step<T>(p, t0, s)) return rc;
        ++nl;
      } else {
        if (int rc = lazy_pass<T>(p, flush, s)) return rc;
      }
      tm.mark(flush ? 2 : 1, s, false);
      nl += 2;
      if (flush) {
        t0 = t + 1;
        if (p.gram) {
          gram_reset_kernel<<<reset_blocks, 256, 0, s>>>(p);
          ++nl;
        }
      }
    }
  }
  RPLU_CUDA(cudaGetLastError());
  *launches = nl;
  return RPLU_OK;
}

// After an early stop the residual holds R^(t0) of the last flush; apply
// the pending steps t0..done-1 (no-op when the loop ran to the end).
template <typename T>
static int lazy_final_flush(const DenseParams& base, long long done, cudaStream_t s) {
  const long long block = base.gram ? gram_block() : lazy_block<T>(base.fused != 0);
  const long long t0 = (done / block) * block;
  if (done <= t0 || done >= base.steps) return RPLU_OK;
  DenseParams p = base;
  p.lazy = 1;
  p.force = 1;
  p.t = done - 1;
  p.t0 = t0;
  if (int rc = lazy_pass<T>(p, true, s)) return rc;
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

// Shared-memory bytes the resident loop needs for this residual (0: the
// residual does not fit in the SMs' shared memory or a row is too long).
template <typename T>
static size_t resident_bytes(long long n, long long m, long long ld) {
  if (m > 1024LL * Scalar<T>::kVec || n <= 0) return 0;
  static const size_t cap = [] {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, dense_resident_kernel<T>);
    const long long c = (long long)optin - (long long)fa.sharedSizeBytes - 1024;
    return (size_t)(c > 0 ? c : 0);
  }();
  const ResidentLayout L = resident_layout<T>(n, ld, sm_count());
  return L.bytes <= cap ? L.bytes : 0;
}

template <typename T>
static int launch_persistent(rplu_ctx* ctx, const DenseParams& p, cudaStream_t s,
                             cudaEvent_t* ev) {
  auto kern = dense_resident_kernel<T>;
  const int smem = (int)resident_bytes<T>(p.n, p.m, p.ld);
  static int attr_smem = -1;
  if (smem > attr_smem) {
    RPLU_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_smem = smem;
  }
  int per_sm = 0;
  RPLU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 1024, smem));
  if (per_sm < 1) {
    set_error("shared-memory-resident dense loop does not fit on an SM");
    return RPLU_ERR_CUDA;
  }
  int rc;
  if ((rc = ctx->masses2.ensure(sizeof(double) * (size_t)(p.n > 0 ? p.n : 1)))) return rc;
  if ((rc = ctx->gbar.ensure(2 * sizeof(unsigned)))) return rc;
  RPLU_CUDA(cudaMemsetAsync(ctx->gbar.ptr, 0, 2 * sizeof(unsigned), s));
  DenseParams q = p;
  double* m2 = reinterpret_cast<double*>(ctx->masses2.ptr);
  unsigned* sync = reinterpret_cast<unsigned*>(ctx->gbar.ptr);
  // RPLU_PERSIST_TRACE=1: CTA 0's phase timestamps of the first 1024 steps
  // (draws / update / barrier), printed to stderr (diagnostics)
  static const bool tracing = getenv("RPLU_PERSIST_TRACE") != nullptr;
  long long* trace = nullptr;
  if (tracing) {
    RPLU_CUDA(cudaMalloc(&trace, sizeof(long long) * 8 * 1024));
    RPLU_CUDA(cudaMemsetAsync(trace, 0, sizeof(long long) * 8 * 1024, s));
  }
  void* args[] = {&q, &m2, &sync, &trace};
  const unsigned grid = (unsigned)sm_count();
  if (ev[0]) RPLU_CUDA(cudaEventRecord(ev[0], s));
  RPLU_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(1024), args,
                                        (size_t)smem, s));
  if (ev[1]) RPLU_CUDA(cudaEventRecord(ev[1], s));
  if (tracing) {
    std::vector<long long> h(8 * 1024);
    RPLU_CUDA(cudaMemcpyAsync(h.data(), trace, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, s));
    RPLU_CUDA(cudaStreamSynchronize(s));
    cudaFree(trace);
    // 0 start, 4 row CDF built, 5 row drawn, 6 pivot row published/acquired,
    // 7 column CDF built, 1 column drawn, 2 rows updated, 3 barrier passed
    const int order[8] = {0, 4, 5, 6, 7, 1, 2, 3};
    const char* names[7] = {"row cdf", "row find", "publish", "col cdf", "col find", "update", "barrier"};
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    long long k = 0;
    for (; k < 1024 && h[8 * k + 3] != 0; ++k)
      for (int q = 0; q < 7; ++q) acc[q] += (double)(h[8 * k + order[q + 1]] - h[8 * k + order[q]]);
    if (k > 0) {
      fprintf(stderr, "[rplu] resident loop, CTA 0, %lld steps (us/step):", k);
      for (int q = 0; q < 7; ++q) fprintf(stderr, " %s %.2f", names[q], acc[q] / k / 1e3);
      fprintf(stderr, "\n");
    }
  }
  return RPLU_OK;
}

int dense_run_impl(rplu_ctx* ctx, const rplu_dense_args* a, rplu_dense_out* out) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(a->stream);
  const long long n = a->n, m = a->m, steps = a->steps;
  int rc;
  if ((rc = ctx->state.ensure(sizeof(DevState)))) return rc;
  if ((rc = ctx->masses.ensure(sizeof(double) * (size_t)(n > 0 ? n : 1)))) return rc;
  if ((rc = ctx->pivots.ensure(sizeof(long long) * (size_t)(2 * steps + 2)))) return rc;
  if ((rc = ctx->resid.ensure(sizeof(double) * (size_t)(steps + 1)))) return rc;
  if (a->rule == RPLU_RULE_CPLU) {
    if ((rc = ctx->rowmax.ensure(sizeof(double) * (size_t)n))) return rc;
    if ((rc = ctx->rowarg.ensure(sizeof(long long) * (size_t)n))) return rc;
  }
  long long nu = (a->rule == RPLU_RULE_RPLU) ? a->n_uniforms : 0;
  if ((rc = ctx->uniforms.ensure(sizeof(double) * (size_t)(nu > 0 ? nu : 1)))) return rc;
  if (nu > 0)
    RPLU_CUDA(cudaMemcpyAsync(ctx->uniforms.ptr, a->uniforms, sizeof(double) * nu,
                              cudaMemcpyHostToDevice, s));
  DevState* st = reinterpret_cast<DevState*>(ctx->state.ptr);

  DenseParams p{};
  p.R = a->R;
  p.ld = a->ld;
  p.n = n;
  p.m = m;
  p.Lt = a->Lt;
  p.U = a->U;
  p.ldu = a->ldu;
  p.masses = reinterpret_cast<double*>(ctx->masses.ptr);
  p.rowmax = reinterpret_cast<double*>(ctx->rowmax.ptr);
  p.rowarg = reinterpret_cast<long long*>(ctx->rowarg.ptr);
  p.st = st;
  p.steps = steps;
  p.uniforms = reinterpret_cast<const double*>(ctx->uniforms.ptr);
  p.n_uniforms = nu;
  p.resid = reinterpret_cast<double*>(ctx->resid.ptr);
  p.pivots = reinterpret_cast<long long*>(ctx->pivots.ptr);
  p.stop_tol = a->stop_tol;
  p.rule = a->rule;
  p.fused = (a->flags & RPLU_FLAG_EXACT) ? 0 : 1;  // delayed-update loop only
  // Gram masses for the fp64 delayed-update loop with the reference's
  // arithmetic (RPLU_GRAM=0 disables)
  static const int gram_env = env_int("RPLU_GRAM", 1);
  if (gram_env && a->dtype == RPLU_F64 && !p.fused && !(a->flags & RPLU_FLAG_NO_GRAM)) {
    if ((rc = ctx->gram.ensure(sizeof(double) * (3 * (size_t)(n > 0 ? n : 1) + 256))))
      return rc;
    double* gb = reinterpret_cast<double*>(ctx->gram.ptr);
    p.m0 = gb;
    p.lin = gb + n;
    p.quad = gb + 2 * n;
    p.gmat = gb + 3 * n;
    p.gram = 1;
  }

  LoopTiming tm;
  tm.on = (a->flags & RPLU_FLAG_TIME_KERNELS) != 0;
  long long launches = 0;
  // Small residuals (per-step GPU time of a few microseconds) are host-launch
  // bound: enqueue the whole loop as one CUDA graph.
  // (per-kernel CUDA-event timing needs plain stream launches: events
  // recorded by graph nodes cannot be timed)
  static const int graph_env = [] {  // RPLU_GRAPH=always|never (experiments)
    const char* e = getenv("RPLU_GRAPH");
    if (!e) return 0;
    return e[0] == 'a' ? 1 : (e[0] == 'n' ? -1 : 0);
  }();
  const bool small = (double)n * (double)m <= 64.0 * 1024 * 1024;
  const bool graph = (a->flags & (RPLU_FLAG_NO_GRAPH | RPLU_FLAG_TIME_KERNELS)) == 0 &&
                     steps >= 4 && graph_env >= 0 && (small || graph_env > 0);
  // Residuals that do not fit in L2 take the delayed-update loop (one read
  // of R per step instead of read + write); RPLU_LAZY=0/1 overrides.
  const int esize = a->dtype == RPLU_F32 ? 4 : (a->dtype == RPLU_F64 ? 8 : 16);
  const int vec = 16 / esize;
  const bool vec_ok = (a->ld % vec == 0) && ((uintptr_t)a->R % 16 == 0) &&
                      (a->ldu % vec == 0) && ((uintptr_t)a->U % 16 == 0);
  static const int lazy_env = env_int("RPLU_LAZY", -1);
  int want = -1;  // -1 auto, 0 eager, 1 lazy
  if (a->flags & RPLU_FLAG_EAGER) want = 0;
  else if (a->flags & RPLU_FLAG_LAZY) want = 1;
  else if (lazy_env >= 0) want = lazy_env;
  const bool lazy = a->rule != RPLU_RULE_CPLU && vec_ok && steps >= 2 &&
                    (want == 1 || (want < 0 && (double)n * m * esize > 256.0e6));
  // Residuals that fit in the SMs' shared memory: the whole loop as one
  // persistent cooperative launch with R resident on chip (RPLU_PERSIST=0
  // disables, for comparisons)
  static const int persist_env = env_int("RPLU_PERSIST", 1);
  size_t res_bytes = 0;
  if (!lazy && persist_env != 0 && !(a->flags & RPLU_FLAG_STEPWISE) &&
      a->rule != RPLU_RULE_CPLU && steps >= 1 && want != 1 && vec_ok) {
    switch (a->dtype) {
      case RPLU_F64: res_bytes = resident_bytes<double>(n, m, a->ld); break;
      case RPLU_F32: res_bytes = resident_bytes<float>(n, m, a->ld); break;
      case RPLU_C128: res_bytes = resident_bytes<double2>(n, m, a->ld); break;
    }
  }
  const bool persist = res_bytes > 0;
  if (persist) {
    cudaEvent_t pe[2] = {nullptr, nullptr};
    if (tm.on) {
      RPLU_CUDA(cudaEventCreate(&pe[0]));
      RPLU_CUDA(cudaEventCreate(&pe[1]));
    }
    init_state_kernel<<<1, 1, 0, s>>>(st);
    switch (a->dtype) {
      case RPLU_F64: rc = launch_persistent<double>(ctx, p, s, pe); break;
      case RPLU_F32: rc = launch_persistent<float>(ctx, p, s, pe); break;
      case RPLU_C128: rc = launch_persistent<double2>(ctx, p, s, pe); break;
      default: set_error("unknown dtype"); rc = RPLU_ERR_ARG;
    }
    if (rc) return rc;
    launches = 2;
    if (tm.on) {
      tm.ev.push_back(pe[0]);
      tm.ev.push_back(pe[1]);
      tm.kind.push_back(3);  // whole loop in one launch
    }
  } else {
  rc = run_maybe_graph(ctx, s, graph, 0, [&](cudaStream_t q) -> int {
    init_state_kernel<<<1, 1, 0, q>>>(st);
    switch (a->dtype) {
      case RPLU_F64:
        return lazy ? dense_loop_lazy<double>(p, q, tm, &launches)
                    : dense_loop<double>(p, q, tm, &launches);
      case RPLU_F32:
        return lazy ? dense_loop_lazy<float>(p, q, tm, &launches)
                    : dense_loop<float>(p, q, tm, &launches);
      case RPLU_C128:
        return lazy ? dense_loop_lazy<double2>(p, q, tm, &launches)
                    : dense_loop<double2>(p, q, tm, &launches);
    }
    set_error("unknown dtype");
    return RPLU_ERR_ARG;
  });
  if (rc) return rc;
  }

  DevState hs;
  RPLU_CUDA(cudaMemcpyAsync(&hs, st, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaStreamSynchronize(s));
  const long long done = hs.done;
  if (lazy && done < steps) {
    switch (a->dtype) {
      case RPLU_F64: rc = lazy_final_flush<double>(p, done, s); break;
      case RPLU_F32: rc = lazy_final_flush<float>(p, done, s); break;
      case RPLU_C128: rc = lazy_final_flush<double2>(p, done, s); break;
    }
    if (rc) return rc;
    RPLU_CUDA(cudaStreamSynchronize(s));
  }
  out->lazy_block = lazy ? (p.gram ? gram_block() : dense_lazy_block_default(a->dtype, p.fused != 0))
                         : 0;
  out->sweep_bytes = 0.0;
  if (done > 0)
    RPLU_CUDA(cudaMemcpy(out->pivots, p.pivots, sizeof(long long) * 2 * done,
                         cudaMemcpyDeviceToHost));
  RPLU_CUDA(cudaMemcpy(out->resid_fro, p.resid, sizeof(double) * (done + 1),
                       cudaMemcpyDeviceToHost));
  out->steps_done = done;
  out->kernel_launches = launches + 1;  // + init_state
  out->sweep_ms = out->select_ms = 0.0;
  out->sweep_launches = 0;
  if (tm.on) {
    // only launches that did work count (early-exit launches after a stop are
    // a few microseconds and are excluded from the per-launch average)
    for (size_t q = 0; q < tm.kind.size(); ++q) {
      float ms = 0.f;
      RPLU_CUDA(cudaEventElapsedTime(&ms, tm.ev[2 * q], tm.ev[2 * q + 1]));
      if (tm.kind[q] == 3) {  // persistent loop: K1 + every step's update
        out->sweep_ms += ms;
        out->sweep_launches += 1;
        out->sweep_bytes += (double)n * m * esize * (1.0 + 2.0 * (double)done);
      } else if (tm.kind[q] >= 1) {
        // algorithmic bytes: eager update and lazy flush read + write R,
        // a lazy pass reads it
        const double pass_bytes = (double)n * m * esize * ((lazy && tm.kind[q] == 1) ? 1 : 2);
        if ((long long)out->sweep_launches < done) {
          out->sweep_ms += ms;
          out->sweep_launches++;
          out->sweep_bytes += pass_bytes;
        }
      } else {
        out->select_ms += ms;
      }
    }
  }
  out->uniforms_consumed = hs.ucount;
  out->near_boundary_draws = hs.near_boundary;
  out->clean_early_stop = (hs.status == kCleanStop);
  out->tol_stop = (hs.status == kTolStop);
  out->zero_pivot_i = hs.err_i;
  out->zero_pivot_j = hs.err_j;
  return hs.status;
}

}  // namespace rplu

namespace rplu {

int row_masses_impl(rplu_ctx* ctx, int dtype, const void* R, long long n, long long m,
                    long long ld, double* masses, cudaStream_t s) {
  (void)ctx;
  if (n == 0) return RPLU_OK;
  DenseParams p{};
  p.R = const_cast<void*>(R);
  p.ld = ld;
  p.n = n;
  p.m = m;
  p.masses = masses;
  p.ldu = m;
  switch (dtype) {
    case RPLU_F64: sweep<double>(p, false, false, s); break;
    case RPLU_F32: sweep<float>(p, false, false, s); break;
    case RPLU_C128: sweep<double2>(p, false, false, s); break;
    default: set_error("unknown dtype"); return RPLU_ERR_ARG;
  }
  RPLU_CUDA(cudaGetLastError());
  RPLU_CUDA(cudaStreamSynchronize(s));
  return RPLU_OK;
}

}  // namespace rplu

// ---------------------------------------------------------------------------
// sample_index (rng.py:50-74) as a standalone device call: the same K2 CDF
// code the pivot loops use, exposed so its tie / zero / clamp semantics are
// testable against the reference on arbitrary weight vectors.
namespace rplu {

struct SampleOut {
  long long idx;
  int status;  // 0 ok, 1 negative weight, 2 all zero
  int near;
  double total;  // the CDF's total (the draw's own summation order)
};
static_assert(sizeof(SampleOut) == kSampleOutBytes, "SampleOut layout (rplu_internal.h)");

// mode 0: u in [0,1) scaled by the CDF total (sample_index); mode 1: u is an
// absolute target in [0, total] (the owner shard's draw of a sharded
// elimination); mode 2: total only.
__global__ void __launch_bounds__(1024) sample_index_kernel(const double* w, long long n, double u,
                                                            int mode, SampleOut* out) {
  constexpr int B = 1024;
  __shared__ CdfSmem<B> sm;
  __shared__ int neg;
  if (threadIdx.x == 0) neg = 0;
  __syncthreads();
  for (long long k = threadIdx.x; k < n; k += B)
    if (w[k] < 0.0) neg = 1;
  __syncthreads();
  if (neg) {
    if (threadIdx.x == 0) { out->status = 1; out->idx = -1; out->near = 0; out->total = 0.0; }
    return;
  }
  auto wf = [&](long long k) { return w[k]; };
  Cdf<B> c = cdf_build<B>(wf, n, sm);
  if (mode == 2 || !(c.total > 0.0)) {
    if (threadIdx.x == 0) {
      out->status = (mode == 2) ? 0 : 2;
      out->idx = -1;
      out->near = 0;
      out->total = c.total;
    }
    return;
  }
  const double tg = (mode == 1) ? u : u * c.total;
  long long i = cdf_find_target<B>(wf, n, c, tg, sm);
  if (threadIdx.x == 0) {
    double tol = kNearBoundaryRel * c.total;
    out->near = (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) ? 1 : 0;
    out->idx = i;
    out->status = 0;
    out->total = c.total;
  }
}

// Large-n draws (the plan path's row / column draws over 2^20 weights, the
// CUR row draws over 2e6): the single-CTA walk is latency bound (222 us at
// 2^20).  Two levels instead: chunks of kChunk weights, each chunk's total
// built by one CTA with the single-CTA CDF arithmetic (cdf_build on the
// chunk), a sequential prefix over the chunk totals, then the single-CTA
// search inside the owner chunk offset by the chunk's exclusive prefix.  The
// CDF association therefore differs from the single-CTA one for n above the
// threshold (both differ from np.cumsum only within rounding of a boundary,
// counted as near-boundary draws).
__global__ void __launch_bounds__(1024) sample_chunk_totals_kernel(const double* w, long long n,
                                                                   double* ctot, int* neg) {
  chunk_totals_block(w, n, ctot, neg);
}

__global__ void __launch_bounds__(1024) sample_chunked_kernel(const double* w, long long n,
                                                              double u, int mode,
                                                              const double* ctot, long long nch,
                                                              const int* neg, SampleOut* out) {
  __shared__ CdfSmem<1024> sm;
  if (*neg) {
    if (threadIdx.x == 0) { out->status = 1; out->idx = -1; out->near = 0; out->total = 0.0; }
    return;
  }
  double total;
  int near;
  const long long i = chunked_draw_block(w, n, u, mode, ctot, nch, sm, &total, &near);
  if (threadIdx.x == 0) {
    if (mode == 2 || !(total > 0.0)) {
      out->status = (mode == 2) ? 0 : 2;
      out->idx = -1;
      out->near = 0;
    } else {
      out->near = near;
      out->idx = i;
      out->status = 0;
    }
    out->total = total;
  }
}

// Enqueue one draw into result slot `slot` (0 or 1) of the context's sample
// scratch and return the device address of its SampleOut (no host
// synchronisation): callers chain further kernels on the drawn index and read
// everything back with one synchronisation.
static int sample_index_launch(rplu_ctx* ctx, const double* w, long long n, double u, int mode,
                               int slot, cudaStream_t s, SampleOut** dout) {
  int rc;
  const long long nch = (n + kChunk - 1) / kChunk;
  // per slot: SampleOut | neg flag (16 B) | chunk totals; slots of equal size
  const size_t per = (sizeof(SampleOut) + 16 + sizeof(double) * (size_t)nch + 63) & ~size_t(63);
  // (the scratch only grows: a later, smaller draw keeps the larger stride
  // consistent because both slots are addressed from the call's own `per`)
  if ((rc = ctx->scratch[7].ensure(2 * per))) return rc;
  char* base = reinterpret_cast<char*>(ctx->scratch[7].ptr) + (size_t)slot * per;
  SampleOut* d = reinterpret_cast<SampleOut*>(base);
  if (n >= kChunkedMinN) {
    int* neg = reinterpret_cast<int*>(base + sizeof(SampleOut));
    double* ctot = reinterpret_cast<double*>(reinterpret_cast<char*>(neg) + 16);
    RPLU_CUDA(cudaMemsetAsync(neg, 0, sizeof(int), s));
    count_launches(2);
    sample_chunk_totals_kernel<<<(unsigned)nch, 1024, 0, s>>>(w, n, ctot, neg);
    sample_chunked_kernel<<<1, 1024, 0, s>>>(w, n, u, mode, ctot, nch, neg, d);
  } else {
    count_launches(1);
    sample_index_kernel<<<1, 1024, 0, s>>>(w, n, u, mode, d);
  }
  RPLU_CUDA(cudaGetLastError());
  *dout = d;
  return RPLU_OK;
}

static int sample_status(const SampleOut& h) {
  if (h.status == 1) { set_error("weights must be nonnegative"); return RPLU_ERR_ARG; }
  if (h.status == 2) { set_error("all weights are zero; nothing to sample"); return RPLU_ERR_ARG; }
  return RPLU_OK;
}

int sample_index_impl(rplu_ctx* ctx, const double* w, long long n, double u, int mode,
                      long long* idx, int* near, double* total, cudaStream_t s) {
  SampleOut* d = nullptr;
  int rc;
  if ((rc = sample_index_launch(ctx, w, n, u, mode, 0, s, &d))) return rc;
  SampleOut h;
  RPLU_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaStreamSynchronize(s));
  if ((rc = sample_status(h))) return rc;
  if (idx) *idx = h.idx;
  if (near) *near = h.near;
  if (total) *total = h.total;
  return RPLU_OK;
}

// value[0..1] <- gather[idx] of the draw in `d` (complex128 element)
__global__ void sample_gather_kernel(const SampleOut* d, const double2* gather, long long n,
                                     double2* value) {
  const long long i = d->idx;
  *value = (d->status == 0 && i >= 0 && i < n) ? gather[i] : make_double2(0.0, 0.0);
}

// sample_index(w, u) and the element gather[idx] of a complex128 array in one
// host synchronisation (the plan path's column draw + pivot value).
int sample_index_gather_impl(rplu_ctx* ctx, const double* w, long long n, double u,
                             const void* gather, long long* idx, int* near, double* value2,
                             cudaStream_t s) {
  SampleOut* d = nullptr;
  int rc;
  if ((rc = sample_index_launch(ctx, w, n, u, 0, 0, s, &d))) return rc;
  if ((rc = ctx->csync.ensure(1024))) return rc;
  double2* slot = reinterpret_cast<double2*>(reinterpret_cast<char*>(ctx->csync.ptr) + 512);
  count_launches(1);
  sample_gather_kernel<<<1, 1, 0, s>>>(d, reinterpret_cast<const double2*>(gather), n, slot);
  RPLU_CUDA(cudaGetLastError());
  SampleOut h;
  double2 v;
  RPLU_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaMemcpyAsync(&v, slot, sizeof(v), cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaStreamSynchronize(s));
  if ((rc = sample_status(h))) return rc;
  *idx = h.idx;
  if (near) *near = h.near;
  value2[0] = v.x;
  value2[1] = v.y;
  return RPLU_OK;
}

// Plan-path proposal: draw i ~ bounds with u, then hand the drawn index to the
// caller's row kernels on the device (init(d) is enqueued by the caller
// through `after_draw`), total of wbuf in slot 1; one synchronisation in the
// caller.  Returns the two device result slots.
int sample_two_launch(rplu_ctx* ctx, const double* w0, long long n0, double u0,
                      const std::function<int(const void*)>& after_draw, const double* w1,
                      long long n1, cudaStream_t s, const void** d0, const void** d1) {
  SampleOut* a = nullptr;
  SampleOut* b = nullptr;
  int rc;
  // size the scratch for the larger of the two draws first, so that both
  // slots use one stride
  const long long nmax = n0 > n1 ? n0 : n1;
  {
    const long long nch = (nmax + kChunk - 1) / kChunk;
    const size_t per = (sizeof(SampleOut) + 16 + sizeof(double) * (size_t)nch + 63) & ~size_t(63);
    if ((rc = ctx->scratch[7].ensure(2 * per))) return rc;
  }
  if ((rc = sample_index_launch(ctx, w0, n0, u0, 0, 0, s, &a))) return rc;
  if ((rc = after_draw(a))) return rc;
  if ((rc = sample_index_launch(ctx, w1, n1, 0.0, 2, 1, s, &b))) return rc;
  *d0 = a;
  *d1 = b;
  return RPLU_OK;
}

int sample_out_unpack(const void* host_copy, long long* idx, int* near, double* total) {
  const SampleOut& h = *reinterpret_cast<const SampleOut*>(host_copy);
  int rc;
  if ((rc = sample_status(h))) return rc;
  if (idx) *idx = h.idx;
  if (near) *near = h.near;
  if (total) *total = h.total;
  return RPLU_OK;
}

}  // namespace rplu

namespace rplu {

int dense_sweep_launch(int dtype, void* R, long long ld, long long n, long long m, void* Lt,
                       void* U, long long ldu, double* masses, DevState* st, long long t,
                       bool update, cudaStream_t s) {
  DenseParams p{};
  p.R = R;
  p.ld = ld;
  p.n = n;
  p.m = m;
  p.Lt = Lt;
  p.U = U;
  p.ldu = ldu;
  p.masses = masses;
  p.st = st;
  p.t = t;
  switch (dtype) {
    case RPLU_F64: sweep<double>(p, update, false, s); break;
    case RPLU_F32: sweep<float>(p, update, false, s); break;
    case RPLU_C128: sweep<double2>(p, update, false, s); break;
    default: set_error("unknown dtype"); return RPLU_ERR_ARG;
  }
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

template <typename T>
static int lazy_step_t(const DenseParams& p, bool pivcol, bool flush, cudaStream_t s) {
  if (pivcol) {
    const int blocks = (int)((p.n + 255) / 256 < 1024 ? (p.n + 255) / 256 : 1024);
    lazy_pivcol_kernel<T><<<blocks, 256, 0, s>>>(p);
  }
  if (p.gram && !flush) return gram_step<T>(p, p.t0, s);
  if (int rc = lazy_pass<T>(p, flush, s)) return rc;
  if (p.gram && flush && !p.force) {
    const int rb = (int)std::min<long long>((p.n + 255) / 256, 1024);
    gram_reset_kernel<<<rb, 256, 0, s>>>(p);
  }
  return RPLU_OK;
}

static void set_gram(DenseParams& p, double* gram) {
  if (!gram) return;
  p.gram = 1;
  p.m0 = gram;
  p.lin = gram + p.n;
  p.quad = gram + 2 * p.n;
  p.gmat = gram + 3 * p.n;
}

int dense_gram_reset_launch(long long n, double* masses, double* gram, cudaStream_t s) {
  if (n == 0) return RPLU_OK;
  DenseParams p{};
  p.n = n;
  p.masses = masses;
  set_gram(p, gram);
  gram_reset_kernel<<<(int)std::min<long long>((n + 255) / 256, 1024), 256, 0, s>>>(p);
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

int dense_gram_block() { return gram_block(); }

int dense_lazy_step_launch(int dtype, void* R, long long ld, long long n, long long m, void* Lt,
                           void* U, long long ldu, double* masses, DevState* st, long long t,
                           long long t0, bool pivcol, bool flush, bool force, cudaStream_t s,
                           double* gram, bool rel, long long u_rows) {
  if (n == 0) return RPLU_OK;
  if (gram && dtype != RPLU_F64) {
    set_error("Gram-mass delayed updates are fp64 only");
    return RPLU_ERR_ARG;
  }
  DenseParams p{};
  p.R = R;
  p.ld = ld;
  p.n = n;
  p.m = m;
  p.Lt = Lt;
  p.U = U;
  p.ldu = ldu;
  p.masses = masses;
  p.st = st;
  p.t = t;
  p.t0 = t0;
  p.lazy = 1;
  p.force = force ? 1 : 0;
  p.rel = rel ? 1 : 0;      // t, t0: block-relative, absolute step from st->step
  p.u_rows = u_rows;
  set_gram(p, gram);
  int rc;
  switch (dtype) {
    case RPLU_F64: rc = lazy_step_t<double>(p, pivcol, flush, s); break;
    case RPLU_F32: rc = lazy_step_t<float>(p, pivcol, flush, s); break;
    case RPLU_C128: rc = lazy_step_t<double2>(p, pivcol, flush, s); break;
    default: set_error("unknown dtype"); return RPLU_ERR_ARG;
  }
  if (rc) return rc;
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

int dense_lazy_block_default(int dtype, bool fused) {
  switch (dtype) {
    case RPLU_F64: return lazy_block<double>(fused);
    case RPLU_F32: return lazy_block<float>(fused);
    default: return lazy_block<double2>(fused);
  }
}

}  // namespace rplu
