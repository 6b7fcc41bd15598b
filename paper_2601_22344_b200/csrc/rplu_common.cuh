// Shared device helpers for the RPLU pivot loop (sm_100a).
//
// * Scalar traits for the three residual element types the reference path
//   supports (fp32, fp64, complex128).  The reference computes everything in
//   complex128 (dense_pivots.py:196-199, accessors.py:416); a real input has a
//   zero imaginary part, so the real instantiations reproduce its arithmetic
//   exactly (see numpy_cdiv / cmul_np below and DESIGN.md §"numerics").
// * numpy-exact complex kernels: division (Smith, numpy loops.c divide),
//   multiplication (npyv SIMD: fma(ar,br,-ai*bi), fma(ar,bi,ai*br)) and the
//   AVX-512 cabs (L*sqrt(fma(r,r,1))).  All "_rn" intrinsics: no contraction.
// * Block-wide chunked inverse-CDF search with the exact tie/zero semantics of
//   rplu.rng.sample_index (rng.py:50-74): first index whose running sum is
//   strictly greater than u*total (searchsorted side='right'), top clamp,
//   walk-back over zero weights, first-positive fallback.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rplu {

constexpr double kNearBoundaryRel = 1e-12;  // BASELINE north star: draws within
                                            // 1e-12 relative of a CDF boundary

// ---------------------------------------------------------------------------
// complex helpers (double2 = {re, im})

__device__ __forceinline__ double2 cmul_np(double2 a, double2 b) {
  // numpy complex multiply as dispatched on x86-64 (AVX2/AVX-512 npyv path).
  double re = __fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y));
  double im = __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x));
  return make_double2(re, im);
}

// Smith-division coefficients of a pivot value a, hoisted out of the column
// loop.  branch 0: |ar| >= |ai|; branch 1 otherwise.
struct CDivCoef {
  double rat, scl;
  int branch;
};

__device__ __forceinline__ CDivCoef cdiv_coef(double2 b) {
  CDivCoef c;
  if (fabs(b.x) >= fabs(b.y)) {
    c.branch = 0;
    c.rat = __ddiv_rn(b.y, b.x);
    c.scl = __ddiv_rn(1.0, __dadd_rn(b.x, __dmul_rn(b.y, c.rat)));
  } else {
    c.branch = 1;
    c.rat = __ddiv_rn(b.x, b.y);
    c.scl = __ddiv_rn(1.0, __dadd_rn(b.y, __dmul_rn(b.x, c.rat)));
  }
  return c;
}

__device__ __forceinline__ double2 cdiv_apply(double2 a, const CDivCoef& c) {
  double re, im;
  if (c.branch == 0) {
    re = __dmul_rn(__dadd_rn(a.x, __dmul_rn(a.y, c.rat)), c.scl);
    im = __dmul_rn(__dsub_rn(a.y, __dmul_rn(a.x, c.rat)), c.scl);
  } else {
    re = __dmul_rn(__dadd_rn(__dmul_rn(a.x, c.rat), a.y), c.scl);
    im = __dmul_rn(__dsub_rn(__dmul_rn(a.y, c.rat), a.x), c.scl);
  }
  return make_double2(re, im);
}

__device__ __forceinline__ double2 cdiv_np(double2 a, double2 b) {
  return cdiv_apply(a, cdiv_coef(b));
}

__device__ __forceinline__ double cabs_np(double2 a) {
  double x = fabs(a.x), y = fabs(a.y);
  double L = fmax(x, y), S = fmin(x, y);
  if (L == 0.0) return 0.0;
  double r = __ddiv_rn(S, L);
  return __dmul_rn(L, __dsqrt_rn(__fma_rn(r, r, 1.0)));
}

// ---------------------------------------------------------------------------
// fast FP64 reciprocal: MUFU.RCP64H seed (relative error <= 2^-19.9 over 2^30
// samples on B200, scripts/probes/rcp_probe.cu) + ONE cubic step
//   e = 1 - d r0,  r1 = r0 (1 + e + e^2)      (error e^3 ~ 2^-60 + rounding)
// in three DFMA: <= 2 ulp (0.03% of arguments differ from the correctly
// rounded 1/d at all).  Two Newton steps reproduce the correctly rounded
// value for every sample but cost four DFMA -- one of K5's 9 (p = 1) or 27
// (p = 4) FP64 instructions per generated entry.  The masses are sums of
// ~m such terms and only feed the sampling weights.
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double e = fma(-d, r, 1.0);
  const double t = fma(e, e, e);
  return fma(r, t, r);
}

// ---------------------------------------------------------------------------
// scalar traits

template <typename T> struct Scalar;

template <> struct Scalar<double> {
  using coef_t = double;  // reciprocal of the pivot, x*(1/a) (numpy Smith, ai=0)
  static constexpr int kVec = 2;
  __device__ static __forceinline__ double mass(double v) { return v * v; }
  // column weight |r|^2 with |.| = np.abs (exact for real values)
  __device__ static __forceinline__ double weight(double v) { return __dmul_rn(v, v); }
  __device__ static __forceinline__ double absval(double v) { return fabs(v); }
  __device__ static __forceinline__ bool is_zero(double v) { return v == 0.0; }
  __device__ static __forceinline__ coef_t make_coef(double a) { return __ddiv_rn(1.0, a); }
  __device__ static __forceinline__ double scale(double c, coef_t k) { return __dmul_rn(c, k); }
  __device__ static __forceinline__ double sub_outer(double r, double l, double p) {
    return __dsub_rn(r, __dmul_rn(l, p));
  }
  __device__ static __forceinline__ double zero() { return 0.0; }
};

template <> struct Scalar<float> {
  using coef_t = float;
  static constexpr int kVec = 4;
  __device__ static __forceinline__ double mass(float v) { double d = v; return d * d; }
  __device__ static __forceinline__ double weight(float v) { double d = v; return d * d; }
  __device__ static __forceinline__ double absval(float v) { return fabs((double)v); }
  __device__ static __forceinline__ bool is_zero(float v) { return v == 0.0f; }
  __device__ static __forceinline__ coef_t make_coef(float a) { return __fdiv_rn(1.0f, a); }
  __device__ static __forceinline__ float scale(float c, coef_t k) { return __fmul_rn(c, k); }
  __device__ static __forceinline__ float sub_outer(float r, float l, float p) {
    return __fsub_rn(r, __fmul_rn(l, p));
  }
  __device__ static __forceinline__ float zero() { return 0.0f; }
};

template <> struct Scalar<double2> {
  using coef_t = CDivCoef;
  static constexpr int kVec = 1;
  __device__ static __forceinline__ double mass(double2 v) { return v.x * v.x + v.y * v.y; }
  __device__ static __forceinline__ double weight(double2 v) {
    double a = cabs_np(v);
    return __dmul_rn(a, a);
  }
  __device__ static __forceinline__ double absval(double2 v) { return cabs_np(v); }
  __device__ static __forceinline__ bool is_zero(double2 v) { return v.x == 0.0 && v.y == 0.0; }
  __device__ static __forceinline__ coef_t make_coef(double2 a) { return cdiv_coef(a); }
  __device__ static __forceinline__ double2 scale(double2 c, const coef_t& k) { return cdiv_apply(c, k); }
  __device__ static __forceinline__ double2 sub_outer(double2 r, double2 l, double2 p) {
    double2 q = cmul_np(l, p);
    return make_double2(__dsub_rn(r.x, q.x), __dsub_rn(r.y, q.y));
  }
  __device__ static __forceinline__ double2 zero() { return make_double2(0.0, 0.0); }
};

// ---------------------------------------------------------------------------
// warp / block primitives

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// argmax with lowest-index tie break (np.argmax semantics)
__device__ __forceinline__ void argmax_merge(double& v, long long& i, double v2, long long i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

__device__ __forceinline__ void warp_argmax(double& v, long long& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    long long i2 = __shfl_xor_sync(0xffffffffu, i, o);
    argmax_merge(v, i, v2, i2);
  }
}

// Shared scratch for the single-CTA select kernels.
template <int BLOCK>
struct CdfSmem {
  double wexcl[BLOCK / 32];  // CDF value before warp segment w
  double wincl[BLOCK / 32];  // CDF value at the end of warp segment w
  long long idx;
  double lo_c, hi_c;
  double wsel;    // weight of the selected element (when known without a reload)
  int has_wsel;
  int owner;
};

// CDF layout (one CTA of BLOCK threads).  The n weights are split into
// BLOCK/32 contiguous warp segments of S elements (S a multiple of 32), each
// walked in slabs of 32 consecutive elements (one coalesced load per lane).
// Segment totals T_w (lane-private sums + fixed-order warp reduction) are
// accumulated sequentially into excl_w / incl_w = excl_w + T_w; the owner is
// the first segment with incl_w > target.  Inside the owner segment the walk
// uses slab scans: the CDF value of element k (slab s, lane l) is
//     c_k = excl_w + (r_s + p_l),
// p_l the warp inclusive scan of the slab, r_s the sequential sum of the
// previous slabs; if rounding leaves every c_k <= target < incl_w, the last
// element of the segment is chosen (its interval ends at incl_w).  (The
// reference's np.cumsum is one sequential sum; the association differs, so
// GPU and reference draws agree except within rounding of a boundary —
// counted as near-boundary draws.)
template <int BLOCK>
struct Cdf {
  long long seg;  // segment length S
  double total;
};

constexpr int kCdfUnroll = 8;  // slabs in flight per warp

__device__ __forceinline__ double warp_incl_scan(double x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

template <int BLOCK, typename WF>
__device__ Cdf<BLOCK> cdf_build(const WF& wf, long long n, CdfSmem<BLOCK>& s) {
  constexpr int W = BLOCK / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Cdf<BLOCK> c;
  c.seg = (((n + W - 1) / W) + 31) / 32 * 32;
  if (c.seg < 32) c.seg = 32;
  const long long lo = min((long long)w * c.seg, n), hi = min(lo + c.seg, n);
  // Segment total: lane-private sums (2-3 instructions per element) then a
  // fixed-order warp reduction.  The owner search below walks the segment
  // with slab scans; if rounding puts the target between its running sum and
  // this total, the segment's last element is taken (a near-boundary draw).
  double run = 0.0;
  for (long long base = lo; base < hi; base += 32 * kCdfUnroll) {
    double xs[kCdfUnroll];
#pragma unroll
    for (int u = 0; u < kCdfUnroll; ++u) {
      const long long k = base + 32 * u + lane;
      xs[u] = (k < hi) ? wf(k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kCdfUnroll; ++u) run += xs[u];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) run += __shfl_down_sync(0xffffffffu, run, o);
  if (lane == 0) s.wincl[w] = run;  // segment total (temporarily)
  __syncthreads();
  if (threadIdx.x == 0) {
    // sequential prefix over the segment totals (all loads issued first)
    double tv[W];
#pragma unroll
    for (int q = 0; q < W; ++q) tv[q] = s.wincl[q];
    double e = 0.0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      s.wexcl[q] = e;
      e = e + tv[q];
      s.wincl[q] = e;
    }
  }
  __syncthreads();
  c.total = s.wincl[W - 1];
  return c;
}

// sample_index(w, u) on a built CDF.  Returns the index (block-uniform); the
// CDF values bracketing the draw are left in s.lo_c / s.hi_c for the caller's
// near-boundary accounting.
template <int BLOCK, typename WF>
__device__ long long cdf_find_target(const WF& wf, long long n, const Cdf<BLOCK>& c,
                                     double target, CdfSmem<BLOCK>& s, double cbase = 0.0,
                                     bool walk_back = true);

template <int BLOCK, typename WF>
__device__ __forceinline__ long long cdf_find(const WF& wf, long long n, const Cdf<BLOCK>& c,
                                              double u, CdfSmem<BLOCK>& s) {
  return cdf_find_target<BLOCK>(wf, n, c, u * c.total, s);
}

// Same search against an absolute target in [0, total] (sharded draws).
// `cbase` offsets every CDF value of this block (c_k = base + (excl_w + ...)):
// the chunked large-n draw runs the search on its owner chunk with base = the
// chunk's exclusive prefix (cbase = 0 adds nothing: identical results).
// walk_back = false leaves a zero-weight selection to the caller.
template <int BLOCK, typename WF>
__device__ long long cdf_find_target(const WF& wf, long long n, const Cdf<BLOCK>& c,
                                     double target, CdfSmem<BLOCK>& s, double cbase,
                                     bool walk_back) {
  constexpr int W = BLOCK / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w == 0) {  // owner = first segment whose running sum exceeds the target
    static_assert(W <= 32, "one lane per segment");
    const bool gt = lane < W && cbase + s.wincl[lane] > target;
    const unsigned hit = __ballot_sync(0xffffffffu, gt);
    const int owner = hit ? __ffs(hit) - 1 : -1;
    if (lane == 0) {
      s.owner = owner;
      s.has_wsel = 0;
      if (owner < 0) {
        // u*total >= every partial sum: searchsorted returns n, clamp to n-1
        s.idx = n - 1;
        s.lo_c = cbase + c.total;
        s.hi_c = cbase + c.total;
      }
    }
  }
  __syncthreads();
  if (w == s.owner) {
    const long long lo = min((long long)w * c.seg, n), hi = min(lo + c.seg, n);
    const double ex = s.wexcl[w];
    double run = 0.0, prev = cbase + ex;
    bool done = false;
    for (long long base = lo; base < hi && !done; base += 32 * kCdfUnroll) {
      double xs[kCdfUnroll];
#pragma unroll
      for (int u = 0; u < kCdfUnroll; ++u) {
        const long long k = base + 32 * u + lane;
        xs[u] = (k < hi) ? wf(k) : 0.0;
      }
      // CTAs of <= 512 threads (register budget >= 128): the slabs' inclusive
      // scans all interleaved round by round -- the same shuffle-add sequence
      // per slab as warp_incl_scan, so identical values; one after the other
      // they are the draw's longest serial chain (C2 resident loop: 3.6 -> 3.3
      // us per draw).  With 1024 threads (64 registers) the eight live scans
      // spill and the draws got slower (C1 resident loop 58k -> 50k steps/s),
      // so those kernels scan slab by slab.
      constexpr bool kInterleave = BLOCK <= 512;
      double ps[kCdfUnroll];
      if constexpr (kInterleave) {
#pragma unroll
        for (int u = 0; u < kCdfUnroll; ++u) ps[u] = xs[u];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
          for (int u = 0; u < kCdfUnroll; ++u) {
            const double y = __shfl_up_sync(0xffffffffu, ps[u], o);
            if (lane >= o) ps[u] += y;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kCdfUnroll; ++u) {
        const long long sb = base + 32 * u;
        if (done || sb >= hi) break;
        double p;
        if constexpr (kInterleave) p = ps[u];
        else p = warp_incl_scan(xs[u]);
        const double ck = cbase + (ex + (run + p));
        const unsigned hit = __ballot_sync(0xffffffffu, (sb + lane < hi) && ck > target);
        if (hit) {
          const int L = __ffs(hit) - 1;
          const double hc = __shfl_sync(0xffffffffu, ck, L);
          const double pc = __shfl_sync(0xffffffffu, ck, L > 0 ? L - 1 : 0);
          const double wv = __shfl_sync(0xffffffffu, xs[u], L);
          if (lane == 0) {
            s.idx = sb + L;
            s.hi_c = hc;
            s.lo_c = L > 0 ? pc : prev;
            s.wsel = wv;
            s.has_wsel = 1;
          }
          done = true;
        } else {
          run += __shfl_sync(0xffffffffu, p, 31);
          prev = cbase + (ex + run);
        }
      }
    }
    if (!done && lane == 0) {
      // target within rounding of the segment's end: its last element owns
      // the interval up to incl_w
      s.idx = hi - 1;
      s.lo_c = prev;
      s.hi_c = cbase + s.wincl[w];
    }
  }
  __syncthreads();
  long long i = s.idx;
  // walk back over zero weights (rng.py:70-73)
  const double wi = s.has_wsel ? s.wsel : wf(i);
  __syncthreads();
  if (walk_back && !(wi > 0.0)) {
    // largest k <= i with w(k) > 0, else smallest k with w(k) > 0
    long long best_lo = -1, best_any = n;
    for (long long k = threadIdx.x; k < n; k += BLOCK) {
      if (wf(k) > 0.0) {
        if (k <= i && k > best_lo) best_lo = k;
        if (k < best_any) best_any = k;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      best_lo = max(best_lo, __shfl_xor_sync(0xffffffffu, best_lo, o));
      best_any = min(best_any, __shfl_xor_sync(0xffffffffu, best_any, o));
    }
    __shared__ long long wlo[BLOCK / 32], wany[BLOCK / 32];
    if (lane == 0) { wlo[w] = best_lo; wany[w] = best_any; }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long a = -1, b = n;
      for (int q = 0; q < BLOCK / 32; ++q) { a = max(a, wlo[q]); b = min(b, wany[q]); }
      s.idx = (a >= 0) ? a : b;
    }
    __syncthreads();
    i = s.idx;
    __syncthreads();
  }
  return i;
}

// Block argmax of wf(k) over [0,n) with lowest-index ties.
template <int BLOCK, typename WF>
__device__ long long block_argmax(const WF& wf, long long n, double* out_val) {
  double v = -1.0;
  long long idx = n;
  for (long long k = threadIdx.x; k < n; k += BLOCK) argmax_merge(v, idx, wf(k), k);
  warp_argmax(v, idx);
  __shared__ double sv[BLOCK / 32];
  __shared__ long long si[BLOCK / 32];
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = v; si[threadIdx.x >> 5] = idx; }
  __syncthreads();
  if (threadIdx.x < 32) {
    v = (threadIdx.x < BLOCK / 32) ? sv[threadIdx.x] : -1.0;
    idx = (threadIdx.x < BLOCK / 32) ? si[threadIdx.x] : n;
    warp_argmax(v, idx);
    if (threadIdx.x == 0) { sv[0] = v; si[0] = idx; }
  }
  __syncthreads();
  long long r = si[0];
  if (out_val) *out_val = sv[0];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------
// Large-n draws (the plan path's row / column draws over 2^20 weights, the
// CUR row draws over 2e6): the single-CTA walk is latency bound (222 us at
// 2^20).  Two levels instead: chunks of kChunk weights, each chunk's total
// built by one CTA with the single-CTA CDF arithmetic (cdf_build on the
// chunk), a sequential prefix over the chunk totals, then the single-CTA
// search inside the owner chunk offset by the chunk's exclusive prefix.  The
// CDF association therefore differs from the single-CTA one for n above the
// threshold (both differ from np.cumsum only within rounding of a boundary,
// counted as near-boundary draws).
constexpr long long kChunk = 32768;
constexpr long long kChunkedMinN = 4 * kChunk;

// one CTA of 1024 threads per chunk (blockIdx.x = chunk): its total into
// ctot[chunk]; *neg |= 1 on a negative weight
__device__ __forceinline__ void chunk_totals_block(const double* w, long long n, double* ctot,
                                                   int* neg) {
  constexpr int B = 1024;
  __shared__ CdfSmem<B> sm;
  const long long c0 = (long long)blockIdx.x * kChunk;
  const long long nc = min(kChunk, n - c0);
  const double* wc = w + c0;
  bool bad = false;
  for (long long k = threadIdx.x; k < nc; k += B) bad |= wc[k] < 0.0;
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(neg, 1);
  auto wf = [&](long long k) { return wc[k]; };
  Cdf<B> c = cdf_build<B>(wf, nc, sm);
  if (threadIdx.x == 0) ctot[blockIdx.x] = c.total;
}

// The draw over the chunk totals (one CTA of 1024): mode 0 u * total, mode
// 1 absolute target, mode 2 total only.  Returns the index (block-uniform;
// meaningless when *total_out is not positive or mode == 2); *near_out = 1
// when the target lies within 1e-12 total of a CDF boundary.
static __device__ __noinline__ long long chunked_draw_block(const double* w, long long n, double u,
                                                     int mode, const double* ctot,
                                                     long long nch, CdfSmem<1024>& sm,
                                                     double* total_out, int* near_out) {
  constexpr int B = 1024;
  __shared__ double s_excl, s_total;
  __shared__ long long s_owner;
  if (threadIdx.x == 0) {  // sequential prefix over the chunk totals
    double e = 0.0;
    for (long long q = 0; q < nch; ++q) e = e + ctot[q];
    s_total = e;
  }
  __syncthreads();
  const double total = s_total;
  *total_out = total;
  *near_out = 0;
  if (mode == 2 || !(total > 0.0)) return -1;
  const double tg = (mode == 1) ? u : u * total;
  if (threadIdx.x == 0) {
    double e = 0.0;
    long long own = -1;
    for (long long q = 0; q < nch; ++q) {
      const double inc = e + ctot[q];
      if (inc > tg) { own = q; break; }
      e = inc;
    }
    s_owner = own;
    s_excl = e;
  }
  __syncthreads();
  long long i;
  if (s_owner < 0) {  // target >= every partial sum: clamp to n - 1
    i = n - 1;
    if (threadIdx.x == 0) { sm.lo_c = total; sm.hi_c = total; }
  } else {
    const long long c0 = s_owner * kChunk;
    const long long nc = min(kChunk, n - c0);
    const double* wc = w + c0;
    auto wf = [&](long long k) { return wc[k]; };
    Cdf<B> c = cdf_build<B>(wf, nc, sm);
    i = c0 + cdf_find_target<B>(wf, nc, c, tg, sm, s_excl, false);
  }
  __syncthreads();
  // walk back over zero weights over the whole array (rng.py:70-73)
  if (!(w[i] > 0.0)) {
    long long best_lo = -1, best_any = n;
    for (long long k = threadIdx.x; k < n; k += B) {
      if (w[k] > 0.0) {
        if (k <= i && k > best_lo) best_lo = k;
        if (k < best_any) best_any = k;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      best_lo = max(best_lo, __shfl_xor_sync(0xffffffffu, best_lo, o));
      best_any = min(best_any, __shfl_xor_sync(0xffffffffu, best_any, o));
    }
    __shared__ long long wlo[B / 32], wany[B / 32];
    if ((threadIdx.x & 31) == 0) { wlo[threadIdx.x >> 5] = best_lo; wany[threadIdx.x >> 5] = best_any; }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long a = -1, b = n;
      for (int q = 0; q < B / 32; ++q) { a = max(a, wlo[q]); b = min(b, wany[q]); }
      sm.idx = (a >= 0) ? a : b;
    }
    __syncthreads();
    i = sm.idx;
  }
  const double tol = kNearBoundaryRel * total;
  *near_out = (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) ? 1 : 0;
  __syncthreads();
  return i;
}

// ---------------------------------------------------------------------------
// Grid-wide synchronisation for the persistent (cooperative) loops.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* a, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_count(const unsigned* c, unsigned target) {
  while (ld_acquire_u32(c) < target) {
  }
}
// sync[0]: grid-barrier arrivals
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    wait_count(bar, target);
    __threadfence();
  }
  __syncthreads();
}

}  // namespace rplu
