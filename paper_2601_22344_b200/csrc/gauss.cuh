// Gaussian-kernel entry evaluation shared by the CUR kernels (cur.cu) and
// the device-resident CUR loop (mf.cu).
#pragma once
#include <cuda_runtime.h>

namespace rplu {

// exp(-d2) for d2 >= 0 (the kernel's exponent), table-driven.  With
// y = -d2 * 32/ln2, k = round(y) = 32 n + j (0 <= j < 32) and s = y - k
// (|s| <= 1/2, formed as fma(-K, d2, -k): one rounding, so the Cody-Waite
// hi/lo reduction of a separately rounded y is not needed),
//   exp(-d2) = 2^n * 2^(j/32) * p(s),   p(s) ~ exp(s ln2/32) of degree 5
// (a relative least-squares fit; 2.5e-16 max relative error).  2^(j/32) comes from a 32-entry table held
// one entry per lane (fetched with a warp shuffle: no shared-memory bank
// conflicts), 2^n is added to the table value's exponent field with integer
// ops, k is read from the low word of the round-to-nearest shifter sum, and
// the underflow cut (exp(-d2) < 1e-307 -> 0) is an integer compare on k —
// so an entry costs 16 FP64-pipe operations including the distance and the
// accumulate (the hi/lo reduction and the FP64 compare of an earlier
// variant cost 19, the degree-6 Taylor polynomial 17).  A 64-entry table
// with a degree-4 polynomial would save one more DFMA but needs two 64-bit
// shuffles per entry (a 64-entry / degree-5 variant measured 2% slower,
// DESIGN.md §10).  Relative error ~ 1.5 ulp + d2 * 2^-53 (the rounding of
// K d2).
// Every lane of the warp must call it (warp-synchronous shuffle).
static __constant__ double kExp2Tab[32] = {
    1.0, 1.0218971486541166, 1.0442737824274138, 1.0671404006768237,
    1.0905077326652577, 1.1143867425958924, 1.1387886347566916, 1.1637248587775775,
    1.189207115002721, 1.215247359980469, 1.241857812073484, 1.2690509571917332,
    1.2968395546510096, 1.3252366431597413, 1.3542555469368927, 1.383909881963832,
    1.4142135623730951, 1.4451808069770467, 1.4768261459394993, 1.5091644275934228,
    1.5422108254079407, 1.5759808451078865, 1.6104903319492543, 1.645755478153965,
    1.681792830507429, 1.718619298122478, 1.7562521603732995, 1.7947090750031072,
    1.8340080864093424, 1.8741676341103, 1.9152065613971474, 1.9571441241754002};

using ExpTab = double;  // this lane's 2^(lane/32)

__device__ __forceinline__ ExpTab exp2tab_lane() { return kExp2Tab[threadIdx.x & 31]; }

__device__ __forceinline__ double exp_neg(double d2, ExpTab tab) {
  const double shifter = 6755399441055744.0;  // 1.5 * 2^52: round-to-nearest
  const double K = 46.16624130844683;          // 32 / ln2
  const double sft = fma(d2, -K, shifter);
  const double kd = sft - shifter;
  const int k = __double2loint(sft);
  const double s = fma(d2, -K, -kd);           // y - k, |s| <= 1/2
  // degree-5 fit of exp(s ln2/32) on |s| <= 1/2 (relative least squares at
  // Chebyshev nodes, extended precision): 2.5e-16 max / 0.36 ulp mean
  // relative error in FMA Horner, against 0.51 ulp for the degree-6 Taylor
  // polynomial -- one DFMA less per entry
  double p = 3.9736907164886624e-11;
  p = fma(p, s, 9.172616497450463e-09);
  p = fma(p, s, 1.6938509725336998e-06);
  p = fma(p, s, 0.00023459619819720352);
  p = fma(p, s, 0.021660849392498283);
  p = fma(p, s, 1.0);
  const double t = __shfl_sync(0xffffffffu, tab, k & 31);
  const double ts = __hiloint2double(__double2hiint(t) + ((k >> 5) << 20), __double2loint(t));
  const double e = p * ts;
  return k < -32700 ? 0.0 : e;                 // k < -32*1021.9: below 1e-307
}

// polynomial coefficients as constant-bank operands (as immediates they were
// re-materialised into uniform registers every trip: ~1 extra issue slot per
// entry)
static __constant__ double kExpPoly[5] = {3.9736907164886624e-11, 9.172616497450463e-09,
                                          1.6938509725336998e-06, 0.00023459619819720352,
                                          0.021660849392498283};

template <int E>
__device__ __forceinline__ void exp_tab_units_v(const double (&y)[E], double (&e)[E],
                                                ExpTab tab) {
  // k = round(y) and the reduced argument s = y - k (exact, |s| <= 1/2).  The
  // rounding and the integer come from the conversion unit (FRND.F64,
  // F2I.F64: both round to nearest even, so they agree) instead of the
  // shifter trick's two DADDs: the FP64 pipe keeps 11 instructions per entry
  // of the factored GEMV (3 dot + 1 subtract + 5 polynomial + scale +
  // accumulate) (same box, n = m = 10^6: 903 against 929 ms).
  double s[E], p[E];
  int k[E];
#pragma unroll
  for (int i = 0; i < E; ++i) s[i] = rint(y[i]);
#pragma unroll
  for (int i = 0; i < E; ++i) k[i] = __double2int_rn(y[i]);
#pragma unroll
  for (int i = 0; i < E; ++i) s[i] = y[i] - s[i];
#pragma unroll
  for (int i = 0; i < E; ++i) p[i] = fma(kExpPoly[0], s[i], kExpPoly[1]);
#pragma unroll
  for (int i = 0; i < E; ++i) p[i] = fma(p[i], s[i], kExpPoly[2]);
#pragma unroll
  for (int i = 0; i < E; ++i) p[i] = fma(p[i], s[i], kExpPoly[3]);
#pragma unroll
  for (int i = 0; i < E; ++i) p[i] = fma(p[i], s[i], kExpPoly[4]);
#pragma unroll
  for (int i = 0; i < E; ++i) p[i] = fma(p[i], s[i], 1.0);
  // `tab` is the lane's COMPENSATED table entry (exp2tab_lane_comp): its high
  // word has (lane << 15) subtracted, so adding k << 15 = (n << 20) + (j << 15)
  // to the word fetched from lane j = k mod 32 (the shuffle takes the index
  // modulo 32 itself) lands exactly on 2^n 2^(j/32): one integer instruction
  // and two shuffles per entry beside the FP64 ones.  Every FP64 warp
  // instruction holds the SM sub-partition's dispatch port for two cycles, so
  // each further instruction costs about 1/22 of the entry's FP64 time.
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const int hi = __shfl_sync(0xffffffffu, __double2hiint(tab), k[i]);
    const int lo = __shfl_sync(0xffffffffu, __double2loint(tab), k[i]);
    e[i] = p[i] * __hiloint2double(hi + (k[i] << 15), lo);
  }
}

__device__ __forceinline__ ExpTab exp2tab_lane_comp() {
  const int lane = threadIdx.x & 31;
  const double t = kExp2Tab[lane];
  return __hiloint2double(__double2hiint(t) - (lane << 15), __double2loint(t));
}

// Entry from coordinates prescaled by sc = 1/(sqrt(2) h) (done once per
// point as it is loaded into registers / shared memory), so the exponent
// -|p-q|^2/(2h^2) is just -|p'-q'|^2.
__device__ __forceinline__ double gauss_entry(double px, double py, double pz, double qx,
                                              double qy, double qz, ExpTab tab) {
  const double dx = px - qx, dy = py - qy, dz = pz - qz;
  const double d2 = fma(dz, dz, fma(dy, dy, dx * dx));
  return exp_neg(d2, tab);
}

}  // namespace rplu
