// Barycentric rational kernels for the CUR-AAA consumer.
//
// Reference: rplu.rational (pkg/src/rplu/rational.py).
//   KL  loewner_fill   L[i,j] = (f_o[i] - f_s[j]) / (z_o[i] - z_s[j])
//                      (_loewner_weights, rational.py:124-127): the divided-
//                      difference matrix whose smallest right singular vector
//                      gives the barycentric weights.  numpy-exact elementwise
//                      arithmetic (complex subtract, Smith division).
//   KB  bary_eval      r(z) = sum_j c_j w_j f_j / sum_j c_j w_j with
//                      c_j = 1/(z - t_j) generated in registers — a Cauchy
//                      GEMV against two right-hand sides, so no C matrix in
//                      HBM (rational.py:63-80 and the AAA refit :165-169).
//                      mode 0: BarycentricRational evaluation — exact-hit
//                      branch (|z - t_j| <= tol*scale returns f_j, the last
//                      matching j winning as in the reference loop :71-75)
//                      and the near-pole flag (|den| < 1e3*tiny or a
//                      non-finite quotient, :70);  mode 1: the AAA refit —
//                      non-finite quotients become 0 (:168).
// Support sets are small (degree <= a few hundred) and evaluation sets large:
// one thread per evaluation point, the support staged through shared memory
// in tiles, FP64-pipe bound: per (z, t_j) pair 2 sub + |d|^2 (2) + one IEEE
// reciprocal + 2 mul + two complex MACs (8 FMA).  The entries are
// conj(d)/|d|^2 (Smith division only where |d|^2 would leave the normal
// range); the sums are order-dependent anyway (the reference's are BLAS
// zgemv), so parity is to rounding, not bits.
#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "rplu_common.cuh"
#include "rplu_internal.h"

namespace rplu {

__global__ void __launch_bounds__(256) loewner_fill_kernel(const double2* __restrict__ zo,
                                                           const double2* __restrict__ fo,
                                                           long long no,
                                                           const double2* __restrict__ zs,
                                                           const double2* __restrict__ fs,
                                                           long long k, double2* __restrict__ out) {
  const long long total = no * k;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / k, j = e - i * k;
    const double2 a = fo[i], b = fs[j], c = zo[i], d = zs[j];
    const double2 num = make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
    const double2 den = make_double2(__dsub_rn(c.x, d.x), __dsub_rn(c.y, d.y));
    out[e] = cdiv_np(num, den);
  }
}

constexpr int kBaryTile = 512;

__device__ __forceinline__ double2 cmac(double2 acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
  return acc;
}

__global__ void __launch_bounds__(256) bary_eval_kernel(const double2* __restrict__ z, long long nz,
                                                        const double2* __restrict__ t,
                                                        const double2* __restrict__ f,
                                                        const double2* __restrict__ w, int k,
                                                        double hit_tol, int mode,
                                                        double2* __restrict__ out,
                                                        int32_t* __restrict__ near_pole) {
  __shared__ double2 st[kBaryTile], swf[kBaryTile], sw[kBaryTile];
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const double2 zi = i < nz ? z[i] : make_double2(0.0, 0.0);
  double2 num = make_double2(0.0, 0.0), den = make_double2(0.0, 0.0);
  int hit = -1;
  const double hit2 = hit_tol * hit_tol * (1.0 + 1e-12);
  for (int j0 = 0; j0 < k; j0 += kBaryTile) {
    const int cnt = min(kBaryTile, k - j0);
    __syncthreads();
    for (int c = threadIdx.x; c < cnt; c += blockDim.x) {
      st[c] = t[j0 + c];
      sw[c] = w[j0 + c];
      swf[c] = cmul_np(w[j0 + c], f[j0 + c]);  // r.weights * r.values (:66)
    }
    __syncthreads();
    for (int c = 0; c < cnt; ++c) {
      const double dx = zi.x - st[c].x, dy = zi.y - st[c].y;
      const double d2 = fma(dx, dx, dy * dy);
      // exact-hit test |z - t_j| <= tol (np.abs = hypot): cheap prefilter on
      // |d|^2, hypot only for the candidates
      if (mode == 0 && d2 <= hit2 && hypot(dx, dy) <= hit_tol) hit = j0 + c;
      double2 cj;
      // |d|^2 inside [2^-960, 2^960) by an integer test on its exponent field
      // (FP64 compares run on the FP64 pipe, which bounds this kernel)
      const unsigned ex = ((unsigned)__double2hiint(d2) >> 20) & 0x7ffu;
      if (ex - 63u < 1920u) {             // 1/(z - t) = conj(d) / |d|^2
        const double r = rcp_nr(d2);      // seed + one cubic step: <= 2 ulp in 3 DFMA
        cj = make_double2(dx * r, -dy * r);
      } else {                            // over/underflow-safe Smith division
        cj = cdiv_np(make_double2(1.0, 0.0), make_double2(dx, dy));
      }
      num = cmac(num, cj, swf[c]);
      den = cmac(den, cj, sw[c]);
    }
  }
  if (i >= nz) return;
  double2 r = cdiv_np(num, den);
  const bool finite = isfinite(r.x) && isfinite(r.y);
  if (mode == 1) {
    if (!finite) r = make_double2(0.0, 0.0);
    out[i] = r;
    return;
  }
  int flag = (hypot(den.x, den.y) < 1e3 * DBL_MIN) || !finite;
  if (hit >= 0) {
    r = f[hit];
    flag = 0;
  }
  out[i] = r;
  near_pole[i] = flag;
}

int loewner_fill_impl(const void* zo, const void* fo, long long no, const void* zs,
                      const void* fs, long long k, void* out, cudaStream_t s) {
  const long long total = no * k;
  if (total == 0) return 0;
  const long long blocks = std::min<long long>((total + 255) / 256, 148LL * 16);
  count_launches(1);
  loewner_fill_kernel<<<(unsigned)blocks, 256, 0, s>>>(
      (const double2*)zo, (const double2*)fo, no, (const double2*)zs, (const double2*)fs, k,
      (double2*)out);
  RPLU_CUDA(cudaGetLastError());
  return 0;
}

int bary_eval_impl(const void* z, long long nz, const void* t, const void* f, const void* w,
                   long long k, double hit_tol, int mode, void* out, int32_t* near_pole,
                   cudaStream_t s) {
  if (nz == 0) return 0;
  const long long blocks = (nz + 255) / 256;
  count_launches(1);
  bary_eval_kernel<<<(unsigned)blocks, 256, 0, s>>>(
      (const double2*)z, nz, (const double2*)t, (const double2*)f, (const double2*)w, (int)k,
      hit_tol, mode, (double2*)out, near_pole);
  RPLU_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace rplu
