// Modified Gram-Schmidt Arnoldi step for restarted GMRES.
//
// Reference: rplu.precond.gmres (pkg/src/rplu/precond.py:137-192), inner loop
// :160-166:
//     for t in range(j + 1):
//         H[t, j] = vdot(V[:, t], w);  w = w - H[t, j] * V[:, t]
//     H[j + 1, j] = norm(w);  if > 0: V[:, j + 1] = w / H[j + 1, j]
// One cooperative launch performs the whole step.  Pass t fuses the
// subtraction of step t-1 with the inner product of step t (the MGS order is
// kept: H[t, j] is taken against the already-updated w), so an Arnoldi step
// of j+1 projections streams j+2 passes over (V_{t-1}, V_t, w) instead of the
// reference's 2(j+1)+2 separate BLAS-1 sweeps.  Inner products are reduced
// per CTA into a double-buffered partials array, then — after one grid
// barrier — every CTA sums the partials in the same fixed order, so all CTAs
// hold the identical H[t, j] without a second barrier.  HBM-bound: per pass
// 3 vector reads + 1 write of 16 n bytes.
//
// Basis layout: V is (restart + 1) rows of n complex128, row t = basis vector
// t (contiguous, 16-byte aligned): every pass is a unit-stride 128-bit stream.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "rplu_common.cuh"
#include "rplu_internal.h"

namespace rplu {

constexpr int kMgsThreads = 512;

__device__ __forceinline__ double2 block_sum2(double2 v, double2* red) {
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane] : make_double2(0.0, 0.0);
    for (int o = 16; o > 0; o >>= 1) {
      v.x += __shfl_down_sync(0xffffffffu, v.x, o);
      v.y += __shfl_down_sync(0xffffffffu, v.y, o);
    }
  }
  return v;  // valid in thread 0
}

// Sum of the grid's partials in a fixed order (identical in every CTA).
__device__ __forceinline__ double2 grid_total(const double2* part, int nblk, double2* red) {
  double2 v = make_double2(0.0, 0.0);
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
    const double2 pb = __ldcg(part + b);  // written by other SMs: bypass L1
    v.x += pb.x;
    v.y += pb.y;
  }
  v = block_sum2(v, red);
  __shared__ double2 bc;
  if (threadIdx.x == 0) bc = v;
  __syncthreads();
  return bc;
}

__global__ void __launch_bounds__(kMgsThreads) mgs_arnoldi_kernel(const double2* __restrict__ V,
                                                                  long long n, int j,
                                                                  double2* __restrict__ w,
                                                                  double2* __restrict__ vnext,
                                                                  double2* __restrict__ h,
                                                                  double2* __restrict__ part,
                                                                  unsigned* bar) {
  __shared__ double2 red[kMgsThreads / 32];
  const int nblk = gridDim.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double2 hp = make_double2(0.0, 0.0);
  unsigned nb = 0;
  for (int t = 0; t <= j + 1; ++t) {
    const double2* Vp = t > 0 ? V + (long long)(t - 1) * n : nullptr;  // subtract h_{t-1} V_{t-1}
    const double2* Vt = t <= j ? V + (long long)t * n : nullptr;       // then <V_t, w>
    double2 acc = make_double2(0.0, 0.0);
    for (long long i = i0; i < n; i += stride) {
      double2 wi = w[i];
      if (Vp) {
        const double2 pv = cmul_np(hp, __ldg(Vp + i));  // H[t-1, j] * V[:, t-1]
        wi.x = __dsub_rn(wi.x, pv.x);
        wi.y = __dsub_rn(wi.y, pv.y);
        w[i] = wi;
      }
      if (Vt) {  // vdot: conj(v) . w
        const double2 v = __ldg(Vt + i);
        acc.x = fma(v.x, wi.x, fma(v.y, wi.y, acc.x));
        acc.y = fma(v.x, wi.y, fma(-v.y, wi.x, acc.y));
      } else {
        acc.x = fma(wi.x, wi.x, fma(wi.y, wi.y, acc.x));
      }
    }
    acc = block_sum2(acc, red);
    double2* pb = part + (t & 1) * nblk;
    if (threadIdx.x == 0) pb[blockIdx.x] = acc;
    grid_barrier(bar, (unsigned)nblk * (++nb));
    hp = grid_total(pb, nblk, red);
    if (t > j) hp = make_double2(sqrt(hp.x), 0.0);  // H[j+1, j] = ||w||
    if (blockIdx.x == 0 && threadIdx.x == 0) h[t] = hp;
  }
  if (vnext && hp.x > 0.0) {  // V[:, j+1] = w / H[j+1, j]  (Smith: w * (1/h))
    const double s = __ddiv_rn(1.0, hp.x);
    for (long long i = i0; i < n; i += stride) {
      const double2 wi = w[i];
      vnext[i] = make_double2(__dmul_rn(wi.x, s), __dmul_rn(wi.y, s));
    }
  }
}

int mgs_arnoldi_impl(rplu_ctx* ctx, const void* V, long long n, int j, void* w, void* vnext,
                     void* h, cudaStream_t s) {
  int dev = 0, per_sm = 0;
  RPLU_CUDA(cudaGetDevice(&dev));
  RPLU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mgs_arnoldi_kernel,
                                                          kMgsThreads, 0));
  per_sm = std::max(1, std::min(per_sm, 2));
  long long want = (n + kMgsThreads - 1) / kMgsThreads;
  int grid = (int)std::max(1LL, std::min<long long>(want, (long long)ctx->sm_count * per_sm));
  if (int rc = ctx->krylov.ensure(sizeof(double2) * 2 * grid + 64)) return rc;
  double2* part = (double2*)ctx->krylov.ptr;
  unsigned* bar = (unsigned*)(part + 2 * grid);
  RPLU_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned), s));
  const double2* Vp = (const double2*)V;
  double2* wp = (double2*)w;
  double2* vn = (double2*)vnext;
  double2* hp = (double2*)h;
  void* args[] = {&Vp, &n, &j, &wp, &vn, &hp, &part, &bar};
  count_launches(1);
  RPLU_CUDA(cudaLaunchCooperativeKernel((const void*)mgs_arnoldi_kernel, dim3(grid),
                                        dim3(kMgsThreads), args, 0, s));
  return 0;
}

}  // namespace rplu
