// Diagnostics: FP64 pipe peak probe (the roofline denominator for the
// generated-entry paths; MEASURED_PEAKS.json carries no FP64 figure).
#include <cuda_runtime.h>

#include "rplu_internal.h"

namespace rplu {

// 8 independent DFMA chains per thread; the result is stored so the compiler
// cannot drop the work.
__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters, double a, double b) {
  double v0 = threadIdx.x * 1e-9, v1 = v0 + 1e-9, v2 = v0 + 2e-9, v3 = v0 + 3e-9;
  double v4 = v0 + 4e-9, v5 = v0 + 5e-9, v6 = v0 + 6e-9, v7 = v0 + 7e-9;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      v0 = fma(v0, a, b); v1 = fma(v1, a, b); v2 = fma(v2, a, b); v3 = fma(v3, a, b);
      v4 = fma(v4, a, b); v5 = fma(v5, a, b); v6 = fma(v6, a, b); v7 = fma(v7, a, b);
    }
  }
  double s = ((v0 + v1) + (v2 + v3)) + ((v4 + v5) + (v6 + v7));
  if (s == 12345.678) out[blockIdx.x] = s;  // practically never taken
}

// FP64 tensor-core (DMMA m8n8k4) issue rate: 8 independent accumulator
// tiles per warp, the K11 roofline denominator.
__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters) {
  double acc[8][2];
  const double a = 1e-3 * threadIdx.x, b = 0.5;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c][0] = acc[c][1] = c;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[blockIdx.x] = s;
}

int dmma_peak_impl(rplu_ctx* ctx, double* tflops, double* ms_out) {
  int rc;
  if ((rc = ctx->scratch[6].ensure(sizeof(double) * 4096))) return rc;
  double* out = reinterpret_cast<double*>(ctx->scratch[6].ptr);
  const int blocks = ctx->sm_count * 2;
  const int iters = 4096;
  cudaEvent_t e0, e1;
  RPLU_CUDA(cudaEventCreate(&e0));
  RPLU_CUDA(cudaEventCreate(&e1));
  dmma_peak_kernel<<<blocks, 256>>>(out, 64);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    RPLU_CUDA(cudaEventRecord(e0));
    dmma_peak_kernel<<<blocks, 256>>>(out, iters);
    RPLU_CUDA(cudaEventRecord(e1));
    RPLU_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    RPLU_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  // 8 x 8 x 4 FMAs per DMMA, 8 per iteration per warp
  const double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * (blocks * 256 / 32);
  *tflops = flops / (best * 1e-3) / 1e12;
  if (ms_out) *ms_out = best;
  return RPLU_OK;
}

int fp64_peak_impl(rplu_ctx* ctx, double* tflops, double* ms_out) {
  int rc;
  if ((rc = ctx->scratch[6].ensure(sizeof(double) * 4096))) return rc;
  double* out = reinterpret_cast<double*>(ctx->scratch[6].ptr);
  const int blocks = ctx->sm_count * 8;
  const int iters = 2048;
  cudaEvent_t e0, e1;
  RPLU_CUDA(cudaEventCreate(&e0));
  RPLU_CUDA(cudaEventCreate(&e1));
  fp64_peak_kernel<<<blocks, 256>>>(out, 64, 0.999999, 1e-7);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    RPLU_CUDA(cudaEventRecord(e0));
    fp64_peak_kernel<<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
    RPLU_CUDA(cudaEventRecord(e1));
    RPLU_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    RPLU_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double flops = 2.0 * 8 * 16 * (double)iters * 256.0 * blocks;
  *tflops = flops / (best * 1e-3) / 1e12;
  if (ms_out) *ms_out = best;
  return RPLU_OK;
}

}  // namespace rplu
