// FP64 tensor (DMMA, mma.sync m8n8k4 f64) vs DFMA throughput probe on one B200.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
  double acc[CHAINS][2];
  double a = 1e-3 * threadIdx.x, b = 0.5;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c][0] = acc[c][1] = c;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) dmma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1234.5) out[blockIdx.x] = s;
}

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double v[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = threadIdx.x * 1e-9 + c;
  for (int k = 0; k < iters; ++k)
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = fma(v[c], a, b);
  double s = 0;
  for (int c = 0; c < 8; ++c) s += v[c];
  if (s == 1234.5) out[blockIdx.x] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  double* out; cudaMalloc(&out, 1 << 20);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps, threads = 32 * wpb;
      float ms = timeit([&] { dmma_kernel<8><<<blocks, threads>>>(out, iters); });
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (blocks * wpb);
      printf("DMMA chains=8 warps/blk=%d blk/SM=%d: %.3f ms  %.2f TFLOP/s\n", wpb, bps, ms,
             flops / ms / 1e9);
    }
  }
  {
    int blocks = sms * 4, threads = 256;
    float ms = timeit([&] { dmma_kernel<4><<<blocks, threads>>>(out, iters); });
    double flops = 2.0 * 8 * 8 * 4 * 4.0 * iters * (blocks * 8);
    printf("DMMA chains=4 8w x4: %.2f TFLOP/s\n", flops / ms / 1e9);
  }
  {
    int blocks = sms * 8, threads = 256, it = 2048;
    float ms = timeit([&] { dfma_kernel<<<blocks, threads>>>(out, it, 0.999999, 1e-7); });
    double flops = 2.0 * 8 * 16 * (double)it * threads * blocks;
    printf("DFMA: %.2f TFLOP/s\n", flops / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
