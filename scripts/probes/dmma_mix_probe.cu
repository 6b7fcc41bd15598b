// Do the FP64 tensor (DMMA m8n8k4) and FP64 vector (DFMA) pipes of a B200 SM
// run concurrently?  A kernel issuing NF DFMA and NM DMMA per loop trip
// (independent chains) against the same kernel with only one kind: if the
// mixed time equals the SUM of the two, the pipes share hardware; if it
// approaches the MAX, they overlap.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int NF, int NM>
__global__ void mix_kernel(double* out, int iters, double a, double b) {
  double v[NF > 0 ? NF : 1];
  double acc[NM > 0 ? NM : 1][2];
#pragma unroll
  for (int c = 0; c < NF; ++c) v[c] = threadIdx.x * 1e-9 + c;
#pragma unroll
  for (int c = 0; c < NM; ++c) acc[c][0] = acc[c][1] = c;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int c = 0; c < NF; ++c) v[c] = fma(v[c], a, b);
#pragma unroll
      for (int c = 0; c < NM; ++c) dmma(acc[c], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < NF; ++c) s += v[c];
#pragma unroll
  for (int c = 0; c < NM; ++c) s += acc[c][0] + acc[c][1];
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
  const int iters = 2048, blocks = sms * 4, threads = 256;
  const double a = 0.999999, b = 1e-7;
  // DFMA: 32 FMA per warp instruction; DMMA m8n8k4: 256 FMA per warp instruction
  float f8 = timeit([&] { mix_kernel<8, 0><<<blocks, threads>>>(out, iters, a, b); });
  float m1 = timeit([&] { mix_kernel<0, 1><<<blocks, threads>>>(out, iters, a, b); });
  float m2 = timeit([&] { mix_kernel<0, 2><<<blocks, threads>>>(out, iters, a, b); });
  float m4 = timeit([&] { mix_kernel<0, 4><<<blocks, threads>>>(out, iters, a, b); });
  float x81 = timeit([&] { mix_kernel<8, 1><<<blocks, threads>>>(out, iters, a, b); });
  float x82 = timeit([&] { mix_kernel<8, 2><<<blocks, threads>>>(out, iters, a, b); });
  float x84 = timeit([&] { mix_kernel<8, 4><<<blocks, threads>>>(out, iters, a, b); });
  const double warps = (double)blocks * threads / 32, trips = 4.0 * iters;
  printf("DFMA x8 only:        %.3f ms  (%.2f TFLOP/s)\n", f8, 2.0 * 32 * 8 * trips * warps / f8 / 1e9);
  printf("DMMA x1 / x2 / x4:   %.3f / %.3f / %.3f ms  (x4: %.2f TFLOP/s)\n", m1, m2, m4,
         2.0 * 256 * 4 * trips * warps / m4 / 1e9);
  printf("DFMA x8 + DMMA x1:   %.3f ms  (sum %.3f, max %.3f)\n", x81, f8 + m1, f8 > m1 ? f8 : m1);
  printf("DFMA x8 + DMMA x2:   %.3f ms  (sum %.3f, max %.3f)\n", x82, f8 + m2, f8 > m2 ? f8 : m2);
  printf("DFMA x8 + DMMA x4:   %.3f ms  (sum %.3f, max %.3f)\n", x84, f8 + m4, f8 > m4 ? f8 : m4);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
