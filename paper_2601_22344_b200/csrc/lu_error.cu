// K11: fused L·U reconstruction error on the FP64 tensor cores.
//
// Reference: EliminationTrace.approximation() = L @ U (dense_pivots.py:82-83)
// and the error the sweeps report, ||A - L U||_F / ||A||_F (cli.py:151-157,
// :200-206).  Here  sum (A - X Y)^2  and  sum A^2  come out of one kernel:
// the X Y tile is accumulated by DMMA (mma.sync m8n8k4 f64, the only FP64
// tensor-core path on sm_100a: tcgen05 has no f64 kind), the subtraction, the
// square and the sum run in the epilogue on the accumulator registers, and
// no panel of L U or A - L U ever reaches memory.
//
// Layout: X^T (k x n, the Lt layout the dense loop fills) and Y (k x m, U)
// are first copied into zero-padded fp64 panels Xp (Kp x Np) and Yp (Kp x Mp)
// (Kp = k rounded up to 16, Np / Mp to 128), so the main loop has no bounds
// tests; a complex128 A is handled as two real products over augmented
// factors, Re(LU) = [Lr, -Li][Ur; Ui] and Im(LU) = [Lr, Li][Ui; Ur].
//
// Main kernel: persistent, one 256-thread CTA per SM walking 128 x 128
// output tiles in grouped order (8 tile-rows share their Y panels in L2).
// Per k-chunk of 16 a 3-stage cp.async ring stages X (16 x 128) and Y
// (16 x 128) in shared memory with rows padded to 132 doubles (every
// fragment load is bank-conflict free); 8 warps as 2 x 4, each warp owning a
// 64 x 32 sub-tile = 8 x 4 DMMA tiles = 64 fp64 accumulators per thread.
// The epilogue reads the A tile (prefetched into L2 when the tile starts)
// once.  Per-CTA partial sums are written in a fixed order and summed by one
// CTA, so the result is deterministic.
#include <cuda_runtime.h>

#include <cstdlib>

#include "rplu_common.cuh"
#include "rplu_internal.h"

namespace rplu {
namespace {

constexpr int kBK = 16, kStages = 3;
constexpr int kGroup = 8;

// Tile configuration: CTA tile BM x BN, WM x WN warps, each warp owning a
// (BM/WM) x (BN/WN) sub-tile of 8x8 DMMA tiles.
template <int BM_, int BN_, int WM_, int WN_, int MINB_>
struct LuCfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, MINB = MINB_;
  static constexpr int kThreads = WM * WN * 32;
  static constexpr int MT = BM / WM / 8, NT = BN / WN / 8;
  static constexpr int LDX = BM + 4, LDY = BN + 4;  // == 4 mod 16: conflict-free fragments
  struct Smem {
    double x[kStages][kBK][LDX];
    double y[kStages][kBK][LDY];
    double red[2][kThreads / 32];
  };
};
// 64 x 64 tiles, 4 warps of 32 x 32, four CTAs per SM: each CTA's epilogue,
// prologue and barriers overlap the other CTAs' tensor-core work (measured
// at C3: 31.1 TFLOP/s against 29.6 for 128 x 64 x 2 CTAs and 27.8 for
// 128 x 128 x 1 CTA, RPLU_K11_CFG sweep).
using LuDefault = LuCfg<64, 64, 2, 2, 4>;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// D = A(8x4, row) * B(4x8, col) + D; lane l holds A[l/4][l%4], B[l%4][l/4],
// D[l/4][2(l%4) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// the pair A[r][c], A[r][c+1] (c even); one 16-byte load when A is a real
// double matrix with an even leading dimension and a 16-byte aligned base
template <typename TA, int AS>
__device__ __forceinline__ void load_pair(const TA* p, bool vec_ok, bool has1, double& a0,
                                          double& a1) {
  if constexpr (sizeof(TA) == 8 && AS == 1) {
    if (vec_ok && has1) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(p));
      a0 = v.x;
      a1 = v.y;
      return;
    }
  }
  a0 = static_cast<double>(__ldg(p));
  a1 = has1 ? static_cast<double>(__ldg(p + AS)) : 0.0;
}

// AS: element stride of A in TA units (1 real, 2 one part of complex128)
template <class C, typename TA, int AS>
__global__ void __launch_bounds__(C::kThreads, C::MINB)
lu_error_kernel(const TA* __restrict__ A, long long lda, int n, int m,
                const double* __restrict__ Xp, long long ldxp, const double* __restrict__ Yp,
                long long ldyp, int kp, int tiles_m, int tiles_n, double* __restrict__ partials) {
  constexpr int BM = C::BM, BN = C::BN, MT = C::MT, NT = C::NT, NTHR = C::kThreads;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  auto& sm = *reinterpret_cast<typename C::Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / C::WN, wn = warp % C::WN;
  const int g = lane >> 2, q = lane & 3;
  const int nk = kp / kBK;
  const int tiles = tiles_m * tiles_n;
  const bool vec_ok = ((lda * AS) % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  double s_err = 0.0, s_a = 0.0;

  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int per_group = kGroup * tiles_n;
    const int first_m = (tile / per_group) * kGroup;
    const int gsz = min(tiles_m - first_m, kGroup);
    const int in_group = tile % per_group;
    const int i0 = (first_m + in_group % gsz) * BM;
    const int j0 = (in_group / gsz) * BN;

    // A tile -> L2 while the product runs (read once, in the epilogue)
    {
      constexpr int kLineElems = 128 / (sizeof(TA) * AS) > 0 ? 128 / (sizeof(TA) * AS) : 1;
      constexpr int kLinesPerRow = (BN + kLineElems - 1) / kLineElems;
      for (int idx = tid; idx < BM * kLinesPerRow; idx += NTHR) {
        const int r = i0 + idx / kLinesPerRow;
        const int c = j0 + (idx % kLinesPerRow) * kLineElems;
        if (r < n && c < m) {
          const TA* p = A + (long long)r * lda + (long long)c * AS;
          asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
        }
      }
    }

    auto load_stage = [&](int stage, int kc) {
      const double* xs = Xp + (long long)kc * kBK * ldxp + i0;
      const double* ys = Yp + (long long)kc * kBK * ldyp + j0;
#pragma unroll
      for (int idx = tid; idx < kBK * BM / 2; idx += NTHR) {
        const int r = idx / (BM / 2), c = (idx % (BM / 2)) * 2;
        cp_async16(&sm.x[stage][r][c], xs + (long long)r * ldxp + c);
      }
#pragma unroll
      for (int idx = tid; idx < kBK * BN / 2; idx += NTHR) {
        const int r = idx / (BN / 2), c = (idx % (BN / 2)) * 2;
        cp_async16(&sm.y[stage][r][c], ys + (long long)r * ldyp + c);
      }
    };

    double acc[MT][NT][2];
#pragma unroll
    for (int a = 0; a < MT; ++a)
#pragma unroll
      for (int b = 0; b < NT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
      if (s < nk) load_stage(s, s);
      cp_async_commit();
    }
    for (int kc = 0; kc < nk; ++kc) {
      cp_async_wait<kStages - 2>();
      __syncthreads();
      const int next = kc + kStages - 1;
      if (next < nk) load_stage(next % kStages, next);
      cp_async_commit();
      const int st = kc % kStages;
#pragma unroll
      for (int kk = 0; kk < kBK; kk += 4) {
        double af[MT], bf[NT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
          af[mt] = sm.x[st][kk + q][wm * (BM / C::WM) + mt * 8 + g];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          bf[nt] = sm.y[st][kk + q][wn * (BN / C::WN) + nt * 8 + g];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt], af[mt], bf[nt]);
      }
    }
    cp_async_wait<0>();
    __syncthreads();  // the next tile's prologue overwrites the ring

    // epilogue: (A - X Y)^2 and A^2 straight from the accumulators.  The A
    // values are loaded in batches of EB row-tiles before any is consumed,
    // so a batch costs one L2 round trip (loads interleaved with their use
    // serialise into one round trip per load).
    constexpr int EB = MT >= 2 ? 2 : 1;
#pragma unroll
    for (int mb = 0; mb < MT; mb += EB) {
      double av[EB][NT][2];
#pragma unroll
      for (int e = 0; e < EB; ++e) {
        const int row = i0 + wm * (BM / C::WM) + (mb + e) * 8 + g;
        const TA* arow = A + (long long)min(row, n - 1) * lda;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int col = j0 + wn * (BN / C::WN) + nt * 8 + 2 * q;
          if (row < n && col < m)
            load_pair<TA, AS>(arow + (long long)col * AS, vec_ok, col + 1 < m, av[e][nt][0],
                              av[e][nt][1]);
          else
            av[e][nt][0] = av[e][nt][1] = 0.0;
        }
      }
#pragma unroll
      for (int e = 0; e < EB; ++e) {
        const int row = i0 + wm * (BM / C::WM) + (mb + e) * 8 + g;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int col = j0 + wn * (BN / C::WN) + nt * 8 + 2 * q;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (row < n && col + h < m) {
              const double a = av[e][nt][h];
              const double d = a - acc[mb + e][nt][h];
              s_err = fma(d, d, s_err);
              s_a = fma(a, a, s_a);
            }
          }
        }
      }
    }
  }

  s_err = warp_sum(s_err);
  s_a = warp_sum(s_a);
  if (lane == 0) {
    sm.red[0][warp] = s_err;
    sm.red[1][warp] = s_a;
  }
  __syncthreads();
  if (tid == 0) {
    double e = 0.0, a = 0.0;
    for (int w = 0; w < NTHR / 32; ++w) {
      e += sm.red[0][w];
      a += sm.red[1][w];
    }
    partials[2 * blockIdx.x] = e;
    partials[2 * blockIdx.x + 1] = a;
  }
}

// sums the per-CTA partials of `passes` launches in a fixed order
__global__ void lu_error_reduce_kernel(const double* partials, int count, double* out) {
  __shared__ double se[32], sa[32];
  double e = 0.0, a = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    e += partials[2 * i];
    a += partials[2 * i + 1];
  }
  e = warp_sum(e);
  a = warp_sum(a);
  if ((threadIdx.x & 31) == 0) {
    se[threadIdx.x >> 5] = e;
    sa[threadIdx.x >> 5] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double te = 0.0, ta = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      te += se[w];
      ta += sa[w];
    }
    out[0] = te;
    out[1] = ta;
  }
}

// Zero-padded fp64 panel P (kp x np_, row stride np_) from a k x n factor
// (row stride ld, element type by dtype).  Complex factors: part selects the
// augmented layout: rows [0,k) take `first` (0 = re, 1 = im), rows [k,2k)
// take `second` with sign `sgn2`.
template <typename T>
__global__ void lu_pad_kernel(const T* src, long long ld, int k, int n, double* dst, int kp,
                              long long np_) {
  const long long total = (long long)kp * np_;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(idx / np_);
    const long long i = idx % np_;
    double v = 0.0;
    if (t < k && i < n) v = static_cast<double>(src[(long long)t * ld + i]);
    dst[idx] = v;
  }
}

__global__ void lu_pad_complex_kernel(const double2* src, long long ld, int k, int n,
                                      double* dst, int kp, long long np_, int first, int second,
                                      double sgn2) {
  const long long total = (long long)kp * np_;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(idx / np_);
    const long long i = idx % np_;
    double v = 0.0;
    if (i < n && t < 2 * k) {
      const double2 z = src[(long long)(t % k) * ld + i];
      if (t < k) v = first ? z.y : z.x;
      else v = sgn2 * (second ? z.y : z.x);
    }
    dst[idx] = v;
  }
}

inline long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }

template <class C>
int lu_error_run(rplu_ctx* ctx, int dtype, const void* A, long long lda, long long n,
                 long long m, const void* Xt, long long ldx, const void* Y, long long ldy,
                 long long k, double* out_sq, double* kernel_ms, cudaStream_t s) {
  const bool cplx = dtype == RPLU_C128;
  const long long kk = cplx ? 2 * k : k;
  const long long kp = round_up(kk, kBK);
  const long long np_ = round_up(n, C::BM), mp = round_up(m, C::BN);
  const int tiles_m = (int)(np_ / C::BM), tiles_n = (int)(mp / C::BN);
  const int grid =
      (int)std::min<long long>((long long)tiles_m * tiles_n, (long long)ctx->sm_count * C::MINB);
  const int passes = cplx ? 2 : 1;
  const size_t xbytes = sizeof(double) * kp * np_, ybytes = sizeof(double) * kp * mp;
  int rc;
  if ((rc = ctx->lu_pad.ensure(xbytes + ybytes))) return rc;
  if ((rc = ctx->lu_part.ensure(sizeof(double) * (2 * (size_t)grid * passes + 2)))) return rc;
  double* xp = reinterpret_cast<double*>(ctx->lu_pad.ptr);
  double* yp = xp + kp * np_;
  double* part = reinterpret_cast<double*>(ctx->lu_part.ptr);
  double* res = part + 2 * (size_t)grid * passes;
  const size_t smem = sizeof(typename C::Smem);
  RPLU_CUDA(cudaFuncSetAttribute(lu_error_kernel<C, double, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  RPLU_CUDA(cudaFuncSetAttribute(lu_error_kernel<C, float, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  RPLU_CUDA(cudaFuncSetAttribute(lu_error_kernel<C, double, 2>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int pad_grid = ctx->sm_count * 4;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (kernel_ms) {
    RPLU_CUDA(cudaEventCreate(&e0));
    RPLU_CUDA(cudaEventCreate(&e1));
  }
  float total_ms = 0.f;
  long long launches = 0;
  for (int pass = 0; pass < passes; ++pass) {
    if (!cplx) {
      if (dtype == RPLU_F64) {
        lu_pad_kernel<double><<<pad_grid, 256, 0, s>>>(static_cast<const double*>(Xt), ldx,
                                                       (int)k, (int)n, xp, (int)kp, np_);
        lu_pad_kernel<double><<<pad_grid, 256, 0, s>>>(static_cast<const double*>(Y), ldy,
                                                       (int)k, (int)m, yp, (int)kp, mp);
      } else {
        lu_pad_kernel<float><<<pad_grid, 256, 0, s>>>(static_cast<const float*>(Xt), ldx,
                                                      (int)k, (int)n, xp, (int)kp, np_);
        lu_pad_kernel<float><<<pad_grid, 256, 0, s>>>(static_cast<const float*>(Y), ldy,
                                                      (int)k, (int)m, yp, (int)kp, mp);
      }
    } else {
      // pass 0: Re(LU) = [Lr, -Li] [Ur; Ui];  pass 1: Im(LU) = [Lr, Li] [Ui; Ur]
      const double2* L2 = static_cast<const double2*>(Xt);
      const double2* U2 = static_cast<const double2*>(Y);
      lu_pad_complex_kernel<<<pad_grid, 256, 0, s>>>(L2, ldx, (int)k, (int)n, xp, (int)kp, np_,
                                                     0, 1, pass == 0 ? -1.0 : 1.0);
      lu_pad_complex_kernel<<<pad_grid, 256, 0, s>>>(U2, ldy, (int)k, (int)m, yp, (int)kp, mp,
                                                     pass == 0 ? 0 : 1, pass == 0 ? 1 : 0, 1.0);
    }
    RPLU_CUDA(cudaGetLastError());
    if (kernel_ms) RPLU_CUDA(cudaEventRecord(e0, s));
    double* pp = part + 2 * (size_t)grid * pass;
    if (dtype == RPLU_F64)
      lu_error_kernel<C, double, 1><<<grid, C::kThreads, smem, s>>>(
          static_cast<const double*>(A), lda, (int)n, (int)m, xp, np_, yp, mp, (int)kp, tiles_m,
          tiles_n, pp);
    else if (dtype == RPLU_F32)
      lu_error_kernel<C, float, 1><<<grid, C::kThreads, smem, s>>>(
          static_cast<const float*>(A), lda, (int)n, (int)m, xp, np_, yp, mp, (int)kp, tiles_m,
          tiles_n, pp);
    else
      lu_error_kernel<C, double, 2><<<grid, C::kThreads, smem, s>>>(
          static_cast<const double*>(A) + pass, 2 * lda, (int)n, (int)m, xp, np_, yp, mp,
          (int)kp, tiles_m, tiles_n, pp);
    RPLU_CUDA(cudaGetLastError());
    if (kernel_ms) {
      RPLU_CUDA(cudaEventRecord(e1, s));
      RPLU_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      RPLU_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      total_ms += ms;
    }
    launches += 3;
  }
  lu_error_reduce_kernel<<<1, 256, 0, s>>>(part, grid * passes, res);
  RPLU_CUDA(cudaGetLastError());
  RPLU_CUDA(cudaMemcpyAsync(out_sq, res, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  RPLU_CUDA(cudaStreamSynchronize(s));
  count_launches(launches + 1);
  if (kernel_ms) {
    *kernel_ms = total_ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return RPLU_OK;
}

}  // namespace

int lu_error_impl(rplu_ctx* ctx, int dtype, const void* A, long long lda, long long n,
                  long long m, const void* Xt, long long ldx, const void* Y, long long ldy,
                  long long k, double* out_sq, double* kernel_ms, cudaStream_t s) {
  if (n <= 0 || m <= 0 || k < 0 || lda < m || (k > 0 && (ldx < n || ldy < m)) ||
      n > (1LL << 31) - 256 || m > (1LL << 31) - 256) {
    set_error("rplu_lu_error: bad shape / leading dimension");
    return RPLU_ERR_ARG;
  }
  if (dtype != RPLU_F32 && dtype != RPLU_F64 && dtype != RPLU_C128) {
    set_error("rplu_lu_error: unsupported dtype");
    return RPLU_ERR_ARG;
  }
  // RPLU_K11_CFG (experiment knob): 0 = 64x64 tiles, 4 warps, 4 CTAs/SM
  // (default); 1 = 128x128, 8 warps of 64x32, 1 CTA/SM; 2 = 128x128, 16
  // warps of 32x32, 1 CTA/SM; 3 = 128x64, 8 warps, 2 CTAs/SM; 4 = 64x128,
  // 8 warps, 2 CTAs/SM
  static const int cfg = [] {
    const char* e = getenv("RPLU_K11_CFG");
    return e ? atoi(e) : 0;
  }();
  if (cfg == 1)
    return lu_error_run<LuCfg<128, 128, 2, 4, 1>>(ctx, dtype, A, lda, n, m, Xt, ldx, Y, ldy, k,
                                                  out_sq, kernel_ms, s);
  if (cfg == 2)
    return lu_error_run<LuCfg<128, 128, 4, 4, 1>>(ctx, dtype, A, lda, n, m, Xt, ldx, Y, ldy, k,
                                                  out_sq, kernel_ms, s);
  if (cfg == 3)
    return lu_error_run<LuCfg<128, 64, 4, 2, 2>>(ctx, dtype, A, lda, n, m, Xt, ldx, Y, ldy, k,
                                                out_sq, kernel_ms, s);
  if (cfg == 4)
    return lu_error_run<LuCfg<64, 128, 2, 4, 2>>(ctx, dtype, A, lda, n, m, Xt, ldx, Y, ldy, k,
                                                 out_sq, kernel_ms, s);
  return lu_error_run<LuDefault>(ctx, dtype, A, lda, n, m, Xt, ldx, Y, ldy, k, out_sq,
                                 kernel_ms, s);
}

}  // namespace rplu
