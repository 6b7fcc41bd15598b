// Certified row-norm upper bounds for Cauchy-like matrices from a quadtree
// interaction plan (reference rplu.treebounds,
// pkg/src/rplu/treebounds.py:183-242, Alg C.2).
//
//   H_s = sum_{j in s} B_:,j B_:,j^H          (p x p, every source node s)
//   u_i = sum_{(s,alpha) in A_leaf(i)} alpha * Re(g_i H_s g_i^H)
//       + sum_{s in E_leaf(i)} sum_{j in s} |g_i . B_:,j|^2 / |x_i - y_j|^2
//
// Gram matrices: one warp per source leaf (lanes over the p^2 entries), then
// one warp per node summing the leaves below it.  Bounds: one CTA per target
// leaf, one thread per target point, the node Grams read through L1/L2
// (broadcast: every thread of the CTA uses the same H_s).  Work per step is
// O((n+m)|A| p^2) instead of the exact norms' O(n m p).
#include <cuda_runtime.h>
#include <stdint.h>

#include "rplu_common.cuh"
#include "rplu_internal.h"

namespace rplu {

struct TreeParams {
  long long n, m;
  int p;
  long long n_tleaves, n_snodes, n_sleaves;
  const long long *tperm, *tstart;
  const long long *agg_start, *agg_node;
  const double* agg_alpha;
  const long long *ex_start, *ex_leaf;
  const long long *spts, *sstart;
  const long long *bstart, *bleaf;
  const double2 *x, *y, *G, *Bt;
  double2* Hleaf;  // n_sleaves x p x p
  double2* Hnode;  // n_snodes x p x p
  double* u;       // n
};

__device__ __forceinline__ double2 cfma_conj(double2 acc, double2 a, double2 b) {
  // acc + a * conj(b)
  acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
  acc.y = fma(a.y, b.x, fma(-a.x, b.y, acc.y));
  return acc;
}

template <int P>
__global__ void tree_gram_leaf_kernel(TreeParams q) {
  const long long leaf = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (leaf >= q.n_sleaves) return;
  double2 acc[2] = {make_double2(0, 0), make_double2(0, 0)};
  for (long long k = q.sstart[leaf]; k < q.sstart[leaf + 1]; ++k) {
    const long long j = q.spts[k];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h;
      if (e < P * P) acc[h] = cfma_conj(acc[h], q.Bt[j * P + e / P], q.Bt[j * P + e % P]);
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int e = lane + 32 * h;
    if (e < P * P) q.Hleaf[leaf * P * P + e] = acc[h];
  }
}

template <int P>
__global__ void tree_gram_node_kernel(TreeParams q) {
  const long long node = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (node >= q.n_snodes) return;
  double2 acc[2] = {make_double2(0, 0), make_double2(0, 0)};
  for (long long k = q.bstart[node]; k < q.bstart[node + 1]; ++k) {
    const long long lf = q.bleaf[k];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h;
      if (e < P * P) {
        const double2 v = q.Hleaf[lf * P * P + e];
        acc[h].x += v.x;
        acc[h].y += v.y;
      }
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int e = lane + 32 * h;
    if (e < P * P) q.Hnode[node * P * P + e] = acc[h];
  }
}

template <int P>
__global__ void __launch_bounds__(64) tree_bounds_kernel(TreeParams q) {
  const long long leaf = blockIdx.x;
  const long long a0 = q.agg_start[leaf], a1 = q.agg_start[leaf + 1];
  const long long e0 = q.ex_start[leaf], e1 = q.ex_start[leaf + 1];
  for (long long k = q.tstart[leaf] + threadIdx.x; k < q.tstart[leaf + 1]; k += blockDim.x) {
    const long long i = q.tperm[k];
    double2 g[P];
#pragma unroll
    for (int l = 0; l < P; ++l) g[l] = q.G[i * P + l];
    const double2 xi = q.x[i];
    double acc = 0.0;
    for (long long e = a0; e < a1; ++e) {  // aggregated: alpha * Re(g H g^H)
      const double2* H = q.Hnode + q.agg_node[e] * P * P;
      double val = 0.0;
#pragma unroll
      for (int a = 0; a < P; ++a) {
        double2 t = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < P; ++b) t = cfma_conj(t, H[a * P + b], g[b]);  // (H conj(g))_a
        val = fma(g[a].x, t.x, fma(-g[a].y, t.y, val));                 // Re(g_a t_a)
      }
      acc = fma(q.agg_alpha[e], val, acc);
    }
    for (long long e = e0; e < e1; ++e) {  // exact: sum over the source leaf's points
      const long long lf = q.ex_leaf[e];
      for (long long s = q.sstart[lf]; s < q.sstart[lf + 1]; ++s) {
        const long long j = q.spts[s];
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int l = 0; l < P; ++l) {
          const double2 b = q.Bt[j * P + l];
          re = fma(g[l].x, b.x, fma(-g[l].y, b.y, re));
          im = fma(g[l].x, b.y, fma(g[l].y, b.x, im));
        }
        const double2 yj = q.y[j];
        const double dr = xi.x - yj.x, di = xi.y - yj.y;
        acc += __ddiv_rn(fma(re, re, im * im), fma(dr, dr, di * di));
      }
    }
    q.u[i] = acc;
  }
}

#define RPLU_TREE_P_SWITCH(p, CALL)                \
  switch (p) {                                     \
    case 1: { constexpr int PP = 1; CALL; } break; \
    case 2: { constexpr int PP = 2; CALL; } break; \
    case 3: { constexpr int PP = 3; CALL; } break; \
    case 4: { constexpr int PP = 4; CALL; } break; \
    case 5: { constexpr int PP = 5; CALL; } break; \
    case 6: { constexpr int PP = 6; CALL; } break; \
    case 7: { constexpr int PP = 7; CALL; } break; \
    case 8: { constexpr int PP = 8; CALL; } break; \
    default: break;                                \
  }

int tree_bounds_impl(rplu_ctx* ctx, const rplu_tree_plan* plan, const void* x, const void* y,
                     const void* G, const void* Bt, double* u, cudaStream_t s) {
  TreeParams q{};
  q.n = plan->n;
  q.m = plan->m;
  q.p = plan->p;
  q.n_tleaves = plan->n_tleaves;
  q.n_snodes = plan->n_snodes;
  q.n_sleaves = plan->n_sleaves;
  q.tperm = reinterpret_cast<const long long*>(plan->tperm);
  q.tstart = reinterpret_cast<const long long*>(plan->tstart);
  q.agg_start = reinterpret_cast<const long long*>(plan->agg_start);
  q.agg_node = reinterpret_cast<const long long*>(plan->agg_node);
  q.agg_alpha = plan->agg_alpha;
  q.ex_start = reinterpret_cast<const long long*>(plan->ex_start);
  q.ex_leaf = reinterpret_cast<const long long*>(plan->ex_leaf);
  q.spts = reinterpret_cast<const long long*>(plan->spts);
  q.sstart = reinterpret_cast<const long long*>(plan->sstart);
  q.bstart = reinterpret_cast<const long long*>(plan->bstart);
  q.bleaf = reinterpret_cast<const long long*>(plan->bleaf);
  q.x = reinterpret_cast<const double2*>(x);
  q.y = reinterpret_cast<const double2*>(y);
  q.G = reinterpret_cast<const double2*>(G);
  q.Bt = reinterpret_cast<const double2*>(Bt);
  q.u = u;
  const size_t pp = (size_t)q.p * q.p;
  int rc;
  if ((rc = ctx->scratch[6].ensure(sizeof(double2) * pp * (size_t)(q.n_sleaves + q.n_snodes))))
    return rc;
  q.Hleaf = reinterpret_cast<double2*>(ctx->scratch[6].ptr);
  q.Hnode = q.Hleaf + pp * q.n_sleaves;
  const unsigned gl = (unsigned)((q.n_sleaves + 7) / 8), gn = (unsigned)((q.n_snodes + 7) / 8);
  RPLU_TREE_P_SWITCH(q.p, (tree_gram_leaf_kernel<PP><<<gl, 256, 0, s>>>(q)));
  RPLU_TREE_P_SWITCH(q.p, (tree_gram_node_kernel<PP><<<gn, 256, 0, s>>>(q)));
  RPLU_TREE_P_SWITCH(q.p, (tree_bounds_kernel<PP><<<(unsigned)q.n_tleaves, 64, 0, s>>>(q)));
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

}  // namespace rplu
