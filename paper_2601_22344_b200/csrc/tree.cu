// Certified row-norm upper bounds for Cauchy-like matrices from a quadtree
// interaction plan (reference rplu.treebounds,
// pkg/src/rplu/treebounds.py:183-242, Alg C.2).
//
//   H_s = sum_{j in s} B_:,j B_:,j^H          (p x p, every source node s)
//   u_i = sum_{(s,alpha) in A_leaf(i)} alpha * Re(g_i H_s g_i^H)
//       + sum_{s in E_leaf(i)} sum_{j in s} |g_i . B_:,j|^2 / |x_i - y_j|^2
//
// Gram matrices: one warp per source leaf (lanes over the p^2 entries), then
// one warp per node summing the leaves below it.  Bounds: one warp per target
// leaf folds the leaf's aggregated interactions into one p x p matrix, then
// evaluates one quadratic form per target point.  Work per step is
// O(m p^2 + |leaves| |A| p^2 + n p^2 + exact pairs) instead of the exact
// norms' O(n m p).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

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
  const long long *cstart, *cidx, *leaf_node;
  const double2 *x, *y, *G, *Bt;
  double2* Hnode;  // n_snodes x p x p
  double* u;       // n
};

__device__ __forceinline__ double2 cfma_conj(double2 acc, double2 a, double2 b) {
  // acc + a * conj(b)
  acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
  acc.y = fma(a.y, b.x, fma(-a.x, b.y, acc.y));
  return acc;
}

// Leaf Grams: one warp per source leaf.  For p^2 <= 16 the warp splits into
// 32 / p^2 groups of p^2 lanes (one entry per lane); group g sums the leaf's
// points g, g + NG, ... and the group sums are added in group order through
// shuffles (deterministic), so every lane is busy and NG point loads are in
// flight per iteration.
template <int P>
__global__ void tree_gram_leaf_kernel(TreeParams q) {
  const long long leaf = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (leaf >= q.n_sleaves) return;
  constexpr int E = P * P;
  const long long k0 = q.sstart[leaf], k1 = q.sstart[leaf + 1];
  if constexpr (E <= 16) {
    constexpr int NG = 32 / E;
    const int e = lane % E, g = lane / E;
    double2 acc = make_double2(0, 0);
    if (g < NG)
      for (long long k = k0 + g; k < k1; k += NG) {
        const long long j = q.spts[k];
        acc = cfma_conj(acc, q.Bt[j * P + e / P], q.Bt[j * P + e % P]);
      }
#pragma unroll
    for (int h = 1; h < NG; ++h) {
      const double ax = __shfl_sync(0xffffffffu, acc.x, e + E * h);
      const double ay = __shfl_sync(0xffffffffu, acc.y, e + E * h);
      if (g == 0) { acc.x += ax; acc.y += ay; }
    }
    if (g == 0) q.Hnode[q.leaf_node[leaf] * E + e] = acc;
  } else {
    double2 acc[2] = {make_double2(0, 0), make_double2(0, 0)};
    for (long long k = k0; k < k1; ++k) {
      const long long j = q.spts[k];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = lane + 32 * h;
        if (e < E) acc[h] = cfma_conj(acc[h], q.Bt[j * P + e / P], q.Bt[j * P + e % P]);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h;
      if (e < E) q.Hnode[q.leaf_node[leaf] * E + e] = acc[h];
    }
  }
}

// Internal node Grams bottom-up, one launch per tree level (deepest first):
// one warp per node, lanes over the P*P entries, H_node = sum of its
// children's H in child order (the reference's _gram_bottom_up,
// treebounds.py:196-210).  O(n_snodes p^2) in ~depth short launches.  (A
// warp — or CTA — per node summing every leaf below it made the root, ~60k
// leaves at C4, a serial 1-7 ms chain.)
template <int P>
__global__ void __launch_bounds__(256) tree_gram_level_kernel(TreeParams q,
                                                              const long long* __restrict__ nodes,
                                                              long long count) {
  const long long w = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= count) return;
  const long long node = nodes[w];
  const long long c0 = q.cstart[node], c1 = q.cstart[node + 1];
  for (int e = lane; e < P * P; e += 32) {
    double2 acc = make_double2(0.0, 0.0);
    for (long long c = c0; c < c1; ++c) {
      const double2 v = q.Hnode[q.cidx[c] * P * P + e];
      acc.x += v.x;
      acc.y += v.y;
    }
    q.Hnode[node * P * P + e] = acc;
  }
}

// All internal levels in one cooperative launch: warps stride over the
// level's nodes, one grid barrier between levels (the per-level launches
// cost ~15 x 5 us at C4 size).
constexpr int kMaxLevels = 62;
struct LevelTable {
  long long start[kMaxLevels + 1];
  int n;
};

template <int P>
__global__ void __launch_bounds__(256) tree_gram_levels_kernel(TreeParams q,
                                                               const long long* __restrict__ nodes,
                                                               LevelTable lt, unsigned* bar) {
  const int lane = threadIdx.x & 31;
  const long long w0 = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const long long nw = (long long)gridDim.x * 8;
  unsigned nb = 0;
  for (int l = 0; l < lt.n; ++l) {
    for (long long w = lt.start[l] + w0; w < lt.start[l + 1]; w += nw) {
      const long long node = nodes[w];
      const long long c0 = q.cstart[node], c1 = q.cstart[node + 1];
      for (int e = lane; e < P * P; e += 32) {
        double2 acc = make_double2(0.0, 0.0);
        for (long long c = c0; c < c1; ++c) {
          const double2 v = __ldcg(q.Hnode + q.cidx[c] * P * P + e);  // written this launch
          acc.x += v.x;
          acc.y += v.y;
        }
        q.Hnode[node * P * P + e] = acc;
      }
    }
    if (l + 1 < lt.n) grid_barrier(bar, gridDim.x * (++nb));
  }
}

// One warp per target leaf.  The aggregated part is linear in the Grams, so
// the warp first folds the leaf's interaction list into one p x p matrix
// M = sum_(s,alpha) alpha H_s in shared memory (lanes over the p^2 entries;
// ~34 nodes per leaf at C4), then each lane evaluates Re(g_i M g_i^H) for its
// target points: O(p^2) per point instead of O(|A| p^2).  The exact part
// sums |g_i . B_:,j|^2 / |x_i - y_j|^2 over the leaf's exact source leaves.
constexpr int kTreeWarps = 4;

template <int P>
__global__ void __launch_bounds__(32 * kTreeWarps) tree_bounds_kernel(TreeParams q) {
  __shared__ double2 Ms[kTreeWarps][P * P];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long leaf = (long long)blockIdx.x * kTreeWarps + wid;
  if (leaf >= q.n_tleaves) return;  // warp-uniform
  const long long a0 = q.agg_start[leaf], a1 = q.agg_start[leaf + 1];
  const long long e0 = q.ex_start[leaf], e1 = q.ex_start[leaf + 1];
  constexpr int E = P * P;
  if constexpr (E <= 16) {
    // 32 / E lane groups split the interaction list (more loads in flight),
    // group sums added in group order (deterministic)
    constexpr int NG = 32 / E;
    const int c = lane % E, g = lane / E;
    double2 acc = make_double2(0.0, 0.0);
    if (g < NG)
#pragma unroll 2
      for (long long e = a0 + g; e < a1; e += NG) {
        const double al = __ldg(q.agg_alpha + e);
        const double2 v = q.Hnode[__ldg(q.agg_node + e) * E + c];
        acc.x = fma(al, v.x, acc.x);
        acc.y = fma(al, v.y, acc.y);
      }
#pragma unroll
    for (int h = 1; h < NG; ++h) {
      const double ax = __shfl_sync(0xffffffffu, acc.x, c + E * h);
      const double ay = __shfl_sync(0xffffffffu, acc.y, c + E * h);
      if (g == 0) { acc.x += ax; acc.y += ay; }
    }
    if (g == 0) Ms[wid][c] = acc;
  } else {
    for (int c = lane; c < E; c += 32) {
      double2 acc = make_double2(0.0, 0.0);
#pragma unroll 4
      for (long long e = a0; e < a1; ++e) {
        const double al = q.agg_alpha[e];
        const double2 v = q.Hnode[q.agg_node[e] * E + c];
        acc.x = fma(al, v.x, acc.x);
        acc.y = fma(al, v.y, acc.y);
      }
      Ms[wid][c] = acc;
    }
  }
  __syncwarp();
  const double2* M = Ms[wid];
  for (long long k = q.tstart[leaf] + lane; k < q.tstart[leaf + 1]; k += 32) {
    const long long i = q.tperm[k];
    double2 g[P];
#pragma unroll
    for (int l = 0; l < P; ++l) g[l] = q.G[i * P + l];
    const double2 xi = q.x[i];
    double acc = 0.0;
    if (a1 > a0) {  // aggregated: Re(g M g^H)
#pragma unroll
      for (int a = 0; a < P; ++a) {
        double2 t = make_double2(0.0, 0.0);
#pragma unroll
        for (int b = 0; b < P; ++b) t = cfma_conj(t, M[a * P + b], g[b]);  // (M conj(g))_a
        acc = fma(g[a].x, t.x, fma(-g[a].y, t.y, acc));                  // Re(g_a t_a)
      }
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
  q.cstart = reinterpret_cast<const long long*>(plan->cstart);
  q.cidx = reinterpret_cast<const long long*>(plan->cidx);
  q.leaf_node = reinterpret_cast<const long long*>(plan->leaf_node);
  q.x = reinterpret_cast<const double2*>(x);
  q.y = reinterpret_cast<const double2*>(y);
  q.G = reinterpret_cast<const double2*>(G);
  q.Bt = reinterpret_cast<const double2*>(Bt);
  q.u = u;
  const size_t pp = (size_t)q.p * q.p;
  int rc;
  if ((rc = ctx->scratch[6].ensure(sizeof(double2) * pp * (size_t)q.n_snodes))) return rc;
  q.Hnode = reinterpret_cast<double2*>(ctx->scratch[6].ptr);
  const unsigned gl = (unsigned)((q.n_sleaves + 7) / 8);
  RPLU_TREE_P_SWITCH(q.p, (tree_gram_leaf_kernel<PP><<<gl, 256, 0, s>>>(q)));
  const long long* lvl_nodes = reinterpret_cast<const long long*>(plan->lvl_nodes);
  if (plan->n_levels > 0 && plan->n_levels <= kMaxLevels) {
    LevelTable lt;
    lt.n = plan->n_levels;
    for (int l = 0; l <= lt.n; ++l) lt.start[l] = plan->lvl_start[l];
    if ((rc = ctx->gbar.ensure(64))) return rc;
    unsigned* bar = reinterpret_cast<unsigned*>(ctx->gbar.ptr);
    RPLU_CUDA(cudaMemsetAsync(bar, 0, sizeof(unsigned), s));
    int per_sm = 1;
    RPLU_TREE_P_SWITCH(q.p, (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                                &per_sm, tree_gram_levels_kernel<PP>, 256, 0)));
    per_sm = per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm);
    long long most = 0;
    for (int l = 0; l < lt.n; ++l) most = std::max(most, lt.start[l + 1] - lt.start[l]);
    int grid = (int)std::min<long long>((most + 7) / 8, (long long)ctx->sm_count * per_sm);
    grid = grid < 1 ? 1 : grid;
    void* args[] = {&q, &lvl_nodes, &lt, &bar};
    RPLU_TREE_P_SWITCH(q.p, (cudaLaunchCooperativeKernel((const void*)tree_gram_levels_kernel<PP>,
                                                         dim3(grid), dim3(256), args, 0, s)));
  } else for (int l = 0; l < plan->n_levels; ++l) {
    const long long b0 = plan->lvl_start[l], cnt = plan->lvl_start[l + 1] - b0;
    if (cnt <= 0) continue;
    const unsigned gb = (unsigned)((cnt + 7) / 8);
    RPLU_TREE_P_SWITCH(q.p, (tree_gram_level_kernel<PP><<<gb, 256, 0, s>>>(q, lvl_nodes + b0, cnt)));
  }
  RPLU_TREE_P_SWITCH(q.p, (tree_bounds_kernel<PP><<<(unsigned)((q.n_tleaves + kTreeWarps - 1) / kTreeWarps),
                                                       32 * kTreeWarps, 0, s>>>(q)));
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

}  // namespace rplu
