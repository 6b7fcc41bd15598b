// Row-block sharded dense RPLU step primitives (multi-GPU).
//
// Rank s owns rows [row_offset, row_offset + n_local) of the residual.  One
// pivot step on every rank:
//   select   (1 CTA)   global CDF over the allgathered shard totals picks the
//                      owning shard with u1 (every rank computes the same
//                      owner from the same totals); the owner draws the local
//                      row (absolute target u1*T - prefix) and the column
//                      (u2 over |R_i,:|^2) and writes the message
//                      header = [i_global, j, a_re, a_im] (fp64) and the pivot
//                      row into U[t,:]; the other ranks write -0.0 everywhere
//   (host)   allreduce(sum) of header and U[t,:]: x + (-0) == x exactly, so
//            the sum reproduces the owner's bits on every rank (root-free: no
//            host round trip to learn the owner)
//   update   post the header into the device state, K3 fused Schur update +
//            masses on the local rows (the same kernel as one GPU), local total
//   (host)   allgather of the local totals for the next step
// The stop rules use the global total, so every rank stops at the same step.
#include <cuda_runtime.h>
#include <stdint.h>

#include "rplu_common.cuh"
#include "rplu_internal.h"

namespace rplu {

template <typename T>
__device__ __forceinline__ double2 to_pair(T v);
template <> __device__ __forceinline__ double2 to_pair<double>(double v) { return make_double2(v, 0.0); }
template <> __device__ __forceinline__ double2 to_pair<float>(float v) { return make_double2((double)v, 0.0); }
template <> __device__ __forceinline__ double2 to_pair<double2>(double2 v) { return v; }

template <typename T>
__device__ __forceinline__ T neg_zero();
template <> __device__ __forceinline__ double neg_zero<double>() { return -0.0; }
template <> __device__ __forceinline__ float neg_zero<float>() { return -0.0f; }
template <> __device__ __forceinline__ double2 neg_zero<double2>() { return make_double2(-0.0, -0.0); }

template <typename T>
__global__ void __launch_bounds__(1024) shard_select_kernel(ShardParams p) {
  using S = Scalar<T>;
  constexpr int B = 1024;
  DevState* st = p.st;
  const long long t = p.t;
  T* urow = reinterpret_cast<T*>(p.U) + t * p.ldu;
  __shared__ CdfSmem<B> sm;
  __shared__ int s_owner, s_stop;
  __shared__ double s_target, s_total;
  if (!st->active) {
    // keep the collective well-formed after a stop: contribute -0
    for (long long k = threadIdx.x; k < p.m; k += B) urow[k] = neg_zero<T>();
    if (threadIdx.x < 4) p.header[threadIdx.x] = -0.0;
    return;
  }
  if (threadIdx.x == 0) {
    // global total over shards, in rank order (identical on every rank)
    double T_all = 0.0;
    for (int s = 0; s < p.world; ++s) T_all += p.totals[s];
    const double resid = sqrt(T_all);
    p.resid[t] = resid;
    if (t == 0) st->fro0 = resid;
    const double fro0 = (t == 0) ? resid : st->fro0;
    int stop = 0;
    if (t > 0 && p.stop_tol > 0.0 && resid <= p.stop_tol * fro0) {
      st->status = kTolStop;
      stop = 1;
    } else if (t >= p.steps) {
      stop = 1;
    } else if (resid == 0.0) {
      st->status = kCleanStop;
      stop = 1;
    } else if (st->ucount + 2 > p.n_uniforms) {
      st->status = kUniformsExhausted;
      stop = 1;
    }
    int owner = -1;
    double target = 0.0;
    if (!stop) {
      const double u1 = p.uniforms[st->ucount];
      const double tg = u1 * T_all;
      double c = 0.0;
      int last_pos = -1;
      for (int s = 0; s < p.world; ++s) {
        if (p.totals[s] > 0.0) last_pos = s;
        const double c2 = c + p.totals[s];
        if (owner < 0 && c2 > tg && p.totals[s] > 0.0) {
          owner = s;
          target = tg - c;  // absolute target inside the owning shard
        }
        c = c2;
      }
      if (owner < 0) {  // top clamp: last shard with positive mass
        owner = last_pos;
        target = p.totals[owner];
      }
      const double tol = kNearBoundaryRel * T_all;
      double cb = 0.0;
      for (int s = 0; s <= owner; ++s) {
        if (fabs(cb - tg) <= tol) st->near_boundary++;
        cb += p.totals[s];
      }
    }
    if (stop) st->active = 0;
    s_stop = stop;
    s_owner = owner;
    s_target = target;
    s_total = T_all;
  }
  __syncthreads();
  if (s_stop) {
    for (long long k = threadIdx.x; k < p.m; k += B) urow[k] = neg_zero<T>();
    if (threadIdx.x < 4) p.header[threadIdx.x] = -0.0;
    return;
  }
  if (s_owner != p.rank) {
    for (long long k = threadIdx.x; k < p.m; k += B) urow[k] = neg_zero<T>();
    if (threadIdx.x < 4) p.header[threadIdx.x] = -0.0;
    if (threadIdx.x == 0) st->ucount += 2;
    return;
  }
  // owner: local row draw against the absolute target, then the column draw
  const T* R = reinterpret_cast<const T*>(p.R);
  const double* masses = p.masses;
  auto wrow = [&](long long k) { return masses[k]; };
  Cdf<B> cr = cdf_build<B>(wrow, p.n_local, sm);
  long long i = cdf_find_target<B>(wrow, p.n_local, cr, s_target, sm);
  const double u2 = p.uniforms[st->ucount + 1];
  const T* row = R + i * p.ld;
  auto wcol = [&](long long k) { return S::weight(row[k]); };
  __syncthreads();
  Cdf<B> cc = cdf_build<B>(wcol, p.m, sm);
  long long j = cdf_find<B>(wcol, p.m, cc, u2, sm);
  long long near = 0;
  if (threadIdx.x == 0) {
    const double tol = kNearBoundaryRel * cc.total, tg = u2 * cc.total;
    if (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) near++;
  }
  for (long long k = threadIdx.x; k < p.m; k += B) urow[k] = row[k];
  if (threadIdx.x == 0) {
    const double2 a = to_pair<T>(row[j]);
    p.header[0] = (double)(p.row_offset + i);
    p.header[1] = (double)j;
    p.header[2] = a.x;
    p.header[3] = a.y;
    st->ucount += 2;
    st->near_boundary += near;
  }
}

// After the allreduce: every rank posts the pivot into its state.
template <typename T>
__global__ void shard_post_kernel(ShardParams p) {
  DevState* st = p.st;
  if (!st->active) return;
  const long long ig = (long long)p.header[0];
  const long long j = (long long)p.header[1];
  T a;
  if constexpr (sizeof(T) == sizeof(double2)) a = make_double2(p.header[2], p.header[3]);
  else a = (T)p.header[2];
  if (Scalar<T>::is_zero(a)) {
    st->status = kZeroPivot;
    st->active = 0;
    st->err_i = ig;
    st->err_j = j;
    return;
  }
  st->pi = ig;
  st->pj = j;
  // reuse the dense coefficient layout (dense.cu store_coef)
  if constexpr (sizeof(T) == sizeof(double2)) {
    CDivCoef c = cdiv_coef(make_double2(p.header[2], p.header[3]));
    st->rat = c.rat;
    st->scl = c.scl;
    st->branch = c.branch;
  } else if constexpr (sizeof(T) == sizeof(double)) {
    st->inv_d = __ddiv_rn(1.0, p.header[2]);
  } else {
    st->inv_f = __fdiv_rn(1.0f, (float)p.header[2]);
  }
  st->a_re = p.header[2];
  st->a_im = p.header[3];
  p.pivots[2 * p.t] = ig;
  p.pivots[2 * p.t + 1] = j;
  st->done = p.t + 1;
}

// local total of the masses, fixed order (chunk sums then serial)
__global__ void __launch_bounds__(1024) shard_total_kernel(const double* masses, long long n,
                                                          double* out) {
  constexpr int B = 1024;
  __shared__ CdfSmem<B> sm;
  auto w = [&](long long k) { return masses[k]; };
  Cdf<B> c = cdf_build<B>(w, n, sm);
  if (threadIdx.x == 0) *out = c.total;
}

template <typename T>
static int shard_select_t(const ShardParams& p, cudaStream_t s) {
  shard_select_kernel<T><<<1, 1024, 0, s>>>(p);
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

template <typename T>
static int shard_post_t(const ShardParams& p, cudaStream_t s) {
  shard_post_kernel<T><<<1, 1, 0, s>>>(p);
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

int shard_select_impl(const ShardParams& p, cudaStream_t s) {
  switch (p.dtype) {
    case RPLU_F64: return shard_select_t<double>(p, s);
    case RPLU_F32: return shard_select_t<float>(p, s);
    case RPLU_C128: return shard_select_t<double2>(p, s);
  }
  set_error("unknown dtype");
  return RPLU_ERR_ARG;
}

int shard_post_impl(const ShardParams& p, cudaStream_t s) {
  switch (p.dtype) {
    case RPLU_F64: return shard_post_t<double>(p, s);
    case RPLU_F32: return shard_post_t<float>(p, s);
    case RPLU_C128: return shard_post_t<double2>(p, s);
  }
  set_error("unknown dtype");
  return RPLU_ERR_ARG;
}

int shard_total_impl(const double* masses, long long n, double* out, cudaStream_t s) {
  shard_total_kernel<<<1, 1024, 0, s>>>(masses, n, out);
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

}  // namespace rplu
