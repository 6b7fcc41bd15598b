// Row-block sharded dense RPLU step primitives (multi-GPU).
//
// Rank s owns rows [row_offset, row_offset + n_local) of the residual.  One
// pivot step on every rank:
//   select   (1 CTA)   global CDF over the allgathered shard totals picks the
//                      owning shard with u1 (every rank computes the same
//                      owner from the same totals); the owner draws the local
//                      row (absolute target u1*T - prefix) and the column
//                      (u2 over |R_i,:|^2) and writes the pivot message
//                      msg = [i_global, j, a_re, a_im (4 fp64) | pivot row];
//                      the other ranks write -0.0 everywhere
//   (host)   ONE allreduce(sum) of msg: x + (-0) == x exactly, so the sum
//            reproduces the owner's bits on every rank (root-free: no host
//            round trip to learn the owner)
//   update   post the header into the device state and copy the pivot row
//            into U[t,:] (multi-CTA), K3 fused Schur update + masses on the
//            local rows (the same kernel as one GPU), local total; the step
//            counter advances on the device
//   (host)   allgather of the local totals for the next step
// With t < 0 every kernel takes the step from the device counter, so one
// step (kernels + collectives) can be captured once in a CUDA graph and
// replayed.  Stop rules use the global total: every rank stops at the same
// step, and stopped ranks keep contributing -0.0 so collectives stay matched.
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

__device__ __forceinline__ long long shard_step(const ShardParams& p) {
  return p.t >= 0 ? p.t : p.st->step;
}

template <typename T>
__device__ __forceinline__ void msg_neg_zero(const ShardParams& p) {
  double* hdr = reinterpret_cast<double*>(p.msg);
  T* prow = reinterpret_cast<T*>(hdr + 4);
  for (long long k = threadIdx.x; k < p.m; k += blockDim.x) prow[k] = neg_zero<T>();
  if (threadIdx.x < 4) hdr[threadIdx.x] = -0.0;
}

template <typename T>
__global__ void __launch_bounds__(1024) shard_select_kernel(ShardParams p) {
  using S = Scalar<T>;
  constexpr int B = 1024;
  DevState* st = p.st;
  __shared__ CdfSmem<B> sm;
  __shared__ int s_owner, s_stop;
  __shared__ double s_target;
  if (!st->active) {
    msg_neg_zero<T>(p);  // keep the collective well-formed after a stop
    return;
  }
  const long long t = shard_step(p);
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
  }
  __syncthreads();
  if (s_stop || s_owner != p.rank) {
    msg_neg_zero<T>(p);
    if (!s_stop && threadIdx.x == 0) st->ucount += 2;
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
  double* hdr = reinterpret_cast<double*>(p.msg);
  T* prow = reinterpret_cast<T*>(hdr + 4);
  for (long long k = threadIdx.x; k < p.m; k += B) prow[k] = row[k];
  if (threadIdx.x == 0) {
    const double2 a = to_pair<T>(row[j]);
    hdr[0] = (double)(p.row_offset + i);
    hdr[1] = (double)j;
    hdr[2] = a.x;
    hdr[3] = a.y;
    st->ucount += 2;
    st->near_boundary += near;
  }
}

// ---------------------------------------------------------------------------
// Delayed-update shards (lazy_block > 0): the local rows keep R^(t0) of the
// last flush; the owner's pivot row is rebuilt on the fly (grid kernel), the
// local pivot column and masses come from the dense lazy kernels.
//   lazy select-row (1 CTA): global owner + local row draw (owner); header
//                             i_global (owner) or -0.0
//   lazy row (grid):          msg pivot row = R^(t0)[i,:] - pending (owner)
//                             or -0.0
//   lazy select-col (1 CTA):  owner's column draw over the message row
template <typename T>
__global__ void __launch_bounds__(1024) shard_lazy_select_row_kernel(ShardParams p) {
  constexpr int B = 1024;
  DevState* st = p.st;
  __shared__ CdfSmem<B> sm;
  __shared__ int s_owner, s_stop;
  __shared__ double s_target;
  double* hdr = reinterpret_cast<double*>(p.msg);
  if (!st->active) {
    if (threadIdx.x < 4) hdr[threadIdx.x] = -0.0;
    if (threadIdx.x == 0) st->aux[0] = 0.0;  // not the owner
    return;
  }
  const long long t = shard_step(p);
  if (threadIdx.x == 0) {
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
      const double tg = p.uniforms[st->ucount] * T_all;
      double c = 0.0;
      int last_pos = -1;
      for (int s = 0; s < p.world; ++s) {
        if (p.totals[s] > 0.0) last_pos = s;
        const double c2 = c + p.totals[s];
        if (owner < 0 && c2 > tg && p.totals[s] > 0.0) {
          owner = s;
          target = tg - c;
        }
        c = c2;
      }
      if (owner < 0) {
        owner = last_pos;
        target = p.totals[owner];
      }
      const double tol = kNearBoundaryRel * T_all;
      double cb = 0.0;
      for (int s = 0; s <= owner; ++s) {
        if (fabs(cb - tg) <= tol) st->near_boundary++;
        cb += p.totals[s];
      }
      st->ucount += 2;  // u1 now, u2 by the column draw (at ucount - 1)
    }
    if (stop) st->active = 0;
    st->aux[0] = (!stop && owner == p.rank) ? 1.0 : 0.0;
    s_stop = stop;
    s_owner = owner;
    s_target = target;
  }
  __syncthreads();
  if (s_stop || s_owner != p.rank) {
    if (threadIdx.x < 4) hdr[threadIdx.x] = -0.0;
    return;
  }
  const double* masses = p.masses;
  auto wrow = [&](long long k) { return masses[k]; };
  Cdf<B> cr = cdf_build<B>(wrow, p.n_local, sm);
  const long long i = cdf_find_target<B>(wrow, p.n_local, cr, s_target, sm);
  if (threadIdx.x == 0) {
    st->pi = i;  // local row (the header carries the global index)
    hdr[0] = (double)(p.row_offset + i);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) shard_lazy_row_kernel(ShardParams p) {
  using S = Scalar<T>;
  const DevState* st = p.st;
  T* prow = reinterpret_cast<T*>(reinterpret_cast<double*>(p.msg) + 4);
  const bool owner = st->active && st->aux[0] != 0.0;
  const long long t = shard_step(p);
  const long long t0 = (t / p.lazy_block) * p.lazy_block;
  const int q = (int)(t - t0);
  const long long i = owner ? st->pi : 0;
  const T* R = reinterpret_cast<const T*>(p.R);
  const T* Lt = reinterpret_cast<const T*>(p.Lt);
  const T* U = reinterpret_cast<const T*>(p.U) + t0 * p.ldu;
  __shared__ T s_l[kLazyMaxBlock];
  if (owner && (int)threadIdx.x < q) s_l[threadIdx.x] = Lt[(t0 + threadIdx.x) * p.n_local + i];
  __syncthreads();
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < p.m;
       k += (long long)gridDim.x * blockDim.x) {
    if (!owner) {
      prow[k] = neg_zero<T>();
      continue;
    }
    T x = R[i * p.ld + k];
    for (int s = 0; s < q; ++s) x = S::sub_outer(x, s_l[s], U[s * p.ldu + k]);
    prow[k] = x;
  }
}

template <typename T>
__global__ void __launch_bounds__(1024) shard_lazy_select_col_kernel(ShardParams p) {
  using S = Scalar<T>;
  constexpr int B = 1024;
  DevState* st = p.st;
  if (!st->active || st->aux[0] == 0.0) return;  // owner only
  __shared__ CdfSmem<B> sm;
  double* hdr = reinterpret_cast<double*>(p.msg);
  const T* prow = reinterpret_cast<const T*>(hdr + 4);
  const double u2 = p.uniforms[st->ucount - 1];
  auto wcol = [&](long long k) { return S::weight(prow[k]); };
  Cdf<B> cc = cdf_build<B>(wcol, p.m, sm);
  const long long j = cdf_find<B>(wcol, p.m, cc, u2, sm);
  if (threadIdx.x == 0) {
    const double tol = kNearBoundaryRel * cc.total, tg = u2 * cc.total;
    if (fabs(sm.lo_c - tg) <= tol || fabs(sm.hi_c - tg) <= tol) st->near_boundary++;
    const double2 a = to_pair<T>(prow[j]);
    hdr[1] = (double)j;
    hdr[2] = a.x;
    hdr[3] = a.y;
  }
}

template <typename T>
static int shard_lazy_select_t(const ShardParams& p, cudaStream_t s) {
  shard_lazy_select_row_kernel<T><<<1, 1024, 0, s>>>(p);
  const int blocks = (int)std::min<long long>((p.m + 255) / 256, 1024);
  shard_lazy_row_kernel<T><<<blocks, 256, 0, s>>>(p);
  shard_lazy_select_col_kernel<T><<<1, 1024, 0, s>>>(p);
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

int shard_lazy_select_impl(const ShardParams& p, cudaStream_t s) {
  switch (p.dtype) {
    case RPLU_F64: return shard_lazy_select_t<double>(p, s);
    case RPLU_F32: return shard_lazy_select_t<float>(p, s);
    case RPLU_C128: return shard_lazy_select_t<double2>(p, s);
  }
  set_error("unknown dtype");
  return RPLU_ERR_ARG;
}

// After the allreduce: every rank posts the pivot into its state (CTA 0,
// thread 0) and copies the reduced pivot row into U[t,:] (all CTAs).
template <typename T>
__global__ void shard_post_kernel(ShardParams p) {
  DevState* st = p.st;
  if (!st->active) return;
  const long long t = shard_step(p);
  const double* hdr = reinterpret_cast<const double*>(p.msg);
  const T* prow = reinterpret_cast<const T*>(hdr + 4);
  T* urow = reinterpret_cast<T*>(p.U) + t * p.ldu;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < p.m;
       k += (long long)gridDim.x * blockDim.x)
    urow[k] = prow[k];
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const long long ig = (long long)hdr[0];
  const long long j = (long long)hdr[1];
  T a;
  if constexpr (sizeof(T) == sizeof(double2)) a = make_double2(hdr[2], hdr[3]);
  else a = (T)hdr[2];
  if (Scalar<T>::is_zero(a)) {
    st->status = kZeroPivot;
    st->active = 0;
    st->err_i = ig;
    st->err_j = j;
    return;
  }
  st->pi = ig;
  st->pj = j;
  // the dense coefficient layout (dense.cu store_coef)
  if constexpr (sizeof(T) == sizeof(double2)) {
    CDivCoef c = cdiv_coef(make_double2(hdr[2], hdr[3]));
    st->rat = c.rat;
    st->scl = c.scl;
    st->branch = c.branch;
  } else if constexpr (sizeof(T) == sizeof(double)) {
    st->inv_d = __ddiv_rn(1.0, hdr[2]);
  } else {
    st->inv_f = __fdiv_rn(1.0f, (float)hdr[2]);
  }
  st->a_re = hdr[2];
  st->a_im = hdr[3];
  p.pivots[2 * t] = ig;
  p.pivots[2 * t + 1] = j;
  st->done = t + 1;
}

// Local total of the masses (the CDF code's fixed association); advances the
// device step counter.
__global__ void __launch_bounds__(1024) shard_total_kernel(const double* masses, long long n,
                                                          double* out, DevState* advance) {
  constexpr int B = 1024;
  __shared__ CdfSmem<B> sm;
  if (n > 0) {
    auto w = [&](long long k) { return masses[k]; };
    Cdf<B> c = cdf_build<B>(w, n, sm);
    if (threadIdx.x == 0) *out = c.total;
  } else if (threadIdx.x == 0) {
    *out = 0.0;
  }
  if (advance && threadIdx.x == 0) advance->step += 1;
}

template <typename T>
static int shard_select_t(const ShardParams& p, cudaStream_t s) {
  shard_select_kernel<T><<<1, 1024, 0, s>>>(p);
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

template <typename T>
static int shard_post_t(const ShardParams& p, cudaStream_t s) {
  const int blocks = (int)((p.m + 1023) / 1024 < 64 ? (p.m + 1023) / 1024 : 64);
  shard_post_kernel<T><<<blocks > 0 ? blocks : 1, 256, 0, s>>>(p);
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

int shard_total_impl(const double* masses, long long n, double* out, DevState* advance,
                     cudaStream_t s) {
  shard_total_kernel<<<1, 1024, 0, s>>>(masses, n, out, advance);
  RPLU_CUDA(cudaGetLastError());
  return RPLU_OK;
}

}  // namespace rplu
