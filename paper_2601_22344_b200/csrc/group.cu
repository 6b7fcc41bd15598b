// Multi-GPU sharded dense RPLU driven from C: one host thread, G devices of
// one node, NCCL over NVLink (SURVEY §8(b) rplu_ctx_create(ngpus, devs) /
// ncclCommInitAll, §8(e) the row-block choreography).
//
// The same per-step choreography as paper_2601_22344_b200.distributed.
// run_sharded, without Python or torch: on every device the shard select
// kernel (global owner from the allgathered totals, the owner's row / column
// draws, the pivot message with -0.0 from non-owners), one grouped
// ncclAllReduce(sum) of the message (a root-free broadcast: x + (-0) == x),
// the shard update (post the pivot, fused update or delayed-update step with
// Gram masses on the local rows, local total) and one grouped ncclAllGather
// of the shard totals.  The device step counter and the global stop rules
// keep every shard in lockstep; the host polls the first shard every 32
// steps.  NCCL is loaded at run time (dlopen of libnccl.so.2: the copy
// torch has already mapped when called from Python, the system one
// otherwise), so the library has no link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "rplu_internal.h"

namespace rplu {

namespace {

struct NcclApi {
  void* h = nullptr;
  decltype(&ncclCommInitAll) commInitAll = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  bool ok() const { return h && commInitAll && allReduce && allGather && groupStart && groupEnd; }
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return a;
    a.commInitAll = reinterpret_cast<decltype(a.commInitAll)>(dlsym(a.h, "ncclCommInitAll"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(a.h, "ncclCommDestroy"));
    a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(a.h, "ncclAllReduce"));
    a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(a.h, "ncclAllGather"));
    a.groupStart = reinterpret_cast<decltype(a.groupStart)>(dlsym(a.h, "ncclGroupStart"));
    a.groupEnd = reinterpret_cast<decltype(a.groupEnd)>(dlsym(a.h, "ncclGroupEnd"));
    a.errorString = reinterpret_cast<decltype(a.errorString)>(dlsym(a.h, "ncclGetErrorString"));
    return a;
  }();
  return api;
}

int nccl_fail(ncclResult_t r, const char* where) {
  const NcclApi& a = nccl();
  set_error(std::string(where) + ": " + (a.errorString ? a.errorString(r) : "NCCL error"));
  return RPLU_ERR_CUDA;
}

#define RPLU_NCCL(call)                                   \
  do {                                                    \
    ncclResult_t _r = (call);                             \
    if (_r != ncclSuccess) return nccl_fail(_r, #call);   \
  } while (0)

struct DevGuard {
  int prev = -1;
  DevGuard() { cudaGetDevice(&prev); }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

}  // namespace rplu

struct rplu_group {
  int ngpus = 0;
  std::vector<int> devs;
  std::vector<rplu_ctx*> ctxs;
  std::vector<ncclComm_t> comms;
  std::vector<cudaStream_t> streams;
};

using namespace rplu;

extern "C" {

int rplu_group_create(int32_t ngpus, const int32_t* devs, rplu_group** out) {
  if (ngpus < 1 || !devs || !out) {
    set_error("rplu_group_create: bad arguments");
    return RPLU_ERR_ARG;
  }
  const NcclApi& api = nccl();
  if (!api.ok()) {
    set_error("rplu_group_create: libnccl.so.2 not found");
    return RPLU_ERR_CAPABILITY;
  }
  DevGuard guard;
  auto* g = new rplu_group();
  g->ngpus = ngpus;
  g->devs.assign(devs, devs + ngpus);
  g->ctxs.assign(ngpus, nullptr);
  g->comms.assign(ngpus, nullptr);
  g->streams.assign(ngpus, nullptr);
  int rc = RPLU_OK;
  for (int d = 0; d < ngpus && rc == RPLU_OK; ++d) {
    rc = rplu_ctx_create(devs[d], &g->ctxs[d]);
    if (rc == RPLU_OK) {
      cudaSetDevice(devs[d]);
      if (cudaStreamCreateWithFlags(&g->streams[d], cudaStreamNonBlocking) != cudaSuccess) {
        set_error("rplu_group_create: stream creation failed");
        rc = RPLU_ERR_CUDA;
      }
    }
  }
  if (rc == RPLU_OK) {
    std::vector<int> dl(g->devs.begin(), g->devs.end());
    ncclResult_t r = api.commInitAll(g->comms.data(), ngpus, dl.data());
    if (r != ncclSuccess) rc = nccl_fail(r, "ncclCommInitAll");
  }
  if (rc != RPLU_OK) {
    rplu_group_destroy(g);
    return rc;
  }
  *out = g;
  return RPLU_OK;
}

int rplu_group_destroy(rplu_group* g) {
  if (!g) return RPLU_OK;
  DevGuard guard;
  const NcclApi& api = nccl();
  for (int d = 0; d < g->ngpus; ++d) {
    if (g->comms[d] && api.commDestroy) api.commDestroy(g->comms[d]);
    if (g->streams[d]) {
      cudaSetDevice(g->devs[d]);
      cudaStreamDestroy(g->streams[d]);
    }
    if (g->ctxs[d]) rplu_ctx_destroy(g->ctxs[d]);
  }
  delete g;
  return RPLU_OK;
}

int rplu_group_dense_run(rplu_group* g, const rplu_group_dense_args* a, rplu_dense_out* out) {
  if (!g || !a || !out || !a->shards || a->steps < 0) {
    set_error("rplu_group_dense_run: bad arguments");
    return RPLU_ERR_ARG;
  }
  const int G = g->ngpus;
  const NcclApi& api = nccl();
  DevGuard guard;
  std::vector<rplu_shard_args> sa(G);
  std::vector<void*> msg(G, nullptr), tot(G, nullptr), totals(G, nullptr);
  const size_t esz = a->dtype == RPLU_F32 ? 4 : (a->dtype == RPLU_F64 ? 8 : 16);
  const size_t msg_bytes = 32 + (size_t)a->m * esz;
  const ncclDataType_t red_t = a->dtype == RPLU_F32 ? ncclFloat32 : ncclFloat64;
  const size_t red_count = msg_bytes / (a->dtype == RPLU_F32 ? 4 : 8);
  int rc = RPLU_OK;
  auto cleanup = [&]() {
    for (int d = 0; d < G; ++d) {
      cudaSetDevice(g->devs[d]);
      if (msg[d]) cudaFree(msg[d]);
      if (tot[d]) cudaFree(tot[d]);
      if (totals[d]) cudaFree(totals[d]);
    }
  };
  for (int d = 0; d < G; ++d) {
    const rplu_group_shard& sh = a->shards[d];
    rplu_shard_args& s = sa[d];
    std::memset(&s, 0, sizeof(s));
    s.dtype = a->dtype;
    s.world = G;
    s.rank = d;
    s.n_local = sh.n_local;
    s.m = a->m;
    s.ld = sh.ld;
    s.row_offset = sh.row_offset;
    s.steps = a->steps;
    s.stop_tol = a->stop_tol;
    s.R = sh.R;
    s.Lt = sh.Lt;
    s.U = sh.U;
    s.ldu = a->ldu;
    s.uniforms = a->uniforms;
    s.n_uniforms = a->n_uniforms;
    s.stream = g->streams[d];
    s.lazy_block = a->lazy_block;
    cudaSetDevice(g->devs[d]);
    if (cudaMalloc(&msg[d], msg_bytes) != cudaSuccess || cudaMalloc(&tot[d], 8) != cudaSuccess ||
        cudaMalloc(&totals[d], 8 * (size_t)G) != cudaSuccess) {
      cleanup();
      set_error("rplu_group_dense_run: device allocation failed");
      return RPLU_ERR_CUDA;
    }
  }
  auto fail = [&](int r) {
    cleanup();
    return r;
  };
  auto allgather_totals = [&]() -> int {
    RPLU_NCCL(api.groupStart());
    for (int d = 0; d < G; ++d)
      RPLU_NCCL(api.allGather(tot[d], totals[d], 1, ncclFloat64, g->comms[d], g->streams[d]));
    RPLU_NCCL(api.groupEnd());
    return RPLU_OK;
  };
  for (int d = 0; d < G; ++d)
    if ((rc = rplu_shard_begin(g->ctxs[d], &sa[d], static_cast<double*>(tot[d])))) return fail(rc);
  if ((rc = allgather_totals())) return fail(rc);
  const bool eager = a->lazy_block == 0;
  // One pivot step on every device: tt >= 0 explicit step, tt == -1 the
  // device step counter (eager), tt < -1 ... block position -1 - tt of a
  // delayed-update block (select takes the counter, update the position).
  auto step = [&](long long tt) -> int {
    int r;
    for (int d = 0; d < G; ++d)
      if ((r = rplu_shard_select(g->ctxs[d], &sa[d], tt < 0 ? -1 : tt,
                                 static_cast<double*>(totals[d]), msg[d])))
        return r;
    RPLU_NCCL(api.groupStart());
    for (int d = 0; d < G; ++d)
      RPLU_NCCL(api.allReduce(msg[d], msg[d], red_count, red_t, ncclSum, g->comms[d],
                              g->streams[d]));
    RPLU_NCCL(api.groupEnd());
    for (int d = 0; d < G; ++d)
      if ((r = rplu_shard_update(g->ctxs[d], &sa[d], tt, msg[d], static_cast<double*>(tot[d]))))
        return r;
    return allgather_totals();
  };
  auto poll_active = [&](int32_t* active) { return rplu_shard_active(g->ctxs[0], &sa[0], active); };

  // Delayed-update shards: after the first block (explicit steps; it also
  // sizes every scratch buffer and sets the kernel attributes) one whole
  // flush block -- b steps of kernels on every device plus the grouped
  // collectives -- is captured into ONE multi-device CUDA graph (stream 0
  // forks to the other devices' streams through events) and replayed once per
  // block: one graph launch per b steps for all GPUs instead of ~12 G
  // launches per step from this one host thread.  RPLU_GROUP_GRAPH=0 keeps
  // the plain loop; a failed capture falls back to it.
  const long long b = eager ? 0 : rplu_shard_lazy_block(&sa[0]);
  const char* genv = getenv("RPLU_GROUP_GRAPH");
  bool use_graph = b > 0 && a->steps >= 2 * b && !(genv && genv[0] == '0');
  long long t = 0;
  int32_t active = 1;
  if (use_graph) {
    for (; t < b; ++t)
      if ((rc = step(t))) return fail(rc);
    if ((rc = poll_active(&active))) return fail(rc);
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::vector<cudaEvent_t> ev(G + 1, nullptr);
    auto drop_graph = [&]() {
      if (exec) cudaGraphExecDestroy(exec);
      if (graph) cudaGraphDestroy(graph);
      for (int d = 0; d <= G; ++d)
        if (ev[d]) cudaEventDestroy(ev[d]);
      exec = nullptr;
      graph = nullptr;
    };
    bool captured = false;
    if (active) {
      for (int d = 0; d < G; ++d) {
        cudaSetDevice(g->devs[d]);
        cudaStreamSynchronize(g->streams[d]);
        cudaEventCreateWithFlags(&ev[d], cudaEventDisableTiming);
      }
      cudaSetDevice(g->devs[0]);
      cudaEventCreateWithFlags(&ev[G], cudaEventDisableTiming);
      int crc = RPLU_OK;
      if (cudaStreamBeginCapture(g->streams[0], cudaStreamCaptureModeRelaxed) == cudaSuccess) {
        cudaEventRecord(ev[G], g->streams[0]);                       // fork
        for (int d = 1; d < G; ++d) cudaStreamWaitEvent(g->streams[d], ev[G], 0);
        for (long long pos = 0; pos < b && crc == RPLU_OK; ++pos) crc = step(-1 - pos);
        for (int d = 1; d < G; ++d) {                                // join
          cudaSetDevice(g->devs[d]);
          cudaEventRecord(ev[d], g->streams[d]);
          cudaStreamWaitEvent(g->streams[0], ev[d], 0);
        }
        cudaSetDevice(g->devs[0]);
        const cudaError_t ce = cudaStreamEndCapture(g->streams[0], &graph);
        if (crc == RPLU_OK && ce == cudaSuccess && graph &&
            cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess)
          captured = true;
      }
      if (!captured) {
        for (int d = 0; d < G; ++d) {
          cudaSetDevice(g->devs[d]);
          cudaGetLastError();
        }
        drop_graph();
      }
    }
    if (captured) {
      cudaSetDevice(g->devs[0]);
      long long k = 1;
      for (; t + b <= a->steps; t += b, ++k) {
        if (cudaGraphLaunch(exec, g->streams[0]) != cudaSuccess) {
          drop_graph();
          set_error("rplu_group_dense_run: graph launch failed");
          return fail(RPLU_ERR_CUDA);
        }
        if (k % 2 == 0) {
          // the other devices' work was forked from stream 0 and joined back
          if ((rc = poll_active(&active))) { drop_graph(); return fail(rc); }
          if (!active) break;
        }
      }
      cudaStreamSynchronize(g->streams[0]);
      drop_graph();
      if (active && (rc = poll_active(&active))) return fail(rc);
    }
  }
  for (; active && t < a->steps; ++t) {
    if ((rc = step(eager ? -1 : t))) return fail(rc);
    if ((t + 1) % 32 == 0) {
      if ((rc = poll_active(&active))) return fail(rc);
    }
  }
  // final residual norm / stop flags
  for (int d = 0; d < G; ++d)
    if ((rc = rplu_shard_select(g->ctxs[d], &sa[d], -1, static_cast<double*>(totals[d]),
                                msg[d])))
      return fail(rc);
  // every shard's finish (the delayed loop applies its pending steps); the
  // replicated results come from shard 0
  for (int d = G - 1; d >= 0; --d) {
    rplu_dense_out o = *out;
    std::vector<long long> piv(2 * (size_t)(a->steps > 0 ? a->steps : 1));
    std::vector<double> res((size_t)a->steps + 1);
    if (d > 0) {
      o.pivots = reinterpret_cast<int64_t*>(piv.data());
      o.resid_fro = res.data();
    }
    if ((rc = rplu_shard_finish(g->ctxs[d], &sa[d], &o))) return fail(rc);
    if (d == 0) *out = o;
  }
  return fail(RPLU_OK);
}

}  // extern "C"
