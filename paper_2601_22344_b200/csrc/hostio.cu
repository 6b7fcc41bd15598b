// Host -> device staging of pageable caller buffers (the reference's callers
// pass plain numpy arrays, dense_pivots.py:86-89 copies them).
//
// A cudaMemcpy from pageable memory is staged by the driver through a small
// pinned bounce buffer by one thread; here the copy is pipelined through a
// ring of large page-locked slots owned by the context: worker threads copy
// chunk c+1 (split across `threads` threads, memcpy bandwidth scales with
// them) while the DMA engine moves chunk c, and a slot is refilled only after
// the event recorded behind its last transfer completes.  The source is no
// longer read when the call returns; the transfers are ordered on `stream`.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "rplu_internal.h"

namespace rplu {

namespace {
constexpr size_t kSlotBytes = 64ull << 20;
constexpr int kSlots = 4;
constexpr size_t kDirectBytes = 16ull << 20;
}  // namespace

int upload_impl(rplu_ctx* ctx, void* dst, const void* src, long long bytes, int threads,
                cudaStream_t s) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) {
    set_error("rplu_upload: bad arguments");
    return RPLU_ERR_ARG;
  }
  if (bytes == 0) return RPLU_OK;
  if ((size_t)bytes <= kDirectBytes) {
    RPLU_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, s));
    return RPLU_OK;
  }
  if (!ctx->ring) {
    void* p = nullptr;
    RPLU_CUDA(cudaHostAlloc(&p, kSlotBytes * kSlots, cudaHostAllocDefault));
    ctx->ring = p;
    for (int i = 0; i < kSlots; ++i) RPLU_CUDA(cudaEventCreateWithFlags(&ctx->ring_ev[i],
                                                                        cudaEventDisableTiming));
  }
  threads = std::max(1, std::min(threads, 32));
  char* ring = static_cast<char*>(ctx->ring);
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  size_t off = 0;
  int slot = 0;
  while (off < (size_t)bytes) {
    const size_t len = std::min(kSlotBytes, (size_t)bytes - off);
    RPLU_CUDA(cudaEventSynchronize(ctx->ring_ev[slot]));  // the slot's last transfer is done
    char* buf = ring + (size_t)slot * kSlotBytes;
    const size_t per = (len + threads - 1) / threads;
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) {
      const size_t a = (size_t)t * per;
      if (a >= len) break;
      const size_t b = std::min(len, a + per);
      pool.emplace_back([=] { std::memcpy(buf + a, in + off + a, b - a); });
    }
    std::memcpy(buf, in + off, std::min(len, per));
    for (auto& th : pool) th.join();
    RPLU_CUDA(cudaMemcpyAsync(out + off, buf, len, cudaMemcpyHostToDevice, s));
    RPLU_CUDA(cudaEventRecord(ctx->ring_ev[slot], s));
    off += len;
    slot = (slot + 1) % kSlots;
  }
  return RPLU_OK;
}

}  // namespace rplu
