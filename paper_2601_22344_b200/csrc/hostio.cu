// Host -> device staging of pageable caller buffers (the reference's callers
// pass plain numpy arrays, dense_pivots.py:86-89 copies them).
//
// A cudaMemcpy from pageable memory is staged by the driver through a small
// pinned bounce buffer by one thread; here the copy is pipelined through a
// ring of large page-locked slots owned by the context.  One pool of worker
// threads lives for the whole call: every worker copies its share of each
// slot with non-temporal 16-byte stores (no read-for-ownership of the pinned
// destination and no cache pollution: a third less host DRAM traffic than
// memcpy on pieces below glibc's streaming threshold), the calling thread
// releases a slot to the workers as soon as the DMA that last read it has
// finished (up to kSlots slots ahead) and issues the slot's DMA when every
// worker has finished it, so host copies and DMA overlap throughout.  The
// source is no longer read when the call returns; the transfers are ordered
// on `stream`.
#include <cuda_runtime.h>
#include <emmintrin.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "rplu_internal.h"

namespace rplu {

namespace {
constexpr size_t kSlotBytes = 64ull << 20;   // ring slot capacity
constexpr size_t kMinSlotBytes = 4ull << 20;
constexpr int kSlots = 4;
constexpr size_t kDirectBytes = 16ull << 20;

// dst 16-byte aligned; streaming stores, unaligned loads
void copy_stream(char* dst, const char* src, size_t len) {
  size_t k = 0;
  const size_t body = len & ~size_t(63);
  for (; k < body; k += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + k));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + k + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + k + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + k + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + k + 48), d);
  }
  if (k < len) std::memcpy(dst + k, src + k, len - k);
  _mm_sfence();
}

struct Pool {
  const char* in = nullptr;
  char* ring = nullptr;
  size_t bytes = 0;
  size_t slot_bytes = kSlotBytes;        // bytes staged per slot use (<= kSlotBytes)
  long long nslots = 0;
  int workers = 1;                       // including the calling thread (worker 0)
  std::atomic<long long> released{0};    // slots 0 .. released-1 may be filled
  std::atomic<long long> done[kSlots];   // per ring slot: cumulative worker completions
  std::atomic<int> abort{0};

  // worker w's piece of slot k (64-byte granules)
  void fill(long long k, int w) const {
    const size_t off = (size_t)k * slot_bytes;
    const size_t len = std::min(slot_bytes, bytes - off);
    const size_t gran = (len + 63) / 64;
    const size_t per = (gran + workers - 1) / workers * 64;
    const size_t a = std::min(len, (size_t)w * per), b = std::min(len, a + per);
    if (b > a) copy_stream(ring + (size_t)(k % kSlots) * kSlotBytes + a, in + off + a, b - a);
  }
  void worker(int w) {
    for (long long k = 0; k < nslots; ++k) {
      while (released.load(std::memory_order_acquire) <= k) {
        if (abort.load(std::memory_order_relaxed)) return;
        std::this_thread::yield();
      }
      if (abort.load(std::memory_order_relaxed)) return;
      fill(k, w);
      done[k % kSlots].fetch_add(1, std::memory_order_release);
    }
  }
};
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
  Pool pool;
  pool.in = static_cast<const char*>(src);
  pool.ring = static_cast<char*>(ctx->ring);
  pool.bytes = (size_t)bytes;
  // small inputs use smaller pieces so that host copies and DMA still overlap
  // (about 8 pieces per call, 4 .. 64 MB each)
  const size_t mb = 1ull << 20;
  pool.slot_bytes = std::min(kSlotBytes, std::max(kMinSlotBytes, ((size_t)bytes / 8 + mb - 1) / mb * mb));
  pool.nslots = (long long)(((size_t)bytes + pool.slot_bytes - 1) / pool.slot_bytes);
  // one worker per >= 4 MB of input (thread start-up is ~30 us each)
  pool.workers = std::max(1, std::min({threads, 32, (int)((size_t)bytes / kMinSlotBytes)}));
  for (int i = 0; i < kSlots; ++i) pool.done[i].store(0);
  std::vector<std::thread> th;
  for (int w = 1; w < pool.workers; ++w) th.emplace_back([&pool, w] { pool.worker(w); });
  char* out = static_cast<char*>(dst);
  cudaError_t err = cudaSuccess;
  long long released = 0;
  for (long long k = 0; k < pool.nslots && err == cudaSuccess; ++k) {
    // release slots ahead: a ring slot is free once the DMA recorded behind
    // its previous use has completed (the first kSlots uses wait for the
    // events of an earlier call, if any)
    while (released < pool.nslots && released < k + kSlots) {
      const int slot = (int)(released % kSlots);
      const cudaError_t q = released <= k ? cudaEventSynchronize(ctx->ring_ev[slot])
                                          : cudaEventQuery(ctx->ring_ev[slot]);
      if (q == cudaErrorNotReady) break;
      if (q != cudaSuccess) { err = q; break; }
      pool.released.store(++released, std::memory_order_release);
    }
    if (err != cudaSuccess) break;
    pool.fill(k, 0);   // the calling thread is worker 0
    const int slot = (int)(k % kSlots);
    const long long want = (long long)(pool.workers - 1) * (k / kSlots + 1);
    while (pool.done[slot].load(std::memory_order_acquire) < want) std::this_thread::yield();
    const size_t off = (size_t)k * pool.slot_bytes;
    const size_t len = std::min(pool.slot_bytes, (size_t)bytes - off);
    err = cudaMemcpyAsync(out + off, pool.ring + (size_t)slot * kSlotBytes, len,
                          cudaMemcpyHostToDevice, s);
    if (err == cudaSuccess) err = cudaEventRecord(ctx->ring_ev[slot], s);
  }
  if (err != cudaSuccess) pool.abort.store(1);
  pool.released.store(pool.nslots, std::memory_order_release);   // let the workers run out
  for (auto& t : th) t.join();
  if (err != cudaSuccess) return cuda_fail(err, "rplu_upload");
  return RPLU_OK;
}

}  // namespace rplu
