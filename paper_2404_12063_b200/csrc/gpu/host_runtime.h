// Host-side runtime support of the C-ABI (vpinn_gpu.cu, its only includer):
// error mapping (Fail / CK / guarded), the per-device block cache, the
// staged pinned-memory uploader with its copy-worker pool, pinned trainer
// words and the device buffer type.
#pragma once

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "vpinn_gpu.h"

namespace {

thread_local std::string g_err;

// vpinn_gpu_set_test_hooks: read by every later vpinn_gpu_create
std::atomic<int> g_test_hooks{0};

struct Fail {
  int code;
  std::string msg;
};

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      throw Fail{VPINN_ERR_DEVICE, std::string(#x) + ": " + cudaGetErrorString(e_)};    \
  } while (0)

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return VPINN_OK;
  } catch (const Fail& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VPINN_ERR_NUMERIC;
  }
}

// Device-memory block cache: blocks released by contexts are kept per device
// and exact byte size and handed to the next allocation of that size, so
// re-creating a context (sweeps, parameter studies, the e2e bench) costs no
// cudaMalloc / cudaFree (cudaFree synchronizes the whole device).  Owners
// release only idle blocks (a context synchronizes its stream first).
struct BlockCache {
  std::mutex mu;
  std::map<std::pair<int, size_t>, std::vector<void*>> blocks;
  size_t cached = 0;
  static constexpr size_t kCap = size_t(8) << 30;
  void* get(size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    auto it = blocks.find({dev, bytes});
    if (it == blocks.end() || it->second.empty()) return nullptr;
    void* p = it->second.back();
    it->second.pop_back();
    cached -= bytes;
    return p;
  }
  void put(void* p, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    {
      std::lock_guard<std::mutex> g(mu);
      if (cached + bytes <= kCap) {
        blocks[{dev, bytes}].push_back(p);
        cached += bytes;
        return;
      }
    }
    cudaFree(p);
  }
  void trim() {
    std::lock_guard<std::mutex> g(mu);
    for (auto& kv : blocks) {
      cudaSetDevice(kv.first.first);
      for (void* p : kv.second) cudaFree(p);
    }
    blocks.clear();
    cached = 0;
  }
};
BlockCache& block_cache() {
  static BlockCache* c = new BlockCache;  // never destroyed: no teardown-order races at exit
  return *c;
}


// ---------------------------------------------------------------------------
// Host -> device uploads of large pageable arrays (the premultiplier tensors
// at vpinn_gpu_create): pageable cudaMemcpy runs at ~8 GB/s on the B200
// boxes; staging through a pinned ring filled by a small host thread pool
// overlaps the host copy of chunk i+1 with the DMA of chunk i at pinned
// bandwidth.  Process-wide, never destroyed (no exit-order races).
struct CopyPool {
  // workers spin briefly on a generation counter between the chunks of one
  // upload (a condition-variable wake-up per 8 MB chunk cost ~30 us each),
  // then block on the condition variable when idle
  int n = 1;
  std::vector<std::thread> workers;
  std::mutex mu;
  std::condition_variable cv;
  std::atomic<unsigned> gen{0};
  std::atomic<int> pending{0};
  char* dst = nullptr;
  const char* src = nullptr;
  size_t len = 0;
  CopyPool() {
    const unsigned hc = std::thread::hardware_concurrency();
    // three quarters of the host threads, at most 12 (gear create on a
    // 16-thread box: 8 threads x 16 MB chunks 3.2-3.4 ms, 12 x 12 MB 3.0-3.2)
    n = std::max(1, std::min(12, (int)(hc ? 3 * hc / 4 : 1)));
    for (int i = 1; i < n; ++i) workers.emplace_back([this, i] { loop(i); });
    for (auto& w : workers) w.detach();
  }
  void slice(int i, char*& d, const char*& s, size_t& l) const {
    const size_t per = (len / n + 63) & ~size_t(63);
    const size_t a = std::min(len, per * i), b = std::min(len, per * (i + 1));
    d = dst + a;
    s = src + a;
    l = b - a;
  }
  void loop(int i) {
    unsigned seen = 0;
    for (;;) {
      // spin ~1 ms for the next chunk, then sleep until notified
      const auto t0 = std::chrono::steady_clock::now();
      while (gen.load(std::memory_order_acquire) == seen) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(1)) {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return gen.load(std::memory_order_acquire) != seen; });
          break;
        }
        std::this_thread::yield();
      }
      seen = gen.load(std::memory_order_acquire);
      char* d;
      const char* s;
      size_t l;
      slice(i, d, s, l);
      if (l) std::memcpy(d, s, l);
      pending.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  void copy(void* d, const void* s, size_t l) {
    if (n == 1 || l < (size_t(1) << 20)) {
      std::memcpy(d, s, l);
      return;
    }
    dst = static_cast<char*>(d);
    src = static_cast<const char*>(s);
    len = l;
    pending.store(n - 1, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> g(mu);
      gen.fetch_add(1, std::memory_order_acq_rel);
    }
    cv.notify_all();
    char* d0;
    const char* s0;
    size_t l0;
    slice(0, d0, s0, l0);
    if (l0) std::memcpy(d0, s0, l0);
    while (pending.load(std::memory_order_acquire) != 0) std::this_thread::yield();
  }
};

struct Stager {
  static constexpr size_t kChunk = size_t(12) << 20;
  static constexpr int kBufs = 3;
  std::mutex mu;
  char* buf[kBufs] = {};
  // one event per (device, buffer); last_dev[k] = the device whose copy out
  // of buf[k] was enqueued last (-1: none).  The pinned buffers are shared by
  // every device, so a reuse waits for the last DMA out of the buffer on
  // whichever device issued it.
  cudaEvent_t ev[16][kBufs] = {};
  int last_dev[kBufs] = {-1, -1, -1};
  CopyPool pool;
  // false: caller falls back to a plain pageable copy
  bool upload(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return false;
    std::lock_guard<std::mutex> g(mu);
    for (int k = 0; k < kBufs; ++k) {
      if (!buf[k] && cudaHostAlloc(&buf[k], kChunk, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        buf[k] = nullptr;
        return false;
      }
      if (!ev[dev][k]) CK(cudaEventCreateWithFlags(&ev[dev][k], cudaEventDisableTiming));
    }
    const char* sp = static_cast<const char*>(src);
    char* dp = static_cast<char*>(dst);
    int k = 0;
    for (size_t off = 0; off < bytes; off += kChunk, k = (k + 1) % kBufs) {
      const size_t l = std::min(kChunk, bytes - off);
      if (last_dev[k] >= 0) CK(cudaEventSynchronize(ev[last_dev[k]][k]));
      pool.copy(buf[k], sp + off, l);
      CK(cudaMemcpyAsync(dp + off, buf[k], l, cudaMemcpyHostToDevice, s));
      CK(cudaEventRecord(ev[dev][k], s));
      last_dev[k] = dev;
    }
    return true;
  }
};
Stager& stager() {
  static Stager* st = new Stager;
  return *st;
}
// page-locked host memory (cudaHostAlloc / cudaHostRegister by the caller):
// the DMA reads it directly, no staging copy
bool host_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}
void upload_bytes(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes >= (size_t(4) << 20) && !host_pinned(src) && stager().upload(dst, src, bytes, s)) return;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
}

// small pinned host words (per-context trainer flags) from one pinned slab:
// cudaMallocHost per context costs ~1 ms
struct PinnedWords {
  std::mutex mu;
  int* slab = nullptr;
  std::vector<int*> free_slots;
  int* get() {
    std::lock_guard<std::mutex> g(mu);
    if (free_slots.empty()) {
      constexpr int kSlots = 1024;
      if (cudaMallocHost(&slab, sizeof(int) * 4 * kSlots) != cudaSuccess) return nullptr;
      for (int i = kSlots - 1; i >= 0; --i) free_slots.push_back(slab + 4 * i);
    }
    int* p = free_slots.back();
    free_slots.pop_back();
    return p;
  }
  void put(int* p) {
    std::lock_guard<std::mutex> g(mu);
    free_slots.push_back(p);
  }
};
PinnedWords& pinned_words() {
  static PinnedWords* w = new PinnedWords;
  return *w;
}

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0, bytes = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) block_cache().put(p, bytes);
    p = nullptr;
    n = bytes = 0;
  }
  // 64 bytes of slack: 1-D bulk copies read 16-byte aligned supersets
  // zero-filled on stream s, i.e. ordered before anything later enqueued on s
  // (a legacy-default-stream memset does NOT order with a non-blocking
  // stream: it could land after, and overwrite, an upload)
  void alloc(size_t count, cudaStream_t s) {
    release();
    n = count;
    bytes = (std::max<size_t>(count, 1) * sizeof(T) + 64 + 255) & ~size_t(255);
    p = static_cast<T*>(block_cache().get(bytes));
    if (!p) CK(cudaMalloc(&p, bytes));
    CK(cudaMemsetAsync(p, 0, bytes, s));
  }
  // the host array may be freed as soon as this returns
  void upload(const T* h, size_t count, cudaStream_t s) {
    if (count) upload_bytes(p, h, count * sizeof(T), s);
  }
  void upload_at(size_t at, const T* h, size_t count, cudaStream_t s) {
    if (count) upload_bytes(p + at, h, count * sizeof(T), s);
  }
};

}  // namespace
