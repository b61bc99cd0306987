// yb_xfer.cu — host<->device copies of caller memory for the C-ABI.
//
// Pinned (page-locked or cudaHostRegister'ed) caller buffers go straight to
// cudaMemcpyAsync. Pageable ones — the reference's own storage is pageable
// (Array3 = std::vector, array3.hpp:120), so every drop-in caller that does
// not pin its buffers lands here — would otherwise take the driver's
// single-threaded staging path. Instead they run through a process-wide
// pipeline: a ring of pinned staging chunks, filled (H2D) or drained (D2H)
// by a small pool of copy threads, with the DMA of chunk i overlapping the
// host copy of chunk i+1, so the transfer runs at PCIe rate rather than at
// one thread's memcpy rate. Semantics match cudaMemcpy from pageable
// memory: yb::copy_h2d returns once the caller's buffer has been read (the
// DMAs are queued on the stream, ordered before later work on it);
// yb::copy_d2h of a pageable buffer returns once it holds the data (a pinned
// one is only queued: the caller synchronizes the stream, as before).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "yb_launch.h"

namespace yb {
namespace {

// Fixed pool of copy threads; the calling thread takes tasks too.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* p = new CopyPool();  // never destroyed: detached workers may outlive static teardown
    return *p;
  }
  int threads() const { return static_cast<int>(th_.size()) + 1; }
  // runs fn(0..n-1) across the pool; returns when all have finished
  void run(int n, const std::function<void(int)>& fn) {
    if (n <= 1 || th_.empty()) {
      for (int t = 0; t < n; ++t) fn(t);
      return;
    }
    std::unique_lock<std::mutex> lk(m_);
    fn_ = &fn;
    n_ = n;
    next_.store(0);
    pending_ = n;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    work(&fn, n);
    lk.lock();
    // every task ran and every worker that joined this round has left it
    done_.wait(lk, [&] { return pending_ == 0 && active_ == 0; });
    fn_ = nullptr;
  }

 private:
  CopyPool() {
    int n = 0;
    if (const char* e = std::getenv("YB_XFER_THREADS")) n = std::atoi(e);
    // three quarters of the cores, at most 16: the caller is blocked in the transfer meanwhile (config 4's
    // streamed readback into pageable memory on 16 cores: 4 / 8 / 12 threads -> 97 / 118-128 / 139 Gcell/s end to end)
    if (n <= 0) n = std::min(16, std::max(2, static_cast<int>(std::thread::hardware_concurrency()) * 3 / 4));
    for (int t = 0; t + 1 < n; ++t) {
      th_.emplace_back([this] { loop(); });
      th_.back().detach();
    }
  }
  void loop() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(m_);
    for (;;) {
      cv_.wait(lk, [&] { return gen_ != seen && fn_ != nullptr; });
      seen = gen_;
      const std::function<void(int)>* f = fn_;
      const int n = n_;
      ++active_;
      lk.unlock();
      work(f, n);
      lk.lock();
      if (--active_ == 0 && pending_ == 0) done_.notify_all();
    }
  }
  void work(const std::function<void(int)>* f, int n) {
    int done = 0;
    for (int t; (t = next_.fetch_add(1)) < n;) {
      (*f)(t);
      ++done;
    }
    if (done) {
      std::lock_guard<std::mutex> g(m_);
      pending_ -= done;
      if (pending_ == 0) done_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0, pending_ = 0, active_ = 0;
  std::atomic<int> next_{0};
  uint64_t gen_ = 0;
};

// memcpy split over the pool in >= 4 MiB pieces
void par_memcpy(void* dst, const void* src, size_t n) {
  constexpr size_t kPiece = size_t(4) << 20;
  CopyPool& P = CopyPool::get();
  const int tasks = static_cast<int>(std::min<size_t>(static_cast<size_t>(P.threads()), (n + kPiece - 1) / kPiece));
  if (tasks <= 1) {
    std::memcpy(dst, src, n);
    return;
  }
  const size_t per = ((n + tasks - 1) / tasks + 63) & ~size_t(63);
  P.run(tasks, [&](int t) {
    const size_t o = static_cast<size_t>(t) * per;
    if (o < n) std::memcpy(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, std::min(per, n - o));
  });
}

// Process-wide ring of pinned staging chunks (allocated on first use).
struct Staging {
  static constexpr int kChunks = 4;
  static constexpr size_t kChunk = size_t(32) << 20;
  std::mutex m;
  void* buf[kChunks] = {};
  cudaEvent_t ev[kChunks] = {};
  int dev[kChunks] = {-1, -1, -1, -1};  // device whose stream last used the chunk (events are per device)
  bool ready = false;
  cudaError_t init() {
    if (ready) return cudaSuccess;
    for (int k = 0; k < kChunks; ++k) {
      cudaError_t e = cudaHostAlloc(&buf[k], kChunk, cudaHostAllocPortable);
      if (e != cudaSuccess) return e;
    }
    ready = true;
    return cudaSuccess;
  }
  // the chunk's previous DMA has finished; its event re-created on the current device
  cudaError_t acquire(int k, int device) {
    if (ev[k]) {
      const cudaError_t e = cudaEventSynchronize(ev[k]);
      if (e != cudaSuccess) return e;
      if (dev[k] != device) {
        cudaEventDestroy(ev[k]);
        ev[k] = nullptr;
      }
    }
    if (!ev[k]) {
      const cudaError_t e = cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
      dev[k] = device;
    }
    return cudaSuccess;
  }
  static Staging& get() {
    static Staging* s = new Staging();
    return *s;
  }
};

}  // namespace

std::mutex& stage_lock() { return Staging::get().m; }
cudaError_t stage_init() { return Staging::get().init(); }
void* stage_buf(int k) { return Staging::get().buf[k]; }
cudaError_t stage_acquire(int k, int device) { return Staging::get().acquire(k, device); }
cudaEvent_t stage_event(int k) { return Staging::get().ev[k]; }
void par_for(int n, const std::function<void(int)>& fn) { CopyPool::get().run(n, fn); }
static_assert(kStageChunks == Staging::kChunks && kStageBytes == Staging::kChunk, "staging ring shape");

bool host_is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

cudaError_t copy_h2d(void* dst, const void* src, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (!host_is_pageable(src) || n < (size_t(1) << 20)) return cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st);
  int device = 0;
  cudaGetDevice(&device);
  Staging& S = Staging::get();
  std::lock_guard<std::mutex> g(S.m);
  cudaError_t e = S.init();
  if (e != cudaSuccess) return e;
  int k = 0;
  for (size_t o = 0; o < n; o += Staging::kChunk, k = (k + 1) % Staging::kChunks) {
    const size_t c = std::min(Staging::kChunk, n - o);
    if ((e = S.acquire(k, device)) != cudaSuccess) return e;
    par_memcpy(S.buf[k], static_cast<const char*>(src) + o, c);  // overlaps the previous chunks' DMAs
    if ((e = cudaMemcpyAsync(static_cast<char*>(dst) + o, S.buf[k], c, cudaMemcpyHostToDevice, st)) != cudaSuccess)
      return e;
    if ((e = cudaEventRecord(S.ev[k], st)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t copy_d2h(void* dst, const void* src, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (!host_is_pageable(dst) || n < (size_t(1) << 20))  // the caller synchronizes the stream
    return cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st);
  int device = 0;
  cudaGetDevice(&device);
  Staging& S = Staging::get();
  std::lock_guard<std::mutex> g(S.m);
  cudaError_t e = S.init();
  if (e != cudaSuccess) return e;
  const size_t nch = (n + Staging::kChunk - 1) / Staging::kChunk;
  auto issue = [&](size_t i) -> cudaError_t {
    const int k = static_cast<int>(i % Staging::kChunks);
    const size_t o = i * Staging::kChunk, c = std::min(Staging::kChunk, n - o);
    cudaError_t r = S.acquire(k, device);
    if (r != cudaSuccess) return r;
    if ((r = cudaMemcpyAsync(S.buf[k], static_cast<const char*>(src) + o, c, cudaMemcpyDeviceToHost, st)) !=
        cudaSuccess)
      return r;
    return cudaEventRecord(S.ev[k], st);
  };
  for (size_t i = 0; i < std::min<size_t>(nch, Staging::kChunks); ++i)
    if ((e = issue(i)) != cudaSuccess) return e;
  for (size_t i = 0; i < nch; ++i) {
    const int k = static_cast<int>(i % Staging::kChunks);
    const size_t o = i * Staging::kChunk, c = std::min(Staging::kChunk, n - o);
    if ((e = cudaEventSynchronize(S.ev[k])) != cudaSuccess) return e;
    par_memcpy(static_cast<char*>(dst) + o, S.buf[k], c);  // overlaps the next chunks' DMAs
    if (i + Staging::kChunks < nch && (e = issue(i + Staging::kChunks)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace yb
