// host_stager.cpp -- pageable host <-> device copies for the drop-in's host
// buffers (numpy arrays: the reference API, reduce.py:69-73 / :379-387,
// takes and returns host arrays).
//
// A pageable cudaMemcpy runs at ~11 GB/s on the B200 box (the driver stages
// it through a small pinned buffer, one thread).  Here the bytes stream
// through a ring of pinned chunks instead: a pool of host threads copies
// chunk c into pinned memory with non-temporal stores (no read-for-ownership
// of the destination: 2 bytes of host DRAM traffic per byte instead of 3)
// while the copy engine moves chunk c-1 to the device, so a transfer runs at
// the slower of PCIe and the parallel host copy.  Device -> host is the
// mirror image.  The pool threads spin only while a transfer is active and
// sleep on a condition variable between transfers.
//
// C ABI (include/tc_collectives.h): tc_h2d_pageable / tc_d2h_pageable.
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "tc_collectives.h"

namespace {

constexpr size_t kChunkDefault = 16u << 20;  // bytes per pinned chunk
constexpr int kRing = 4;                     // chunks in flight

// dst = src with 16-B non-temporal stores (dst 16-B aligned)
void copy_nt(char* dst, const char* src, size_t n) {
  size_t i = 0;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    for (; i + 64 <= n; i += 64) {
      const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
      const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
      const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
      const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
    }
    _mm_sfence();
  }
  if (i < n) memcpy(dst + i, src + i, n - i);
}

class Stager {
 public:
  Stager() {
    unsigned hw = std::thread::hardware_concurrency();
    // copy threads per direction, measured on the B200 box (16 host threads,
    // 2 GiB): H2D 8 threads 40.3 ms (12: 43.4, 16: 46.0 -- more copy
    // threads compete with the copy engine's reads of the pinned ring),
    // D2H 12 threads 42.5 ms (8: 47.8, 16: 52.1)
    nthreads_ = static_cast<int>(std::max(1u, std::min(12u, hw ? hw : 1u)));
    h2d_threads_ = std::min(nthreads_, 8);
    d2h_threads_ = nthreads_;
    if (const char* e = getenv("TC_STAGE_THREADS")) {  // tuning / A-B switch
      nthreads_ = std::max(1, atoi(e));
      h2d_threads_ = d2h_threads_ = nthreads_;
    }
    if (const char* e = getenv("TC_STAGE_CHUNK_MB")) kChunk = std::max<size_t>(1, atoll(e)) << 20;
    for (int t = 1; t < nthreads_; ++t) workers_.emplace_back([this, t] { worker(t); });
  }
  ~Stager() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      quit_ = true;
      active_.store(true);
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }

  // (Re)allocate the pinned ring on first use.
  int ensure_ring() {
    if (ring_[0]) return 0;
    for (int b = 0; b < kRing; ++b) {
      if (cudaHostAlloc(reinterpret_cast<void**>(&ring_[b]), kChunk, cudaHostAllocDefault) !=
          cudaSuccess)
        return -1;
      if (cudaEventCreateWithFlags(&ev_[b], cudaEventDisableTiming) != cudaSuccess) return -1;
      used_[b] = false;
    }
    return 0;
  }

  int h2d(char* dst, const char* src, size_t bytes, cudaStream_t st) {
    std::lock_guard<std::mutex> call(call_mu_);  // one transfer at a time through the ring
    if (ensure_ring()) return -1;
    begin();
    int rc = 0;
    for (size_t off = 0, c = 0; off < bytes; off += kChunk, ++c) {
      const size_t len = std::min(kChunk, bytes - off);
      const int b = static_cast<int>(c % kRing);
      if (used_[b] && cudaEventSynchronize(ev_[b]) != cudaSuccess) { rc = -1; break; }
      parallel_copy(ring_[b], src + off, len, h2d_threads_);
      if (cudaMemcpyAsync(dst + off, ring_[b], len, cudaMemcpyHostToDevice, st) != cudaSuccess ||
          cudaEventRecord(ev_[b], st) != cudaSuccess) {
        rc = -1;
        break;
      }
      used_[b] = true;
    }
    end();
    return rc;
  }

  int d2h(char* dst, const char* src, size_t bytes, cudaStream_t st) {
    std::lock_guard<std::mutex> call(call_mu_);
    if (ensure_ring()) return -1;
    for (int b = 0; b < kRing; ++b)  // an earlier h2d's copies may still read the ring
      if (used_[b] && cudaEventSynchronize(ev_[b]) != cudaSuccess) return -1;
    begin();
    int rc = 0;
    const size_t nchunks = (bytes + kChunk - 1) / kChunk;
    // issue up to kRing device -> pinned copies ahead, drain them in order
    size_t issued = 0;
    auto issue = [&](size_t c) -> bool {
      const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
      const int b = static_cast<int>(c % kRing);
      return cudaMemcpyAsync(ring_[b], src + off, len, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
             cudaEventRecord(ev_[b], st) == cudaSuccess;
    };
    for (; issued < std::min<size_t>(nchunks, kRing); ++issued)
      if (!issue(issued)) { rc = -1; break; }
    for (size_t c = 0; rc == 0 && c < nchunks; ++c) {
      const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
      const int b = static_cast<int>(c % kRing);
      if (cudaEventSynchronize(ev_[b]) != cudaSuccess) { rc = -1; break; }
      parallel_copy(dst + off, ring_[b], len, d2h_threads_);
      if (issued < nchunks) {
        if (!issue(issued)) { rc = -1; break; }
        ++issued;
      }
    }
    for (int b = 0; b < kRing; ++b) used_[b] = false;
    end();
    return rc;
  }

  int threads() const { return nthreads_; }

 private:
  void begin() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      active_.store(true, std::memory_order_release);
    }
    cv_.notify_all();
  }
  void end() { active_.store(false, std::memory_order_release); }

  // dst[0, n) = src[0, n), split over the pool (the calling thread takes slice 0)
  void parallel_copy(char* dst, const char* src, size_t n, int nt) {
    if (nt <= 1 || n < (1u << 20)) {
      copy_nt(dst, src, n);
      return;
    }
    job_dst_ = dst;
    job_src_ = src;
    job_n_ = n;
    job_nt_ = nt;
    pending_.store(nthreads_ - 1, std::memory_order_relaxed);
    gen_.fetch_add(1, std::memory_order_release);
    slice(0, nt, dst, src, n);
    while (pending_.load(std::memory_order_acquire) != 0) _mm_pause();
  }
  void slice(int t, int nt, char* dst, const char* src, size_t n) {
    if (t >= nt) return;
    // 4-KB aligned cut points, so every slice but the last starts aligned
    const size_t per = (((n + nt - 1) / nt) + 4095) & ~size_t(4095);
    const size_t lo = std::min(n, per * t), hi = std::min(n, per * (t + 1));
    if (hi > lo) copy_nt(dst + lo, src + lo, hi - lo);
  }
  void worker(int t) {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return active_.load(std::memory_order_acquire) || quit_; });
        if (quit_) return;
      }
      // spin for jobs while the transfer is active
      while (true) {
        const uint64_t g = gen_.load(std::memory_order_acquire);
        if (g != seen) {
          seen = g;
          slice(t, job_nt_, job_dst_, job_src_, job_n_);
          pending_.fetch_sub(1, std::memory_order_acq_rel);
          continue;
        }
        if (!active_.load(std::memory_order_acquire) || quit_) break;
        for (int k = 0; k < 64; ++k) _mm_pause();
      }
    }
  }

  int nthreads_ = 1;
  size_t kChunk = kChunkDefault;
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_;
  std::atomic<bool> active_{false};
  std::atomic<bool> quit_{false};
  std::atomic<uint64_t> gen_{0};
  std::atomic<int> pending_{0};
  char* job_dst_ = nullptr;
  const char* job_src_ = nullptr;
  size_t job_n_ = 0;
  int job_nt_ = 1;
  int h2d_threads_ = 1, d2h_threads_ = 1;
  char* ring_[kRing] = {};
  cudaEvent_t ev_[kRing] = {};
  bool used_[kRing] = {};
};

// Process-lifetime singleton (never destroyed: no exit-order hazards).  A
// fork()ed child inherits the object but not its pool threads, so the child
// builds its own on first use.
Stager& stager() {
  static std::mutex mu;
  static Stager* s = nullptr;
  static pid_t owner = 0;
  std::lock_guard<std::mutex> lk(mu);
  if (s == nullptr || owner != getpid()) {
    s = new Stager();
    owner = getpid();
  }
  return *s;
}

}  // namespace

extern "C" {

int tc_h2d_pageable(void* dst_dev, const void* src_host, size_t bytes, void* stream) {
  if (bytes == 0) return TC_OK;
  if (!dst_dev || !src_host) return TC_BAD_CONFIG;
  return stager().h2d(static_cast<char*>(dst_dev), static_cast<const char*>(src_host), bytes,
                      static_cast<cudaStream_t>(stream)) == 0
             ? TC_OK
             : TC_CUDA_ERROR;
}

int tc_d2h_pageable(void* dst_host, const void* src_dev, size_t bytes, void* stream) {
  if (bytes == 0) return TC_OK;
  if (!dst_host || !src_dev) return TC_BAD_CONFIG;
  return stager().d2h(static_cast<char*>(dst_host), static_cast<const char*>(src_dev), bytes,
                      static_cast<cudaStream_t>(stream)) == 0
             ? TC_OK
             : TC_CUDA_ERROR;
}

}  // extern "C"
