// Host-frame upload (the RF ingest in front of
// das_beamform): pageable host RF -> pinned staging -> device, in pieces
// whose DMA overlaps the host copy of the next piece, each piece optionally
// followed by a stream-ordered store of a progress counter that a DAS launch
// already running on another stream waits on (g.tx_ready).
//
// The host copy is the part that bounds a one-frame call: a single-threaded
// memcpy of an 11.5 MB cfg2 frame runs at ~17 GB/s on the B200 box's host,
// and a DMA that reads a staging buffer the CPU has just written through its
// caches runs at ~35 instead of ~52 GB/s (tools/stage_probe.py).  So the
// copy is split over a small pool of host threads and uses non-temporal
// (streaming) stores, which leave the staging lines in DRAM, not dirty in
// the CPU caches.
#include <emmintrin.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include "bm_common.cuh"

namespace bm {
namespace {

// dst <- src with streaming stores (dst need not be aligned: an unaligned
// head goes through memcpy), then an sfence so the stores are globally
// visible before the caller signals completion
void stream_copy(char* d, const char* s, size_t n) {
  size_t head = (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15;
  if (head > n) head = n;
  memcpy(d, s, head);
  d += head;
  s += head;
  n -= head;
  size_t i = 0;
  for (; i + 64 <= n; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
  }
  memcpy(d + i, s + i, n - i);
  _mm_sfence();
}

// A fixed pool of copy threads, woken per piece.  Workers spin briefly
// between pieces (the next piece of a frame follows within microseconds),
// then sleep on a condition variable.  Calls from several host threads are
// serialised.  The pool is never destroyed (no join at process exit); a
// forked child (which inherits the pool but not its threads) builds its own.
class CopyPool {
 public:
  static CopyPool& get() {
    static std::atomic<CopyPool*> pool{nullptr};
    static std::mutex make_mu;
    CopyPool* p = pool.load(std::memory_order_acquire);
    if (p == nullptr || p->pid_ != getpid()) {
      std::lock_guard<std::mutex> lk(make_mu);
      p = pool.load(std::memory_order_acquire);
      if (p == nullptr || p->pid_ != getpid()) {
        p = new CopyPool();
        pool.store(p, std::memory_order_release);
      }
    }
    return *p;
  }

  void copy(char* d, const char* s, size_t n) {
    if (n < (size_t(1) << 18) || nthreads_ == 1) {
      stream_copy(d, s, n);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      d_ = d;
      s_ = s;
      n_ = n;
      pending_.store(nthreads_ - 1, std::memory_order_relaxed);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    part(0);
    while (pending_.load(std::memory_order_acquire) != 0) _mm_pause();
  }

  std::mutex& call_mutex() { return call_mu_; }

 private:
  CopyPool() : pid_(getpid()) {
    const unsigned hw = std::thread::hardware_concurrency();
    nthreads_ = (int)std::max(1u, std::min(8u, hw ? hw : 1u));
    for (int i = 1; i < nthreads_; ++i) std::thread([this, i] { worker(i); }).detach();
  }

  void part(int i) {
    // 64-B aligned part boundaries
    const size_t per = ((n_ / nthreads_) + 63) & ~size_t(63);
    const size_t o = std::min(n_, per * i), e = i == nthreads_ - 1 ? n_ : std::min(n_, o + per);
    if (e > o) stream_copy(d_ + o, s_ + o, e - o);
  }

  void worker(int i) {
    uint32_t seen = 0;
    for (;;) {
      uint32_t g;
      int spins = 0;
      while ((g = gen_.load(std::memory_order_acquire)) == seen) {
        if (++spins < 2000) {  // ~0.1 ms: the pieces of one frame, not the gap between frames
          _mm_pause();
        } else {
          std::unique_lock<std::mutex> lk(mu_);
          cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
        }
      }
      seen = g;
      part(i);
      pending_.fetch_sub(1, std::memory_order_release);
    }
  }

  const pid_t pid_;
  int nthreads_ = 1;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_;
  std::atomic<uint32_t> gen_{0};
  std::atomic<int> pending_{0};
  char* d_ = nullptr;
  const char* s_ = nullptr;
  size_t n_ = 0;
};

}  // namespace
}  // namespace bm

using namespace bm;

extern "C" int bm_host_upload(void* dst, const void* src, void* staging, const int64_t* ends,
                              int32_t n_pieces, uint32_t* counter, const uint32_t* values,
                              void* stream) {
  if (!dst || !src || !staging || !ends || n_pieces < 1 || (counter && !values))
    return BM_ERR_INVALID_ARGUMENT;
  for (int k = 0; k < n_pieces; ++k)
    if (ends[k] < (k ? ends[k - 1] : 0)) return BM_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  CopyPool& pool = CopyPool::get();
  std::lock_guard<std::mutex> lk(pool.call_mutex());
  int64_t o = 0;
  for (int k = 0; k < n_pieces; ++k) {
    const int64_t e = ends[k];
    if (e > o) {
      pool.copy(static_cast<char*>(staging) + o, static_cast<const char*>(src) + o,
                (size_t)(e - o));
      if (cudaMemcpyAsync(static_cast<char*>(dst) + o, static_cast<const char*>(staging) + o,
                          (size_t)(e - o), cudaMemcpyHostToDevice, s) != cudaSuccess)
        return BM_ERR_CUDA;
    }
    if (counter) {
      const int r = bm_stream_write_u32(counter, values[k], stream);
      if (r != BM_OK) return r;
    }
    o = e;
  }
  return BM_OK;
}
