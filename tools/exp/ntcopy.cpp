// experiment: multi-threaded memcpy with / without non-temporal stores
#include <immintrin.h>
#include <stdint.h>
#include <string.h>
#include <thread>
#include <vector>

static void nt_range(char* d, const char* s, size_t n) {
  size_t i = 0;
  for (; i + 64 <= n; i += 64) {
    __m512i v = _mm512_loadu_si512((const void*)(s + i));
    _mm512_stream_si512((__m512i*)(d + i), v);
  }
  memcpy(d + i, s + i, n - i);
}

extern "C" void mt_copy(void* dst, const void* src, size_t n, int threads, int nt) {
  std::vector<std::thread> th;
  size_t per = ((n / threads) + 63) & ~(size_t)63;
  for (int t = 0; t < threads; ++t) {
    size_t o = (size_t)t * per;
    if (o >= n) break;
    size_t len = o + per > n ? n - o : per;
    th.emplace_back([=] {
      if (nt) nt_range((char*)dst + o, (const char*)src + o, len);
      else memcpy((char*)dst + o, (const char*)src + o, len);
    });
  }
  for (auto& t : th) t.join();
  if (nt) _mm_sfence();
}
