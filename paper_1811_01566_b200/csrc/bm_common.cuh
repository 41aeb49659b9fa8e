// Shared helpers for the bmode200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>

#include "../../include/bmode200.h"

namespace bm {

// Exactly-rounded scalar arithmetic, one IEEE rounding per operator and no
// FMA contraction: this is what makes the GPU delays and sums bitwise equal to
// the reference's numpy plan + numba kernel (beamform.py:19-22, 211-216).
template <typename T> struct R;
template <> struct R<float> {
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
  static __device__ __forceinline__ float sqrt(float a) { return __fsqrt_rn(a); }
  static __device__ __forceinline__ float floor(float a) { return floorf(a); }
  static __device__ __forceinline__ float from_double(double a) { return __double2float_rn(a); }
};
template <> struct R<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double sqrt(double a) { return __dsqrt_rn(a); }
  static __device__ __forceinline__ double floor(double a) { return ::floor(a); }
  static __device__ __forceinline__ double from_double(double a) { return a; }
};

// bm_debug_set / bm_debug_get storage (one definition across translation units)
inline std::atomic<int> g_debug_overrides[BM_DBG_COUNT];
inline int debug_override(int key) {
  return g_debug_overrides[key].load(std::memory_order_relaxed);
}

inline int cuda_status() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BM_OK : BM_ERR_CUDA;
}

inline int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Transmits of the launch's frame that have landed in device memory, for a
// launch started while its RF is still being copied in (g.tx_ready; the copy
// side advances the counter with bm_stream_write_u32): waits until the
// counter has passed base + need (modulo 2^32) and returns how many
// transmits are then known present.  The acquire orders this thread's later
// RF reads after the copies; a TMA issuer adds fence.proxy.async.  A counter
// that never arrives (a host-side bug) traps after ~10 s instead of leaving
// the device hung.
__device__ __forceinline__ int wait_tx_ready(const uint32_t* ctr, uint32_t base, int need) {
  uint64_t t_first = 0;
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    const int have = (int)(v - base);
    if (have >= need) return have;
    uint64_t now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (t_first == 0)
      t_first = now;
    else if (now - t_first > 10000000000ull)
      __trap();
    __nanosleep(200);
  }
}

// TMA DAS kernel (bm_das_tma.cu)
int das_tma_eligible(const bm_das_geometry& g, int64_t rf_stride);
int das_tma_shape(const bm_das_geometry& g, int n_frames, int32_t* shape);
// returns -1 when this launch cannot use the TMA kernel (caller falls back)
int das_tma_launch(const bm_das_geometry& g, const void* rf, int64_t rf_stride, void* out,
                   int64_t out_stride, int n_frames, int e_begin, int e_end, int accumulate,
                   cudaStream_t s);  // 0 scalar, 1 pair, 2 hybrid

// f64 twin of the TMA kernel (bm_das_tma64.cu)
int das_tma64_eligible(const bm_das_geometry& g, int64_t rf_stride);
int das_tma64_shape(const bm_das_geometry& g, int n_frames, int32_t* shape);
int das_table64_build(const bm_das_geometry& g, double* table, cudaStream_t s);
int das_tma64_launch(const bm_das_geometry& g, const void* rf, int64_t rf_stride, void* out,
                     int64_t out_stride, int n_frames, int e_begin, int e_end, int accumulate,
                     cudaStream_t s);

// DAS kernel selection: 0 auto (TMA where it applies, else generic), 1 generic
inline int das_kernel_choice() { return debug_override(BM_DBG_DAS_KERNEL); }

}  // namespace bm
