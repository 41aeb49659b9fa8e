// Packed-f32x2 arithmetic, shared-memory and cp.async helpers for the DAS
// kernels (sm_100a).  Every floating-point helper rounds exactly once, as the
// reference's numpy/numba operators do (beamform.py:19-22).
#pragma once
#include "bm_common.cuh"

namespace bm {

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
constexpr int kMagicBits = 0x4B400000;

typedef unsigned long long u64;

__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
// split a packed pair into its two 32-bit halves (register-pair views, free)
__device__ __forceinline__ void unpk(u64 r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ float lo_f(u64 r) {
  float a, b;
  unpk(r, a, b);
  (void)b;
  return a;
}
__device__ __forceinline__ float hi_f(u64 r) {
  float a, b;
  unpk(r, a, b);
  (void)a;
  return b;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 add2_rm(u64 a, u64 b) {
  u64 d;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// Product rounded once, as a separate operation.  ptxas (CUDA 12.9) contracts
// mul.rn.f32x2 followed by add.rn.f32x2 into FFMA2 even under --fmad=false,
// which would drop the product's rounding (the reference rounds it:
// beamform.py:178-187).  fma(a, b, +0) = RN(a*b) is not contracted further;
// it differs from mul only in the sign of an exact-zero product, which cannot
// change the running sum (the accumulator starts at +0 and, in round-to-
// nearest, can never become -0, and x + (+-0) == x for every other x).
// tests/test_host.py::test_no_contracted_fma_in_das_kernels checks the SASS.
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(0ull));
  return d;
}



__device__ __forceinline__ float lds0(uint32_t a) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds1(uint32_t a) {
  float v;
  asm("ld.shared.f32 %0, [%1+4];" : "=f"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ void cp_async16(uint32_t smem_addr, const void* gptr, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_addr), "l"(gptr),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait1() {
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
}

// Chunk cursor: q -> (frame in group, transmit e, channel block cb), advanced
// incrementally (no integer division in the loop).  T = fl * n_tx + e.
struct Cursor {
  int fl, e, cb, T;
  // transmits e_lo .. e_hi - 1 of every pass (a launch may cover a range)
  __device__ __forceinline__ void next(int n_chunks, int e_lo, int e_hi) {
    if (++cb == n_chunks) {
      cb = 0;
      ++T;
      if (++e == e_hi) {
        e = e_lo;
        ++fl;
      }
    }
  }
};


}  // namespace bm
