// Per-SM throughput ceilings of the instructions the DAS kernels are built
// from, measured on the B200 itself (the numbers DESIGN.md's roofline uses).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
//   tools/microbench > profiles/microbench.json
//
// Each test runs a fixed number of independent operations per thread on
// 148 x k CTAs and reports warp-instructions per clock per SM (SM clock from
// cudaDevAttrClockRate is NOT used: the kernel reads clock64 per CTA and the
// result is ops / (elapsed SM cycles of the slowest CTA)).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;

__device__ __forceinline__ u64 fadd2(u64 a, u64 b) {
  u64 d;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 ffma2z(u64 a, u64 b) {
  u64 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(0ull));
  return d;
}

__device__ u64 g_sink;
__device__ unsigned long long g_cycles[4096];

constexpr int ITERS = 4096;

template <int KIND>
__global__ void bench(int salt) {
  extern __shared__ float sm[];
  const int tid = threadIdx.x;
  for (int i = tid; i < 8192; i += blockDim.x) sm[i] = (float)(i ^ salt);
  __syncthreads();
  u64 v[8];
  float f[8];
  double dv[8];
  uint32_t addr[8];
  for (int i = 0; i < 8; ++i) {
    v[i] = (u64)(tid + i) * 0x3f8000013f800001ull;
    f[i] = (float)(tid + i);
    dv[i] = (double)(tid + i);
    // conflict-free gather pattern: lanes spread over a 32-word window
    addr[i] = (uint32_t)__cvta_generic_to_shared(sm) + 4u * (uint32_t)((tid * 7 + i * 37) & 8191);
  }
  const u64 one = 0x3f8000003f800000ull;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) v[i] = fadd2(v[i], one);                       // FADD2
      if (KIND == 1) f[i] = __fadd_rn(f[i], 1.0f);                  // FADD
      if (KIND == 2) v[i] = ffma2z(v[i], one);                      // FFMA2 (x*y + 0)
      if (KIND == 3) {                                              // LDS.32 gather
        float x;
        asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(x) : "r"(addr[i]));
        f[i] += x;
        addr[i] ^= 4u;
      }
      if (KIND == 5) {                                              // LDS.32, 1 address
        float x;
        asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(x) : "r"(addr[0] & ~127u));
        f[i] += x;
      }
      if (KIND == 6) dv[i] = __dadd_rn(dv[i], 1.0);                  // DADD
      if (KIND == 7) dv[i] = __dmul_rn(dv[i], 1.0000001);            // DMUL
      if (KIND == 8) {  // LDS.64, lanes on consecutive 8-B words (2 wavefronts)
        double x;
        asm volatile("ld.volatile.shared.f64 %0, [%1];"
                     : "=d"(x)
                     : "r"(((uint32_t)__cvta_generic_to_shared(sm) + 8u * (uint32_t)((tid & 31) + 64 * i)) ^ (uint32_t)(it & 1) * 512u));
        dv[i] += x;
      }
      if (KIND == 4) {                                              // LDS.64
        u64 x;
        asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(x) : "r"(addr[i] & ~7u));
        v[i] ^= x;
        addr[i] ^= 8u;
      }
    }
  }
  __syncthreads();  // the slowest warp ends the interval
  const long long t1 = clock64();
  u64 acc = 0;
  for (int i = 0; i < 8; ++i) acc ^= v[i] ^ (u64)__float_as_uint(f[i]) ^ (u64)__double_as_longlong(dv[i]);
  if (acc == 0x1234567ull) g_sink = acc;
  if (tid == 0) g_cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const char* names[9] = {"fadd2", "fadd", "ffma2_rz", "lds32_gather", "lds64", "lds32_bcast",
                          "dadd", "dmul", "lds64_consecutive"};
  printf("{\"sm_count\": %d", sms);
  for (int kind = 0; kind < 9; ++kind) {
    for (int warps : {4, 8, 16}) {
      const int threads = 32 * warps;
      auto fn = kind == 0 ? bench<0> : kind == 1 ? bench<1> : kind == 2 ? bench<2>
               : kind == 3 ? bench<3> : kind == 4 ? bench<4> : kind == 5 ? bench<5>
               : kind == 6 ? bench<6> : kind == 7 ? bench<7> : bench<8>;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
      fn<<<sms, threads, 32768>>>(1);
      fn<<<sms, threads, 32768>>>(2);
      cudaDeviceSynchronize();
      unsigned long long cyc[4096];
      cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * sms);
      unsigned long long mx = 0;
      for (int i = 0; i < sms; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
      const double warp_instr = (double)warps * ITERS * 8;
      printf(", \"%s_w%d\": %.3f", names[kind], warps, warp_instr / (double)mx);
    }
  }
  printf(", \"unit\": \"warp-instructions per SM clock (one CTA per SM)\"}\n");
  return cudaGetLastError() != cudaSuccess;
}
