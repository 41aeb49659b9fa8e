// Does an LDS.64 whose 32 lanes touch <= 32 distinct 4-B words in distinct
// banks retire in one shared-memory wavefront?  (Decides whether
// frame-pair-interleaved RF windows halve the DAS gather cost.)
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/lds_wavefronts tools/lds_wavefronts.cu
//
// Reports warp-instructions per SM clock for LDS.32 / LDS.64 under lane ->
// word patterns: 'pairs16' (lane l reads 8-B word l/2: 16 distinct 8-B words,
// 32 banks once), 'dense32' (lane l reads 8-B word l: 64 words), 'das'
// (a cfg2-like pattern: 4 rows x 8 columns of pixels, ~14 distinct samples).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ unsigned long long g_cycles[1024];
__device__ unsigned long long g_sink;
constexpr int ITERS = 4096;

template <int W64>
__global__ void bench(const int* __restrict__ pat) {
  extern __shared__ __align__(16) float sm[];
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 8192; i += blockDim.x) sm[i] = (float)i;
  __syncthreads();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  uint32_t addr[8];
  for (int i = 0; i < 8; ++i) addr[i] = base + (uint32_t)(pat[lane] + 64 * i) * (W64 ? 8u : 4u);
  unsigned long long acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (W64) {
        unsigned long long x;
        asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(x) : "r"(addr[i]));
        acc += x;
      } else {
        uint32_t x;
        asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(x) : "r"(addr[i]));
        acc += x;
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (acc == 0x1234567ull) g_sink = acc;
  if (tid == 0) g_cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int pats[3][32];
  for (int l = 0; l < 32; ++l) {
    pats[0][l] = l / 2;
    pats[1][l] = l;
    // cfg2-like: row r = l/8 advances ~4 samples, column c = l%8 ~0.5 sample
    pats[2][l] = (l / 8) * 4 + ((l % 8) * 5) / 8;
  }
  const char* names[3] = {"pairs16", "dense32", "das"};
  int* dpat;
  cudaMalloc(&dpat, sizeof(pats));
  printf("{\"sm_count\": %d", sms);
  for (int p = 0; p < 3; ++p) {
    cudaMemcpy(dpat, pats[p], sizeof(pats[p]), cudaMemcpyHostToDevice);
    for (int w64 = 0; w64 < 2; ++w64) {
      auto fn = w64 ? bench<1> : bench<0>;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      const int warps = 16;
      fn<<<sms, 32 * warps, 65536>>>(dpat);
      fn<<<sms, 32 * warps, 65536>>>(dpat);
      cudaDeviceSynchronize();
      unsigned long long cyc[1024];
      cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * sms);
      unsigned long long mx = 0;
      for (int i = 0; i < sms; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
      printf(", \"%s_lds%d\": %.3f", names[p], w64 ? 64 : 32, (double)warps * ITERS * 8 / (double)mx);
    }
  }
  printf(", \"unit\": \"warp-instructions per SM clock\"}\n");
  return cudaGetLastError() != cudaSuccess;
}
