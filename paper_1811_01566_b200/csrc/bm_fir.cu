// FIR pre-filter on the RF: sigproc.fir_filter
// (sigproc.py:36-45, the `fir_filter` operator pipeline.py:96-105).
//
//   y[n] = sum_m h[m] * x[n - m],  history before sample 0 is zero.
//
// The reference evaluates scipy.signal.lfilter(h, [1.0], x), which for a
// one-coefficient denominator is np.convolve(h, x) in float64 (the result
// type of f64 taps and any real frame), then the operator casts to the frame
// dtype.  Same here: f64 products and sums, written as f64 or rounded once to
// the output dtype.  numpy's convolve sums each output with a BLAS dot whose
// order is implementation-defined, so parity is "f64 round-off" (and f32
// outputs equal up to the final rounding); the sum runs from the oldest tap
// to the newest, the order of lfilter's transposed direct form.
//
// Layout: [outer][n][inner], filtering along n (axis=-1 -> inner = 1).  One
// CTA filters 256 consecutive outputs of one lane from a shared-memory window
// of 255 + M samples (f64), taps in shared memory.  FP64-pipe bound for long
// filters (2 DP ops per tap), HBM bound for short ones.
#include "bm_common.cuh"

namespace bm {

constexpr int kFirTile = 256;

template <typename TI, typename TO>
__global__ void __launch_bounds__(kFirTile) fir_kernel(const TI* __restrict__ x, TO* __restrict__ y,
                                                       const double* __restrict__ taps, int M,
                                                       int64_t n, int64_t inner,
                                                       int64_t tiles_per_lane) {
  extern __shared__ double fsm[];
  double* h = fsm;      // [M]
  double* w = fsm + M;  // [kFirTile + M - 1]: x[k0 - (M-1) .. k0 + kFirTile - 1]
  const int64_t lane = blockIdx.x / tiles_per_lane;
  const int64_t k0 = (blockIdx.x % tiles_per_lane) * kFirTile;
  const int64_t o = lane / inner, i = lane % inner;
  const TI* xl = x + o * n * inner + i;
  for (int m = threadIdx.x; m < M; m += kFirTile) h[m] = taps[m];
  for (int q = threadIdx.x; q < kFirTile + M - 1; q += kFirTile) {
    const int64_t k = k0 - (M - 1) + q;
    w[q] = (k >= 0 && k < n) ? (double)xl[k * inner] : 0.0;
  }
  __syncthreads();
  const int64_t k = k0 + threadIdx.x;
  if (k >= n) return;
  const double* wx = w + threadIdx.x + (M - 1);  // wx[-m] = x[k - m]
  // oldest available tap first; before sample M-1 the sum starts from the
  // zero initial state (lfilter's z = 0) instead of a product of padding
  double acc;
  int m;
  if (k >= M - 1) {
    acc = __dmul_rn(h[M - 1], wx[-(M - 1)]);
    m = M - 2;
  } else {
    acc = 0.0;
    m = (int)k;
  }
  for (; m >= 0; --m) acc = __dadd_rn(__dmul_rn(h[m], wx[-m]), acc);
  y[o * n * inner + k * inner + i] = (TO)acc;
}

// Contiguous lanes (inner == 1): each thread filters kFirR consecutive
// outputs, so a tap costs one shared-memory load of x for kFirR outputs (the
// others slide through registers) plus one broadcast load of h[m]: the loop
// is FP64-pipe bound instead of LSU bound (the one-output kernel above spends
// 3 wavefronts per output and tap).  The window is padded by one double per
// 16 so the stride-kFirR lane pattern hits every bank exactly twice.  The
// sum order per output is the one-output kernel's, bit for bit: the oldest
// tap first, a product of zero padding before sample 0 adds +-0 to the zero
// initial state and leaves it +0.
constexpr int kFirR = 4;
__host__ __device__ __forceinline__ int fir_pad(int q) { return q + (q >> 4); }

template <typename TI, typename TO>
__global__ void __launch_bounds__(kFirTile) fir_rows_kernel(const TI* __restrict__ x,
                                                            TO* __restrict__ y,
                                                            const double* __restrict__ taps, int M,
                                                            int64_t n, int64_t tiles_per_lane) {
  extern __shared__ double fsm[];
  double* h = fsm;      // [M]
  double* w = fsm + M;  // padded [kFirR * kFirTile + M - 1]: x[k0 - (M-1) ..]
  const int64_t lane = blockIdx.x / tiles_per_lane;
  const int64_t k0 = (blockIdx.x % tiles_per_lane) * (kFirR * kFirTile);
  const TI* xl = x + lane * n;
  for (int m = threadIdx.x; m < M; m += kFirTile) h[m] = taps[m];
  for (int q = threadIdx.x; q < kFirR * kFirTile + M - 1; q += kFirTile) {
    const int64_t k = k0 - (M - 1) + q;
    w[fir_pad(q)] = (k >= 0 && k < n) ? (double)xl[k] : 0.0;
  }
  __syncthreads();
  const int t = threadIdx.x;
  const int64_t kb = k0 + (int64_t)kFirR * t;
  if (kb >= n) return;
  // step j handles tap m = M-1-j; xr[r] = x[kb + r - m] = window[kFirR*t + r + j]
  double xr[kFirR], acc[kFirR];
#pragma unroll
  for (int r = 0; r < kFirR; ++r) xr[r] = w[fir_pad(kFirR * t + r)];
  {
    const double hm = h[M - 1];
#pragma unroll
    for (int r = 0; r < kFirR; ++r) {
      const double p = __dmul_rn(hm, xr[r]);
      acc[r] = kb + r >= M - 1 ? p : __dadd_rn(p, 0.0);
    }
  }
  for (int j = 1; j < M; ++j) {
#pragma unroll
    for (int r = 0; r < kFirR - 1; ++r) xr[r] = xr[r + 1];
    xr[kFirR - 1] = w[fir_pad(kFirR * t + kFirR - 1 + j)];
    const double hm = h[M - 1 - j];
#pragma unroll
    for (int r = 0; r < kFirR; ++r) acc[r] = __dadd_rn(__dmul_rn(hm, xr[r]), acc[r]);
  }
  TO* yl = y + lane * n;
#pragma unroll
  for (int r = 0; r < kFirR; ++r)
    if (kb + r < n) yl[kb + r] = (TO)acc[r];
}

template <typename TI, typename TO>
static int fir_launch(const void* x, void* y, int64_t outer, int64_t n, int64_t inner,
                      const double* taps, int M, cudaStream_t s) {
  if (inner == 1 && debug_override(BM_DBG_FIR_ONE_OUTPUT) <= 0) {  // test hook: one-output kernel
    const int win = kFirR * kFirTile + M - 1;
    const size_t smem = (size_t)(M + fir_pad(win - 1) + 1) * sizeof(double);
    if (smem <= 200 * 1024) {
      const int64_t tiles = (n + kFirR * kFirTile - 1) / (kFirR * kFirTile);
      const int64_t blocks = outer * tiles;
      if (blocks > 0x7fffffffLL) return BM_ERR_UNSUPPORTED;
      auto k = fir_rows_kernel<TI, TO>;
      if (smem > 48 * 1024 &&
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return BM_ERR_CUDA;
      k<<<(unsigned)blocks, kFirTile, smem, s>>>((const TI*)x, (TO*)y, taps, M, n, tiles);
      return cuda_status();
    }
  }
  const size_t smem = (size_t)(2 * M + kFirTile - 1) * sizeof(double);
  if (smem > 200 * 1024) return BM_ERR_UNSUPPORTED;
  const int64_t tiles = (n + kFirTile - 1) / kFirTile;
  const int64_t blocks = outer * inner * tiles;
  if (blocks > 0x7fffffffLL) return BM_ERR_UNSUPPORTED;
  auto k = fir_kernel<TI, TO>;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return BM_ERR_CUDA;
  k<<<(unsigned)blocks, kFirTile, smem, s>>>((const TI*)x, (TO*)y, taps, M, n, inner, tiles);
  return cuda_status();
}

}  // namespace bm

extern "C" int bm_fir_filter(int32_t in_dtype, const void* x, int32_t out_dtype, void* y,
                             int64_t outer, int64_t n, int64_t inner, const double* taps,
                             int32_t n_taps, void* stream) {
  using namespace bm;
  if (!x || !y || !taps || outer < 0 || inner < 0) return BM_ERR_INVALID_ARGUMENT;
  if (n_taps < 1) return BM_ERR_INVALID_ARGUMENT;
  if (n < 1) return BM_ERR_AXIS_TOO_SHORT;
  if ((in_dtype != BM_F32 && in_dtype != BM_F64) || (out_dtype != BM_F32 && out_dtype != BM_F64))
    return BM_ERR_INVALID_ARGUMENT;
  if (outer == 0 || inner == 0) return BM_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (in_dtype == BM_F32)
    return out_dtype == BM_F32 ? fir_launch<float, float>(x, y, outer, n, inner, taps, n_taps, s)
                               : fir_launch<float, double>(x, y, outer, n, inner, taps, n_taps, s);
  return out_dtype == BM_F32 ? fir_launch<double, float>(x, y, outer, n, inner, taps, n_taps, s)
                             : fir_launch<double, double>(x, y, outer, n, inner, taps, n_taps, s);
}
