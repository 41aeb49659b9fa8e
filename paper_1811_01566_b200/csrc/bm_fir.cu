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

template <typename TI, typename TO>
static int fir_launch(const void* x, void* y, int64_t outer, int64_t n, int64_t inner,
                      const double* taps, int M, cudaStream_t s) {
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
