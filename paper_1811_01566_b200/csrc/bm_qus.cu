// Quantitative-ultrasound hooks on the envelope:
// qus.sliding_moments (qus.py:122-158) and the dense homodyned-K estimator
// qus.dense_forward / estimate_hk_map (qus.py:161-192).
//
// Moments: one WARP per window placement.  The lanes stride over the window
// (row-major), each keeping compensated (Kahan) f64 sums of x, x^2, x^3; the
// 32 partial sums meet in a shuffle tree and are divided by the window size.
// The reference takes numpy means of a strided view (pairwise summation) and
// x**3 through pow(); both are round-off-level differences, so parity is a
// relative tolerance, and exact wherever the sums are exact (the reference's
// constant-field and small-integer KATs, test_qus.py:24-38).
//
// Dense: one WARP per window; lane o computes neurons o, o+32, ... of each
// layer, out = act(W a + b), with the layer input in shared memory; weights
// and biases are read through the read-only cache.  relu / identity /
// softplus = np.logaddexp(0, z) (numpy's branch structure).
#include "bm_common.cuh"

namespace bm {

__device__ __forceinline__ void kahan_add(double& s, double& c, double v) {
  const double y = v - c;
  const double t = s + y;
  c = (t - s) - y;
  s = t;
}

template <typename T>
__global__ void __launch_bounds__(256) moments_kernel(const T* __restrict__ img, int64_t n_cols,
                                                      int wh, int ww, int sh, int sw,
                                                      int64_t out_r, int64_t out_c,
                                                      double* __restrict__ m1,
                                                      double* __restrict__ m2,
                                                      double* __restrict__ m3) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= out_r * out_c) return;
  const int64_t r0 = (w / out_c) * sh, c0 = (w % out_c) * sw;
  const int64_t cnt = (int64_t)wh * ww;
  double s1 = 0, s2 = 0, s3 = 0, k1 = 0, k2 = 0, k3 = 0;
  // the lane's (row, column) in the window advances by 32 elements per step:
  // dr rows and dc columns, one carry (no 64-bit division per element)
  const int dr = 32 / ww, dc = 32 % ww;
  int qr = lane / ww, qc = lane % ww;
  for (int64_t q = lane; q < cnt; q += 32) {
    const double x = (double)img[(r0 + qr) * n_cols + c0 + qc];
    qr += dr;
    qc += dc;
    if (qc >= ww) {
      qc -= ww;
      ++qr;
    }
    const double x2 = x * x;
    kahan_add(s1, k1, x);
    kahan_add(s2, k2, x2);
    kahan_add(s3, k3, x2 * x);
  }
  s1 -= k1;
  s2 -= k2;
  s3 -= k3;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    s3 += __shfl_xor_sync(0xffffffffu, s3, o);
  }
  if (lane == 0) {
    const double n = (double)cnt;
    m1[w] = s1 / n;
    m2[w] = s2 / n;
    m3[w] = s3 / n;
  }
}

enum { kActRelu = 0, kActIdentity = 1, kActSoftplus = 2 };

__device__ __forceinline__ double activate(double z, int act) {
  if (act == kActRelu) return z > 0.0 ? z : (z == z ? 0.0 : z);  // np.maximum(z, 0)
  if (act == kActSoftplus) {                                    // np.logaddexp(0, z)
    if (z == 0.0) return 0.6931471805599453;                    // x == y: x + log(2)
    return z > 0.0 ? z + log1p(exp(-z)) : log1p(exp(z));
  }
  return z;
}

// params: for each layer, W (out x in, row-major) then b (out), f64.
// dims: [n_layers][3] = {in, out, activation}.
__global__ void __launch_bounds__(128) dense_kernel(const double* __restrict__ x, int64_t n,
                                                    const double* __restrict__ params,
                                                    const int* __restrict__ dims, int n_layers,
                                                    int max_width, double* __restrict__ y) {
  extern __shared__ double dsm[];  // per warp: two activation buffers of max_width
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (row >= n) return;
  double* a = dsm + (size_t)warp * 2 * max_width;
  double* b = a + max_width;
  const int in0 = dims[0];
  for (int i = lane; i < in0; i += 32) a[i] = x[row * in0 + i];
  __syncwarp();
  const double* p = params;
  for (int l = 0; l < n_layers; ++l) {
    const int in_w = dims[3 * l], out_w = dims[3 * l + 1], act = dims[3 * l + 2];
    const double* W = p;
    const double* bias = p + (size_t)out_w * in_w;
    for (int o = lane; o < out_w; o += 32) {
      double acc = 0.0;
      for (int i = 0; i < in_w; ++i) acc += __ldg(W + (size_t)o * in_w + i) * a[i];
      b[o] = activate(acc + __ldg(bias + o), act);
    }
    __syncwarp();
    double* t = a;
    a = b;
    b = t;
    p = bias + out_w;
  }
  const int out_w = dims[3 * (n_layers - 1) + 1];
  for (int o = lane; o < out_w; o += 32) y[row * out_w + o] = a[o];
}

}  // namespace bm

extern "C" int bm_sliding_moments(int32_t dtype, const void* img, int64_t n_rows, int64_t n_cols,
                                  int32_t wh, int32_t ww, int32_t sh, int32_t sw, double* m1,
                                  double* m2, double* m3, void* stream) {
  using namespace bm;
  if (!img || !m1 || !m2 || !m3 || n_rows < 1 || n_cols < 1) return BM_ERR_INVALID_ARGUMENT;
  if (wh < 1 || ww < 1 || sh < 1 || sw < 1 || wh > n_rows || ww > n_cols)
    return BM_ERR_INVALID_ARGUMENT;
  const int64_t out_r = (n_rows - wh) / sh + 1, out_c = (n_cols - ww) / sw + 1;
  const int64_t threads = out_r * out_c * 32;
  const int64_t blocks = (threads + 255) / 256;
  if (blocks > 0x7fffffffLL) return BM_ERR_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == BM_F32)
    moments_kernel<float><<<(unsigned)blocks, 256, 0, s>>>((const float*)img, n_cols, wh, ww, sh,
                                                            sw, out_r, out_c, m1, m2, m3);
  else if (dtype == BM_F64)
    moments_kernel<double><<<(unsigned)blocks, 256, 0, s>>>((const double*)img, n_cols, wh, ww,
                                                             sh, sw, out_r, out_c, m1, m2, m3);
  else
    return BM_ERR_INVALID_ARGUMENT;
  return cuda_status();
}

extern "C" int bm_dense_forward(const double* x, int64_t n, const double* params,
                                const int32_t* dims, int32_t n_layers, int32_t max_width,
                                double* y, void* stream) {
  using namespace bm;
  if (!x || !params || !dims || !y || n < 0 || n_layers < 1 || max_width < 1)
    return BM_ERR_INVALID_ARGUMENT;
  if (n == 0) return BM_OK;
  const size_t smem = (size_t)4 * 2 * max_width * sizeof(double);
  if (smem > 200 * 1024) return BM_ERR_UNSUPPORTED;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return BM_ERR_CUDA;
  const int64_t blocks = (n + 3) / 4;
  if (blocks > 0x7fffffffLL) return BM_ERR_UNSUPPORTED;
  dense_kernel<<<(unsigned)blocks, 128, smem, (cudaStream_t)stream>>>(x, n, params, dims, n_layers,
                                                                      max_width, y);
  return cuda_status();
}
