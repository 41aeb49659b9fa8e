// K2: analytic signal / envelope / dynamic adjustment (sm_100a).
//
// Replaces sigproc.py:48-97 (analytic_signal via scipy.fft, np.abs,
// dynamic_adjustment).  For a power-of-two lane length the whole
//   FFT -> one-sided gain -> IFFT -> |.| -> per-frame max
// chain runs inside one CTA's shared memory (radix-2, L lanes per CTA), so
// the complex I/Q data never touches HBM.  Other lengths use an exact
// O(n^2) DFT per lane (same gain convention, sigproc.py:63-70).
#include "bm_common.cuh"

namespace bm {

template <typename T> struct C2;
template <> struct C2<float> { using type = float2; };
template <> struct C2<double> { using type = double2; };

template <typename T> struct PeakBits;
template <> struct PeakBits<float> {
  using U = unsigned int;
  static __device__ __forceinline__ U bits(float v) { return __float_as_uint(v); }
  static __device__ __forceinline__ float value(U b) { return __uint_as_float(b); }
};
template <> struct PeakBits<double> {
  using U = unsigned long long;
  static __device__ __forceinline__ U bits(double v) { return (U)__double_as_longlong(v); }
  static __device__ __forceinline__ double value(U b) { return __longlong_as_double((long long)b); }
};

// sigproc.py:63-70
template <typename T>
__device__ __forceinline__ T hilbert_gain(int64_t k, int64_t n) {
  if (k == 0) return T(1);
  if ((n & 1) == 0) {
    if (k == n / 2) return T(1);
    return k < n / 2 ? T(2) : T(0);
  }
  return k <= (n - 1) / 2 ? T(2) : T(0);
}

template <typename T>
__device__ __forceinline__ typename C2<T>::type cmul(typename C2<T>::type a,
                                                     typename C2<T>::type b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}

template <typename T>
__device__ __forceinline__ T magnitude(T re, T im) {
  return hypot(re, im);
}

template <typename T>
__device__ __forceinline__ void block_peak(T v, typename PeakBits<T>::U* peak) {
  // warp max then one atomic per warp (values are >= 0, so IEEE bits order
  // like the values)
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(peak, PeakBits<T>::bits(v));
}

enum OutMode { kComplex = 0, kEnvelope = 1 };

// Power-of-two lanes: L (a power of two) lanes of length n per CTA, radix-2
// DIT in shared memory.  All index arithmetic is 32-bit shifts and masks
// (n, L powers of two); consecutive threads touch consecutive lanes on
// global loads/stores (coalesced rows of L values) and consecutive
// butterflies of one lane in shared memory.
template <typename T, int MODE>
__global__ void __launch_bounds__(256) analytic_pow2_kernel(const T* __restrict__ x, T* __restrict__ out,
                                                            typename PeakBits<T>::U* __restrict__ peak,
                                                            int n, int log2n, int64_t inner,
                                                            int log2L) {
  using V = typename C2<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int L = 1 << log2L;
  V* tw = reinterpret_cast<V*>(smem_raw);  // [n/2]
  V* buf = tw + n / 2;                       // [L][n]
  const int64_t o = blockIdx.y;
  const int64_t i_base = (int64_t)blockIdx.x * L;
  const int half_n = n >> 1;
  const int nt = blockDim.x;

  for (int k = threadIdx.x; k < half_n; k += nt) {
    double s, c;
    sincospi(-2.0 * (double)k / (double)n, &s, &c);
    tw[k] = V{(T)c, (T)s};
  }
  const T* xo = x + o * (int64_t)n * inner + i_base;
  const bool full = i_base + L <= inner;
  for (int idx = threadIdx.x; idx < (n << log2L); idx += nt) {
    const int l = idx & (L - 1), k = idx >> log2L;
    const int r = __brev(k) >> (32 - log2n);
    T v = T(0);
    if (full || i_base + l < inner) v = xo[(int64_t)k * inner + l];
    buf[(l << log2n) + r] = V{v, T(0)};
  }
  __syncthreads();

  // FFT -> gain -> bit reversal -> inverse FFT, one warp per lane: the
  // passes only need warp-level synchronisation
  const int warp = threadIdx.x >> 5, wl = threadIdx.x & 31, nwarps = nt >> 5;
  for (int l = warp; l < L; l += nwarps) {
    V* lane = buf + (l << log2n);
    for (int pass = 0; pass < 2; ++pass) {
      const T sign = pass == 0 ? T(1) : T(-1);  // inverse: conjugate twiddles
      for (int s = 1; s <= log2n; ++s) {
        const int h = 1 << (s - 1);
        for (int bb = wl; bb < half_n; bb += 32) {
          const int pos = bb & (h - 1);
          const int i = ((bb >> (s - 1)) << s) + pos;
          V w = tw[pos << (log2n - s)];
          w.y *= sign;
          const V u = lane[i];
          const V t = cmul<T>(w, lane[i + h]);
          lane[i] = V{u.x + t.x, u.y + t.y};
          lane[i + h] = V{u.x - t.x, u.y - t.y};
        }
        __syncwarp();
      }
      if (pass == 0) {
        // one-sided gain, then bit-reverse permutation for the inverse DIT
        for (int k = wl; k < n; k += 32) {
          const int r = __brev(k) >> (32 - log2n);
          if (k > r) continue;
          const T gk = hilbert_gain<T>(k, n), gr = hilbert_gain<T>(r, n);
          const V a = lane[k], bv = lane[r];
          lane[k] = V{bv.x * gr, bv.y * gr};
          lane[r] = V{a.x * gk, a.y * gk};
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();

  const T inv_n = T(1) / T(n);
  T vmax = T(0);
  for (int idx = threadIdx.x; idx < (n << log2L); idx += nt) {
    const int l = idx & (L - 1), k = idx >> log2L;
    if (!full && i_base + l >= inner) continue;
    const V z = buf[(l << log2n) + k];
    const T re = z.x * inv_n, im = z.y * inv_n;
    const int64_t g = o * (int64_t)n * inner + (int64_t)k * inner + i_base + l;
    if (MODE == kComplex) {
      reinterpret_cast<V*>(out)[g] = V{re, im};
    } else {
      const T e = magnitude(re, im);
      out[g] = e;
      vmax = e > vmax ? e : vmax;
    }
  }
  if (MODE == kEnvelope) block_peak<T>(vmax, peak + o);
}

// General n: exact DFT per lane (one lane per CTA).  Positive-frequency bins
// only (the gain zeroes the rest), twiddles from an exact (j*k mod n) table.
template <typename T, int MODE>
__global__ void __launch_bounds__(256) analytic_dft_kernel(const T* __restrict__ x, T* __restrict__ out,
                                                           typename PeakBits<T>::U* __restrict__ peak,
                                                           int64_t n, int64_t inner) {
  using V = typename C2<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* tw = reinterpret_cast<V*>(smem_raw);  // [n]
  const int64_t nb = n / 2 + 1;           // bins 0..n/2
  V* X = tw + n;                           // [nb]
  T* xs = reinterpret_cast<T*>(X + nb);    // [n]
  const int64_t o = blockIdx.y, i = blockIdx.x;
  const int64_t base = o * n * inner + i;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) {
    double s, c;
    sincospi(-2.0 * (double)k / (double)n, &s, &c);
    tw[k] = V{(T)c, (T)s};
    xs[k] = x[base + k * inner];
  }
  __syncthreads();
  for (int64_t k = threadIdx.x; k < nb; k += blockDim.x) {
    T re = 0, im = 0;
    int64_t r = 0;
    for (int64_t j = 0; j < n; ++j) {
      const V w = tw[r];
      re += xs[j] * w.x;
      im += xs[j] * w.y;
      r += k;
      if (r >= n) r -= n;
    }
    const T g = hilbert_gain<T>(k, n);
    X[k] = V{re * g, im * g};
  }
  __syncthreads();
  const T inv_n = T(1) / T(n);
  T vmax = T(0);
  for (int64_t t = threadIdx.x; t < n; t += blockDim.x) {
    T re = 0, im = 0;
    int64_t r = 0;
    for (int64_t k = 0; k < nb; ++k) {
      const V w = tw[r];  // exp(-2 pi i k t / n); inverse uses the conjugate
      const V a = X[k];
      re += a.x * w.x + a.y * w.y;
      im += a.y * w.x - a.x * w.y;
      r += t;
      if (r >= n) r -= n;
    }
    re *= inv_n;
    im *= inv_n;
    if (MODE == kComplex) {
      reinterpret_cast<V*>(out)[base + t * inner] = V{re, im};
    } else {
      const T e = magnitude(re, im);
      out[base + t * inner] = e;
      vmax = e > vmax ? e : vmax;
    }
  }
  if (MODE == kEnvelope) block_peak<T>(vmax, peak + o);
}

template <typename T>
__global__ void envelope_kernel(const T* __restrict__ z, T* __restrict__ e, int64_t count) {
  using V = typename C2<T>::type;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const V v = reinterpret_cast<const V*>(z)[i];
    e[i] = magnitude(v.x, v.y);
  }
}

template <typename T>
__global__ void peak_kernel(const T* __restrict__ e, typename PeakBits<T>::U* __restrict__ peak,
                            int64_t frame_elems) {
  const int64_t f = blockIdx.y;
  const T* ef = e + f * frame_elems;
  T vmax = T(0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < frame_elems;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T v = ef[i];
    vmax = v > vmax ? v : vmax;
  }
  block_peak<T>(vmax, peak + f);
}

template <typename T>
__device__ __forceinline__ T log10_rn(T v);
template <>
__device__ __forceinline__ float log10_rn<float>(float v) {
  // f32 log10 (<= 2 ulp; exact 0 at the peak, where v == 1): the display
  // tolerance vs numpy's own f32 log10 is 2e-6 of a [0, 1] display value
  return log10f(v);
}
template <>
__device__ __forceinline__ double log10_rn<double>(double v) {
  return log10(v);
}

// sigproc.py:90-96, in the input precision: q = e/peak; db = 20*log10(q);
// out = clip(db + R, 0, R) / R; zeros map to 0 without the log.
template <typename T>
__global__ void display_kernel(const T* __restrict__ e, const typename PeakBits<T>::U* __restrict__ peak,
                               T* __restrict__ disp, int32_t* __restrict__ status,
                               int64_t frame_elems, double range_db) {
  using O = R<T>;
  const int64_t f = blockIdx.y;
  const T pk = PeakBits<T>::value(peak[f]);
  if (blockIdx.x == 0 && threadIdx.x == 0 && status) status[f] = pk > T(0) ? 0 : 1;
  const T r = O::from_double(range_db);
  // q = e/peak at least 0.1 % below 10^(-R/20) gives 20 log10 q + R < 0 with
  // a margin far above every rounding of the chain: the clip makes it exactly
  // 0, so the (f64) log is skipped -- most pixels of a 30 dB display
  const T q0 = (T)(pow(10.0, -range_db / 20.0) * 0.999);
  const T* ef = e + f * frame_elems;
  T* df = disp + f * frame_elems;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < frame_elems;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T v = ef[i];
    T outv = T(0);
    const T q = O::div(v, pk);
    if (v > T(0) && pk > T(0) && !(q < q0)) {
      const T db = O::mul(T(20), log10_rn<T>(q));
      T s = O::add(db, r);
      s = s < T(0) ? T(0) : (s > r ? r : s);
      outv = O::div(s, r);
    }
    df[i] = outv;
  }
}

static inline bool is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }
static inline int ilog2(int64_t n) {
  int l = 0;
  while (((int64_t)1 << l) < n) ++l;
  return l;
}


// ---------------------------------------------------------------------------
// f32 lanes of n = 32 * R samples (R = 8, 16, 32: n = 256 .. 1024), one WARP
// per lane, data in REGISTERS.  With j = t + 32 i (t = lane, i < R) and
// k = k1 + R k2:
//   X[k1 + R k2] = sum_t W32^(t k2) * [ Wn^(t k1) * sum_i x[t + 32 i] WR^(i k1) ]
// so a lane's transform is an R-point DFT inside each thread (radix-2 DIF,
// compile-time register indices), a per-thread twiddle, and a 32-point DFT
// across the warp (radix-2 DIF over __shfl_xor).  The spectrum ends up
// bit-reversed in both indices, which the one-sided gain reads directly; the
// inverse runs the mirror image (DIT across lanes, twiddle, DIT in registers)
// and lands in natural order.  Shared memory holds only the twiddle table and
// the CTA's [n][8] tile for coalesced 32-B row loads and stores: two
// __syncthreads per CTA instead of one __syncwarp per radix-2 pass.
__device__ __forceinline__ float2 c_add(float2 a, float2 b) { return {a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ float2 c_sub(float2 a, float2 b) { return {a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ float2 c_mul(float2 a, float2 w) {
  return {a.x * w.x - a.y * w.y, a.x * w.y + a.y * w.x};
}
__device__ __forceinline__ float2 c_conj(float2 a) { return {a.x, -a.y}; }

template <int R>
__device__ __forceinline__ int brev_c(int p) {  // bit reversal of p in log2(R) bits
  int r = 0;
#pragma unroll
  for (int b = 1; b < R; b <<= 1) r = (r << 1) | ((p & b) ? 1 : 0);
  return r;
}

template <int MODE, int R>
__global__ void __launch_bounds__(256) analytic_reg_kernel(const float* __restrict__ x,
                                                           float* __restrict__ out,
                                                           unsigned* __restrict__ peak,
                                                           int64_t inner) {
  constexpr int N = 32 * R, L = 8, LP = L + 1;  // LP: padded tile row (conflict-free columns)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* tw = reinterpret_cast<float2*>(smem_raw);  // [N] Wn^m
  float* tile = reinterpret_cast<float*>(tw + N);     // real: [N][LP]; complex: [N][LP] float2
  const int tid = threadIdx.x, warp = tid >> 5, t = tid & 31;
  const int64_t o = blockIdx.y, i_base = (int64_t)blockIdx.x * L;
  const int lanes = (int)(inner - i_base < L ? inner - i_base : L);

  for (int m = tid; m < N; m += 256) {
    double sn, cs;
    sincospi(-2.0 * (double)m / (double)N, &sn, &cs);
    tw[m] = make_float2((float)cs, (float)sn);
  }
  const float* xo = x + o * (int64_t)N * inner + i_base;
  {
    // all R loads of a thread in flight before the first shared-memory store
    float ld[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int idx = tid + 256 * q, l = idx & (L - 1), k = idx >> 3;
      ld[q] = l < lanes ? __ldg(xo + (int64_t)k * inner + l) : 0.0f;
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int idx = tid + 256 * q;
      tile[(idx >> 3) * LP + (idx & (L - 1))] = ld[q];
    }
  }
  __syncthreads();

  float2 v[R];
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = make_float2(tile[(t + 32 * i) * LP + warp], 0.0f);

  // (1) R-point DFT over i in registers, radix-2 DIF: v[p] = A[brev(p)]
#pragma unroll
  for (int h = R / 2; h >= 1; h >>= 1)
#pragma unroll
    for (int b = 0; b < R; b += 2 * h)
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const float2 a = v[b + j], c = v[b + j + h];
        v[b + j] = c_add(a, c);
        v[b + j + h] = j == 0 ? c_sub(a, c) : c_mul(c_sub(a, c), tw[j * (N / (2 * h))]);
      }
  // (2) twiddle Wn^(t k1)
#pragma unroll
  for (int p = 1; p < R; ++p) v[p] = c_mul(v[p], tw[t * brev_c<R>(p)]);
  // (3) 32-point DIF across the warp: lane t then holds k2 = brev5(t)
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const bool up = (t & h) != 0;
    const float2 w = tw[(t & (h - 1)) * (N / (2 * h))];
#pragma unroll
    for (int p = 0; p < R; ++p) {
      float2 q;
      q.x = __shfl_xor_sync(0xffffffffu, v[p].x, h);
      q.y = __shfl_xor_sync(0xffffffffu, v[p].y, h);
      v[p] = up ? c_mul(c_sub(q, v[p]), w) : c_add(v[p], q);
    }
  }
  // (4) one-sided gain (sigproc.py:63-70) at k = k1 + R k2
  {
    const int k2 = __brev(t) >> 27;
#pragma unroll
    for (int p = 0; p < R; ++p) {
      const int k = brev_c<R>(p) + R * k2;
      const float gk = (k == 0 || k == N / 2) ? 1.0f : (k < N / 2 ? 2.0f : 0.0f);
      v[p] = make_float2(v[p].x * gk, v[p].y * gk);
    }
  }
  // (5) inverse 32-point DIT across the warp (bit-reversed in, natural out)
#pragma unroll
  for (int h = 1; h <= 16; h <<= 1) {
    const bool up = (t & h) != 0;
    const float2 w = c_conj(tw[(t & (h - 1)) * (N / (2 * h))]);
#pragma unroll
    for (int p = 0; p < R; ++p) {
      float2 q;
      q.x = __shfl_xor_sync(0xffffffffu, v[p].x, h);
      q.y = __shfl_xor_sync(0xffffffffu, v[p].y, h);
      const float2 tmp = c_mul(up ? v[p] : q, w);
      v[p] = up ? c_sub(q, tmp) : c_add(v[p], tmp);
    }
  }
  // (6) twiddle Wn^(-t k1)
#pragma unroll
  for (int p = 1; p < R; ++p) v[p] = c_mul(v[p], c_conj(tw[t * brev_c<R>(p)]));
  // (7) inverse R-point DIT in registers: v[i] = n * x'[t + 32 i]
#pragma unroll
  for (int h = 1; h < R; h <<= 1)
#pragma unroll
    for (int b = 0; b < R; b += 2 * h)
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const float2 a = v[b + j];
        const float2 c = j == 0 ? v[b + j + h] : c_mul(v[b + j + h], c_conj(tw[j * (N / (2 * h))]));
        v[b + j] = c_add(a, c);
        v[b + j + h] = c_sub(a, c);
      }

  __syncthreads();  // tile reused for the output
  const float inv_n = 1.0f / (float)N;
  float vmax = 0.0f;
  if (MODE == kComplex) {
    float2* tc = reinterpret_cast<float2*>(tile);
#pragma unroll
    for (int i = 0; i < R; ++i)
      tc[(t + 32 * i) * LP + warp] = make_float2(v[i].x * inv_n, v[i].y * inv_n);
  } else {
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const float e = magnitude(v[i].x * inv_n, v[i].y * inv_n);
      tile[(t + 32 * i) * LP + warp] = e;
      if (warp < lanes) vmax = e > vmax ? e : vmax;
    }
  }
  __syncthreads();
  const int64_t g0 = o * (int64_t)N * inner + i_base;
  for (int idx = tid; idx < N * L; idx += 256) {
    const int l = idx & (L - 1), k = idx >> 3;
    if (l >= lanes) continue;
    if (MODE == kComplex)
      reinterpret_cast<float2*>(out)[g0 + (int64_t)k * inner + l] =
          reinterpret_cast<const float2*>(tile)[k * LP + l];
    else
      out[g0 + (int64_t)k * inner + l] = tile[k * LP + l];
  }
  if (MODE == kEnvelope) block_peak<float>(vmax, peak + o);
}

template <typename T, int MODE>
static int launch_analytic_reg(const T*, T*, typename PeakBits<T>::U*, int64_t, int64_t, int64_t,
                               cudaStream_t) {
  return -1;  // f64: shared-memory radix-2 kernel
}
template <>
int launch_analytic_reg<float, kEnvelope>(const float*, float*, unsigned*, int64_t, int64_t,
                                          int64_t, cudaStream_t);
template <>
int launch_analytic_reg<float, kComplex>(const float*, float*, unsigned*, int64_t, int64_t,
                                         int64_t, cudaStream_t);

template <int MODE>
static int launch_reg_f32(const float* x, float* out, unsigned* peak, int64_t outer, int64_t n,
                          int64_t inner, cudaStream_t s) {
  const char* e = getenv("BM_FFT_KERNEL");  // "smem": the radix-2 shared-memory kernel
  if (e && !strcmp(e, "smem")) return -1;
  if (n != 256 && n != 512 && n != 1024) return -1;
  if (inner > ((int64_t)1 << 34) || outer > 65535) return -1;
  const size_t tile = (size_t)n * 9 * (MODE == kComplex ? 8 : 4);
  const size_t smem = (size_t)n * 8 + tile;
  auto k = n == 256 ? analytic_reg_kernel<MODE, 8>
                    : (n == 512 ? analytic_reg_kernel<MODE, 16> : analytic_reg_kernel<MODE, 32>);
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return BM_ERR_CUDA;
  dim3 grid((unsigned)((inner + 7) / 8), (unsigned)outer);
  k<<<grid, 256, smem, s>>>(x, out, peak, inner);
  return cuda_status();
}
template <>
int launch_analytic_reg<float, kEnvelope>(const float* x, float* out, unsigned* peak, int64_t outer,
                                          int64_t n, int64_t inner, cudaStream_t s) {
  return launch_reg_f32<kEnvelope>(x, out, peak, outer, n, inner, s);
}
template <>
int launch_analytic_reg<float, kComplex>(const float* x, float* out, unsigned* peak, int64_t outer,
                                         int64_t n, int64_t inner, cudaStream_t s) {
  return launch_reg_f32<kComplex>(x, out, peak, outer, n, inner, s);
}

template <typename T, int MODE>
static int launch_analytic(const T* x, T* out, typename PeakBits<T>::U* peak, int64_t outer,
                           int64_t n, int64_t inner, cudaStream_t s) {
  using V = typename C2<T>::type;
  if (outer > 65535) return BM_ERR_UNSUPPORTED;
  {
    const int rc = launch_analytic_reg<T, MODE>(x, out, peak, outer, n, inner, s);
    if (rc >= 0) return rc;
  }
  if (is_pow2(n)) {
    if (n > (1 << 20) || inner > (int64_t)1 << 40) return BM_ERR_UNSUPPORTED;
    const size_t lane_bytes = (size_t)n * sizeof(V);
    const size_t tw_bytes = (size_t)(n / 2) * sizeof(V);
    // lanes per CTA: a power of two, enough for 32 B row segments when the
    // image is wide, few enough to give >= 2 waves of CTAs
    int log2L = 0;
    while ((2 << log2L) <= 8 && (2 << log2L) <= inner &&
           tw_bytes + (size_t)(2 << log2L) * lane_bytes <= 96 * 1024)
      ++log2L;
    const size_t smem = tw_bytes + ((size_t)1 << log2L) * lane_bytes;
    if (smem > 220 * 1024) return BM_ERR_UNSUPPORTED;
    auto k = analytic_pow2_kernel<T, MODE>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return BM_ERR_CUDA;
    const int64_t L = (int64_t)1 << log2L;
    dim3 grid((unsigned)((inner + L - 1) / L), (unsigned)outer);
    k<<<grid, 256, smem, s>>>(x, out, peak, (int)n, ilog2(n), inner, log2L);
  } else {
    const size_t smem = (size_t)n * sizeof(V) + (size_t)(n / 2 + 1) * sizeof(V) + (size_t)n * sizeof(T);
    if (smem > 220 * 1024 || inner > 0x7fffffff) return BM_ERR_UNSUPPORTED;
    auto k = analytic_dft_kernel<T, MODE>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return BM_ERR_CUDA;
    dim3 grid((unsigned)inner, (unsigned)outer);
    k<<<grid, 256, smem, s>>>(x, out, peak, n, inner);
  }
  return cuda_status();
}

static inline int grid_for(int64_t count) {
  int64_t b = (count + 255) / 256;
  const int64_t cap = 8LL * sm_count();
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace bm

using namespace bm;

extern "C" int bm_analytic_signal(int32_t dtype, const void* x, void* z, int64_t outer, int64_t n,
                                  int64_t inner, void* stream) {
  if (!x || !z || outer < 1 || inner < 1) return BM_ERR_INVALID_ARGUMENT;
  if (n < 2) return BM_ERR_AXIS_TOO_SHORT;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == BM_F32)
    return launch_analytic<float, kComplex>((const float*)x, (float*)z, nullptr, outer, n, inner, s);
  if (dtype == BM_F64)
    return launch_analytic<double, kComplex>((const double*)x, (double*)z, nullptr, outer, n, inner, s);
  return BM_ERR_INVALID_ARGUMENT;
}

extern "C" int bm_envelope(int32_t dtype, const void* z, void* e, int64_t count, void* stream) {
  if (!z || !e || count < 0) return BM_ERR_INVALID_ARGUMENT;
  if (count == 0) return BM_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == BM_F32)
    envelope_kernel<float><<<grid_for(count), 256, 0, s>>>((const float*)z, (float*)e, count);
  else if (dtype == BM_F64)
    envelope_kernel<double><<<grid_for(count), 256, 0, s>>>((const double*)z, (double*)e, count);
  else
    return BM_ERR_INVALID_ARGUMENT;
  return cuda_status();
}

extern "C" int bm_envelope_peak(int32_t dtype, const void* rf_img, void* env, void* peak,
                                int32_t n_frames, int64_t n_z, int64_t n_x, void* stream) {
  if (!rf_img || !env || !peak || n_frames < 1 || n_x < 1) return BM_ERR_INVALID_ARGUMENT;
  if (n_z < 2) return BM_ERR_AXIS_TOO_SHORT;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t pb = dtype == BM_F64 ? 8 : 4;
  if (cudaMemsetAsync(peak, 0, pb * n_frames, s) != cudaSuccess) return BM_ERR_CUDA;
  if (dtype == BM_F32)
    return launch_analytic<float, kEnvelope>((const float*)rf_img, (float*)env,
                                             (unsigned int*)peak, n_frames, n_z, n_x, s);
  if (dtype == BM_F64)
    return launch_analytic<double, kEnvelope>((const double*)rf_img, (double*)env,
                                              (unsigned long long*)peak, n_frames, n_z, n_x, s);
  return BM_ERR_INVALID_ARGUMENT;
}

extern "C" int bm_frame_peak(int32_t dtype, const void* e, void* peak, int32_t n_frames,
                             int64_t frame_elems, void* stream) {
  if (!e || !peak || n_frames < 1 || n_frames > 65535 || frame_elems < 0)
    return BM_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t pb = dtype == BM_F64 ? 8 : 4;
  if (cudaMemsetAsync(peak, 0, pb * n_frames, s) != cudaSuccess) return BM_ERR_CUDA;
  if (frame_elems == 0) return BM_OK;
  int gx = grid_for(frame_elems);
  if (gx > 2 * sm_count()) gx = 2 * sm_count();
  dim3 grid(gx, n_frames);
  if (dtype == BM_F32)
    peak_kernel<float><<<grid, 256, 0, s>>>((const float*)e, (unsigned int*)peak, frame_elems);
  else if (dtype == BM_F64)
    peak_kernel<double><<<grid, 256, 0, s>>>((const double*)e, (unsigned long long*)peak, frame_elems);
  else
    return BM_ERR_INVALID_ARGUMENT;
  return cuda_status();
}

extern "C" int bm_display(int32_t dtype, const void* e, const void* peak, void* disp,
                          int32_t* status, int32_t n_frames, int64_t frame_elems, double range_db,
                          void* stream) {
  if (!e || !peak || !disp || n_frames < 1 || n_frames > 65535 || frame_elems < 0)
    return BM_ERR_INVALID_ARGUMENT;
  if (!(range_db > 0) || range_db != range_db) return BM_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  int gx = grid_for(frame_elems);
  if (gx > 2 * sm_count()) gx = 2 * sm_count();
  dim3 grid(gx, n_frames);
  if (dtype == BM_F32)
    display_kernel<float><<<grid, 256, 0, s>>>((const float*)e, (const unsigned int*)peak,
                                              (float*)disp, status, frame_elems, range_db);
  else if (dtype == BM_F64)
    display_kernel<double><<<grid, 256, 0, s>>>((const double*)e, (const unsigned long long*)peak,
                                               (double*)disp, status, frame_elems, range_db);
  else
    return BM_ERR_INVALID_ARGUMENT;
  return cuda_status();
}

extern "C" int bm_dynamic_adjustment(int32_t dtype, const void* e, void* peak_ws, void* disp,
                                     int32_t* status, int32_t n_frames, int64_t frame_elems,
                                     double range_db, void* stream) {
  int rc = bm_frame_peak(dtype, e, peak_ws, n_frames, frame_elems, stream);
  if (rc) return rc;
  return bm_display(dtype, e, peak_ws, disp, status, n_frames, frame_elems, range_db, stream);
}

extern "C" const char* bm_error_string(int code) {
  switch (code) {
    case BM_OK: return "ok";
    case BM_ERR_INVALID_ARGUMENT: return "invalid argument";
    case BM_ERR_UNSUPPORTED: return "unsupported size for this build";
    case BM_ERR_CUDA: return "CUDA runtime error";
    case BM_ERR_AXIS_TOO_SHORT: return "analytic signal needs axis length >= 2";
    default: return "unknown error";
  }
}

extern "C" int bm_abi_version(void) { return BMODE200_ABI_VERSION; }

// Display -> 8-bit pixels for PGM output (formats.py:189-200):
// floor(v * 255 + 0.5) with each operator rounded in the display dtype, as
// numpy evaluates it (a weak python scalar keeps f32 arrays in f32).
namespace bm {
template <typename T>
__global__ void quantize_u8_kernel(const T* __restrict__ d, uint8_t* __restrict__ out, int64_t n) {
  using O = R<T>;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T s = O::add(O::mul(d[i], T(255)), T(0.5));
    out[i] = (uint8_t)floor(s);
  }
}

// f32 with 16-B aligned input and 4-B aligned output: four pixels per thread
// (one 16-B load, one 4-B store); the same per-pixel arithmetic.
__global__ void quantize_u8_f32x4_kernel(const float4* __restrict__ d, uchar4* __restrict__ out,
                                         int64_t n4) {
  using O = R<float>;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = d[i];
    uchar4 q;
    q.x = (uint8_t)floor(O::add(O::mul(v.x, 255.0f), 0.5f));
    q.y = (uint8_t)floor(O::add(O::mul(v.y, 255.0f), 0.5f));
    q.z = (uint8_t)floor(O::add(O::mul(v.z, 255.0f), 0.5f));
    q.w = (uint8_t)floor(O::add(O::mul(v.w, 255.0f), 0.5f));
    out[i] = q;
  }
}
}  // namespace bm

extern "C" int bm_quantize_u8(int32_t dtype, const void* disp, uint8_t* out, int64_t count,
                              void* stream) {
  if (!disp || !out || count < 0) return BM_ERR_INVALID_ARGUMENT;
  if (count == 0) return BM_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == BM_F32 && ((uintptr_t)disp & 15) == 0 && ((uintptr_t)out & 3) == 0) {
    const int64_t n4 = count / 4, tail = count - 4 * n4;
    if (n4)
      bm::quantize_u8_f32x4_kernel<<<grid_for(n4), 256, 0, s>>>((const float4*)disp, (uchar4*)out, n4);
    if (tail)
      bm::quantize_u8_kernel<float><<<1, 32, 0, s>>>((const float*)disp + 4 * n4, out + 4 * n4, tail);
  } else if (dtype == BM_F32)
    quantize_u8_kernel<float><<<grid_for(count), 256, 0, s>>>((const float*)disp, out, count);
  else if (dtype == BM_F64)
    quantize_u8_kernel<double><<<grid_for(count), 256, 0, s>>>((const double*)disp, out, count);
  else
    return BM_ERR_INVALID_ARGUMENT;
  return cuda_status();
}
