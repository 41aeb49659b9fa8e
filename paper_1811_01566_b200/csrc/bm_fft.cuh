// FFT building blocks of K2 (analytic signal, sigproc.py:48-73), sm_100a.
//
// Mixed-radix Cooley-Tukey for any length whose prime factors are <= 61:
//   * forward: decimation in frequency, natural order in, "digit-reversed"
//     order out (bin k of n = r0 r1 ... r_{m-1}, k = d0 + r0 (d1 + r1 (...)),
//     lands at position sum_i d_i * n / (r0 ... r_i));
//   * inverse: decimation in time over the reversed radix sequence, which
//     consumes exactly that order and returns natural order.
// The one-sided gain of the analytic signal is applied in between, at the
// scrambled positions (unscramble() recovers k), so no permutation pass is
// ever needed and every stage works in place: each butterfly reads and
// writes the same R elements.  Radix 8 / 4 / 2 butterflies are specialised;
// odd radices use a direct DFT with the n-point twiddle table.
//
// Twiddles W_n^e = exp(-2 pi i e / n) come from a two-level table,
// W_n^e = hi[e >> sh] * lo[e & (2^sh - 1)], both halves evaluated with f64
// sincospi and rounded once to T.
#pragma once
#include "bm_common.cuh"

namespace bm {

template <typename T> struct C2;
template <> struct C2<float> { using type = float2; };
template <> struct C2<double> { using type = double2; };

template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return {a.x + b.x, a.y + b.y}; }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return {a.x - b.x, a.y - b.y}; }
template <typename V> __device__ __forceinline__ V cmul(V a, V w) {
  return {a.x * w.x - a.y * w.y, a.x * w.y + a.y * w.x};
}
template <typename V> __device__ __forceinline__ V cconj(V a) { return {a.x, -a.y}; }
// multiply by SIGN * i  (forward transforms use SIGN = -1)
template <int SIGN, typename V> __device__ __forceinline__ V rot(V a) {
  return SIGN < 0 ? V{a.y, -a.x} : V{-a.y, a.x};
}

constexpr int kMaxFactors = 24;
constexpr int kMaxRadix = 61;

// Radix sequence of one length (host-built, passed by value).
struct FftPlan {
  int32_t n;
  int32_t m;                      // number of factors; 0 = not smooth
  int32_t pow2;                   // n is a power of two (every radix is 2, 4 or 8)
  int32_t tw_shift;               // two-level twiddle split
  int32_t radix[kMaxFactors];     // DIF order (radix[0] spans the whole lane)
};

inline FftPlan make_plan(int64_t n) {
  FftPlan p{};
  p.n = (int32_t)n;
  int64_t r = n, twos = 0;
  while (r % 2 == 0) { r /= 2; ++twos; }
  p.pow2 = r == 1;
  int m = 0;
  while (twos >= 3 && m < kMaxFactors) { p.radix[m++] = 8; twos -= 3; }
  if (twos == 2 && m < kMaxFactors) p.radix[m++] = 4;
  if (twos == 1 && m < kMaxFactors) p.radix[m++] = 2;
  for (int q = 3; q <= kMaxRadix && r > 1; q += 2)
    while (r % q == 0 && m < kMaxFactors) { p.radix[m++] = q; r /= q; }
  p.m = r == 1 ? m : 0;
  int sh = 0;
  while (((int64_t)1 << (2 * sh)) < n) ++sh;
  p.tw_shift = sh;
  return p;
}

template <typename T>
struct Twiddle {
  using V = typename C2<T>::type;
  const V* hi;
  const V* lo;
  int sh, mask;
  __device__ __forceinline__ V operator()(int e) const {
    return cmul(hi[e >> sh], lo[e & mask]);
  }
};

// W_n^e evaluated directly (global-memory passes; rare lengths)
template <typename T>
struct TwiddleDirect {
  using V = typename C2<T>::type;
  int n;
  __device__ __forceinline__ V operator()(int e) const {
    double s, c;
    sincospi(-2.0 * (double)e / (double)n, &s, &c);
    return {(T)c, (T)s};
  }
};

// Fill the two tables of W_n^e in shared memory (cooperatively).
template <typename T>
__device__ void twiddle_tables(typename C2<T>::type* hi, typename C2<T>::type* lo, int n, int sh,
                               int tid, int nthr) {
  const int nlo = 1 << sh, nhi = (n + nlo - 1) >> sh;
  for (int j = tid; j < nlo + nhi; j += nthr) {
    const int e = j < nlo ? j : (j - nlo) << sh;
    double s, c;
    sincospi(-2.0 * (double)e / (double)n, &s, &c);
    (j < nlo ? lo[j] : hi[j - nlo]) = {(T)c, (T)s};
  }
}

// ---- butterflies on registers (natural order in and out) --------------------
template <int SIGN, typename V>
__device__ __forceinline__ void dft2(V& a, V& b) {
  const V t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <int SIGN, typename V>
__device__ __forceinline__ void dft4(V& v0, V& v1, V& v2, V& v3) {
  const V t0 = cadd(v0, v2), t1 = csub(v0, v2), t2 = cadd(v1, v3), t3 = rot<SIGN>(csub(v1, v3));
  v0 = cadd(t0, t2);
  v1 = cadd(t1, t3);
  v2 = csub(t0, t2);
  v3 = csub(t1, t3);
}

template <int SIGN, typename V>
__device__ __forceinline__ void dft8(V* v) {
  using T = decltype(v[0].x);
  const T h = (T)0.70710678118654752440;
  dft4<SIGN>(v[0], v[2], v[4], v[6]);
  dft4<SIGN>(v[1], v[3], v[5], v[7]);
  // odd half times W8^k, k = 0..3 (W8 = exp(SIGN 2 pi i / 8))
  const V o1 = {h * (v[3].x + rot<SIGN>(v[3]).x), h * (v[3].y + rot<SIGN>(v[3]).y)};
  const V o2 = rot<SIGN>(v[5]);
  const V o3 = {h * (rot<SIGN>(v[7]).x - v[7].x), h * (rot<SIGN>(v[7]).y - v[7].y)};
  const V e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6], o0 = v[1];
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, o1);
  v[5] = csub(e1, o1);
  v[2] = cadd(e2, o2);
  v[6] = csub(e2, o2);
  v[3] = cadd(e3, o3);
  v[7] = csub(e3, o3);
}

template <int R, int SIGN, typename V>
__device__ __forceinline__ void dft_pow2(V* v) {
  if constexpr (R == 2) dft2<SIGN>(v[0], v[1]);
  if constexpr (R == 4) dft4<SIGN>(v[0], v[1], v[2], v[3]);
  if constexpr (R == 8) dft8<SIGN>(v);
}

// ---- one butterfly of a stage, elements at base[r * stride] -----------------
// DIF: y = DFT_R(x); out[q] = y[q] * W_n^(q * e1)
template <int R, typename T, typename P, typename TW>
__device__ __forceinline__ void dif_bfly(P base, int64_t stride, int e1, const TW& tw) {
  using V = typename C2<T>::type;
  V v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = base[r * stride];
  dft_pow2<R, -1>(v);
  base[0] = v[0];
#pragma unroll
  for (int q = 1; q < R; ++q) base[q * stride] = e1 ? cmul(v[q], tw(q * e1)) : v[q];
}

// DIT (inverse): x[r] *= conj(W_n^(r * e1)); out = IDFT_R(x) (unnormalised)
template <int R, typename T, typename P, typename TW>
__device__ __forceinline__ void dit_bfly(P base, int64_t stride, int e1, const TW& tw) {
  using V = typename C2<T>::type;
  V v[R];
  v[0] = base[0];
#pragma unroll
  for (int r = 1; r < R; ++r) {
    const V a = base[r * stride];
    v[r] = e1 ? cmul(a, cconj(tw(r * e1))) : a;
  }
  dft_pow2<R, +1>(v);
#pragma unroll
  for (int q = 0; q < R; ++q) base[q * stride] = v[q];
}

// Odd radix R <= kMaxRadix: direct DFT with W_R^j = W_n^(j n / R).
template <int SIGN, typename T, typename P, typename TW>
__device__ void generic_bfly(P base, int64_t stride, int R, int n, int e1, const TW& tw) {
  using V = typename C2<T>::type;
  V v[kMaxRadix];
  const int step = n / R;
  for (int r = 0; r < R; ++r) {
    V a = base[r * stride];
    if (SIGN > 0 && r && e1) a = cmul(a, cconj(tw(r * e1)));
    v[r] = a;
  }
  for (int q = 0; q < R; ++q) {
    V acc = v[0];
    int j = 0;
    for (int r = 1; r < R; ++r) {
      j += q;
      if (j >= R) j -= R;
      const V w = j ? tw(j * step) : V{(T)1, (T)0};
      acc = cadd(acc, cmul(v[r], SIGN < 0 ? w : cconj(w)));
    }
    if (SIGN < 0 && q && e1) acc = cmul(acc, tw(q * e1));
    base[q * stride] = acc;
  }
}

// Bin index k of the element at scrambled position pos (see header).
__device__ __forceinline__ int unscramble(const FftPlan& p, int pos) {
  int rem = p.n, k = 0, mul = 1;
  for (int i = 0; i < p.m; ++i) {
    rem /= p.radix[i];
    const int d = pos / rem;
    pos -= d * rem;
    k += d * mul;
    mul *= p.radix[i];
  }
  return k;
}

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

// Split a flat index into (lane, butterfly) with nb butterflies per lane.
__device__ __forceinline__ void split_idx(int idx, int nb, int nb_log2, int& l, int& b) {
  if (nb_log2 >= 0) {
    l = idx >> nb_log2;
    b = idx & ((1 << nb_log2) - 1);
  } else {
    l = idx / nb;
    b = idx - l * nb;
  }
}

__device__ __forceinline__ int ilog2_exact(int v) {  // log2 if v is a power of two, else -1
  return (v & (v - 1)) == 0 ? __ffs(v) - 1 : -1;
}

// Forward DIF over nl lanes of a shared-memory buffer (lane l at buf + l*lstride).
template <typename T>
__device__ void lane_dif(typename C2<T>::type* buf, int lstride, int nl, const FftPlan& p,
                         const Twiddle<T>& tw, int tid, int nthr) {
  int span = p.n;
  for (int s = 0; s < p.m; ++s) {
    const int R = p.radix[s], sub = span / R, nb = p.n / R, tstep = p.n / span;
    const int nbl = ilog2_exact(nb), subl = ilog2_exact(sub);
    for (int idx = tid; idx < nb * nl; idx += nthr) {
      int l, b;
      split_idx(idx, nb, nbl, l, b);
      const int g = subl >= 0 ? b >> subl : b / sub, k = b - g * sub;
      auto* base = buf + l * lstride + g * span + k;
      const int e1 = k * tstep;
      if (R == 8) dif_bfly<8, T>(base, sub, e1, tw);
      else if (R == 4) dif_bfly<4, T>(base, sub, e1, tw);
      else if (R == 2) dif_bfly<2, T>(base, sub, e1, tw);
      else generic_bfly<-1, T>(base, sub, R, p.n, e1, tw);
    }
    __syncthreads();
    span = sub;
  }
}

// Inverse DIT over the reversed radix sequence (scrambled in, natural out, x n).
template <typename T>
__device__ void lane_dit(typename C2<T>::type* buf, int lstride, int nl, const FftPlan& p,
                         const Twiddle<T>& tw, int tid, int nthr) {
  int span = 1;
  for (int s = p.m - 1; s >= 0; --s) {
    const int R = p.radix[s], ns = span * R, nb = p.n / R, tstep = p.n / ns;
    const int nbl = ilog2_exact(nb), spl = ilog2_exact(span);
    for (int idx = tid; idx < nb * nl; idx += nthr) {
      int l, b;
      split_idx(idx, nb, nbl, l, b);
      const int g = spl >= 0 ? b >> spl : b / span, k = b - g * span;
      auto* base = buf + l * lstride + g * ns + k;
      const int e1 = k * tstep;
      if (R == 8) dit_bfly<8, T>(base, span, e1, tw);
      else if (R == 4) dit_bfly<4, T>(base, span, e1, tw);
      else if (R == 2) dit_bfly<2, T>(base, span, e1, tw);
      else generic_bfly<+1, T>(base, span, R, p.n, e1, tw);
    }
    __syncthreads();
    span = ns;
  }
}

}  // namespace bm
