// K1: Delay-and-Sum beamforming for STA and PW (sm_100a).
//
// Replaces echopipe's numba `_das_kernel` (beamform.py:122-187) together
// with the table build of `DasPlan.__init__` (beamform.py:204-236): instead of
// streaming [n_elements, n_px] delay LUTs from memory, each CTA rebuilds the
// receive delays of its pixel tile in shared memory with the reference's
// exact operation sequence
//     d_rx[m, p] = fs * (sqrt(dx*dx + z*z) / c),  dx = T(elem_x[m] - x)  (f64 -> T)
//     PW: tx[e, p] = fs * ((z*cos_e + x*sin_e) / c)
// and then accumulates, per pixel, in ascending e then ascending j:
//     t = (tx + d_rx[m]) - t0_e
//     nearest: out += [w *] x[clamp(floor(t + 0.5))]
//     linear : acc = out + ([w*](1 - a)) * x[k0];  out = acc + ([w*]a) * x[k1]
// with every operator individually rounded (no FMA).  The output is therefore
// bitwise identical to the reference's das_beamform in both f32 and f64.
//
// Thread mapping: one thread per pixel; a CTA owns a 4 x 32 (z x x) tile, a
// warp owns 32 adjacent lateral pixels of one row, so the gather addresses of
// a warp for one (e, j) trace fall within a narrow sample window.
#include <algorithm>

#include "bm_common.cuh"

namespace bm {

constexpr int kTileZ = 4;
constexpr int kTileX = 32;
constexpr int kThreads = kTileZ * kTileX;

struct DasArgs {
  bm_das_geometry g;
  const void* rf;
  int64_t rf_stride;
  void* out;
  int64_t out_stride;
  int e_begin, e_end;  // transmits of this launch
  int accumulate;      // continue the sums already in `out`
};

template <typename T>
__device__ __forceinline__ T rx_delay(const bm_das_geometry& g, int m, double px, T pzd, T c,
                                      T fs) {
  using O = R<T>;
  const T dx = O::from_double(g.elem_x[m] - px);
  const T s = O::add(O::mul(dx, dx), O::mul(pzd, pzd));
  return O::mul(fs, O::div(O::sqrt(s), c));
}

template <typename T>
__device__ __forceinline__ T load_or_zero(const T* __restrict__ x, int k, int n) {
  return (unsigned)k < (unsigned)n ? __ldg(x + k) : T(0);
}

// DSMEM: receive delays of the tile cached in shared memory ([n_el][kThreads],
// each thread owns one column, so no barrier is needed).  Without it (huge
// apertures) the delay is recomputed per contribution.
//
// TZ: tile rows (kTileZ by default).  The cached delay table costs
// n_elements * sizeof(T) bytes per pixel (1 KB for 128 f64 elements), so f64
// launches take TZ = 1 or 2: more, smaller CTAs per SM, more resident warps.
template <typename T, bool PW, bool LINEAR, bool UNIFORM, bool DSMEM, int TZ = kTileZ>
__global__ void __launch_bounds__(TZ * kTileX) das_kernel(const DasArgs a) {
  using O = R<T>;
  constexpr int kThreads = TZ * kTileX;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* D = reinterpret_cast<T*>(smem_raw);
  const bm_das_geometry& g = a.g;

  const int tid = threadIdx.x;
  const int tiles_x = (g.n_x + kTileX - 1) / kTileX;
  const int iz = (blockIdx.x / tiles_x) * TZ + tid / kTileX;
  const int ix = (blockIdx.x % tiles_x) * kTileX + tid % kTileX;
  const bool valid = iz < g.n_z && ix < g.n_x;
  const int izc = min(iz, g.n_z - 1), ixc = min(ix, g.n_x - 1);
  const int64_t p = (int64_t)izc * g.n_x + ixc;

  const T c = O::from_double(g.speed_of_sound);
  const T fs = O::from_double(g.sampling_frequency);
  const double px = g.x_pos[ixc];
  const T pzd = O::from_double(g.z_pos[izc]);
  const T pxd = O::from_double(px);
  const T one = T(1), half = T(0.5), lo = T(-1), hi = T(g.n_samples);
  const int n_s = g.n_samples;

  if (DSMEM) {
    for (int m = 0; m < g.n_elements; ++m) D[m * kThreads + tid] = rx_delay<T>(g, m, px, pzd, c, fs);
  }

  // receive apodisation (beamform.py:84-109): weight of element m is
  // window[m - i0] inside the active span [i0, i1], 0 outside.
  int i0 = 0, i1 = g.n_elements - 1;
  const T* hrow = nullptr;
  if (!UNIFORM) {
    if (g.span) {
      i0 = g.span[2 * p];
      i1 = g.span[2 * p + 1];
    }
    if (g.window == BM_HANN) {
      int cnt = i1 - i0 + 1;
      cnt = cnt < 0 ? 0 : (cnt > g.n_elements ? g.n_elements : cnt);
      hrow = reinterpret_cast<const T*>(g.hann) + (int64_t)cnt * g.n_elements;
    }
  }

  const T* __restrict__ rf = reinterpret_cast<const T*>(a.rf) + (int64_t)blockIdx.y * a.rf_stride;
  const T* __restrict__ t0s = reinterpret_cast<const T*>(g.t0_smp);
  T* __restrict__ outp = reinterpret_cast<T*>(a.out) + (int64_t)blockIdx.y * a.out_stride + p;
  T acc = a.accumulate && valid ? *outp : T(0);
  for (int e = a.e_begin; e < a.e_end; ++e) {
    T txd;
    if (PW) {
      const T ca = reinterpret_cast<const T*>(g.cos_a)[e];
      const T sa = reinterpret_cast<const T*>(g.sin_a)[e];
      txd = O::mul(fs, O::div(O::add(O::mul(pzd, ca), O::mul(pxd, sa)), c));
    } else {
      const int te = g.tx_elements[e];
      txd = DSMEM ? D[te * kThreads + tid] : rx_delay<T>(g, te, px, pzd, c, fs);
    }
    const T t0e = t0s[e];
    const int* __restrict__ map = g.rx_map + (int64_t)e * g.n_rx;
    const T* __restrict__ rfe = rf + (int64_t)e * g.n_rx * n_s;
#pragma unroll 4
    for (int j = 0; j < g.n_rx; ++j) {
      const int m = __ldg(map + j);
      const T rxd = DSMEM ? D[m * kThreads + tid] : rx_delay<T>(g, m, px, pzd, c, fs);
      const T t = O::sub(O::add(txd, rxd), t0e);
      const T* __restrict__ x = rfe + (int64_t)j * n_s;
      T w = one;
      if (!UNIFORM) {
        const bool act = m >= i0 && m <= i1;
        w = act ? (hrow ? hrow[m - i0] : one) : T(0);
      }
      if (!LINEAR) {
        T kf = O::floor(O::add(t, half));
        kf = kf < lo ? lo : (kf > hi ? hi : kf);
        const T v = load_or_zero(x, (int)kf, n_s);
        acc = UNIFORM ? O::add(acc, v) : O::add(acc, O::mul(w, v));
      } else {
        const T k0f = O::floor(t);
        const T fr = O::sub(t, k0f);
        T c0 = k0f < lo ? lo : (k0f > hi ? hi : k0f);
        T c1 = O::add(k0f, one);
        c1 = c1 < lo ? lo : (c1 > hi ? hi : c1);
        const T v0 = load_or_zero(x, (int)c0, n_s);
        const T v1 = load_or_zero(x, (int)c1, n_s);
        if (UNIFORM) {
          const T s0 = O::add(acc, O::mul(O::sub(one, fr), v0));
          acc = O::add(s0, O::mul(fr, v1));
        } else {
          const T s0 = O::add(acc, O::mul(O::mul(w, O::sub(one, fr)), v0));
          acc = O::add(s0, O::mul(O::mul(w, fr), v1));
        }
      }
    }
  }
  if (valid) *outp = acc;
}

// beamform.py:66-81, in f64: active iff |elem_x[m] - x| <= z / (2 F).
__global__ void span_kernel(const bm_das_geometry g, double f_number, int32_t* span) {
  const int64_t n_px = (int64_t)g.n_z * g.n_x;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n_px;
       p += (int64_t)gridDim.x * blockDim.x) {
    const double px = g.x_pos[p % g.n_x];
    const double pz = g.z_pos[p / g.n_x];
    const double half = __ddiv_rn(pz, 2.0 * f_number);
    int i0 = -1, i1 = -1;
    for (int m = 0; m < g.n_elements; ++m) {
      if (fabs(__dsub_rn(g.elem_x[m], px)) <= half) {
        if (i0 < 0) i0 = m;
        i1 = m;
      }
    }
    if (i0 < 0) {
      i0 = 0;
      i1 = -1;
    }
    span[2 * p] = i0;
    span[2 * p + 1] = i1;
  }
}

// stream-ordered hold for g.tx_ready launches of the generic kernel
__global__ void tx_wait_kernel(const uint32_t* ctr, uint32_t base, int need) {
  wait_tx_ready(ctr, base, need);
}

template <typename T, bool PW, bool LINEAR, bool UNIFORM, bool DSMEM, int TZ = kTileZ>
static int launch_t(const DasArgs& a, int n_frames, cudaStream_t s) {
  const bm_das_geometry& g = a.g;
  constexpr int kThreads = TZ * kTileX;
  const int tiles = ((g.n_z + TZ - 1) / TZ) * ((g.n_x + kTileX - 1) / kTileX);
  size_t smem = DSMEM ? (size_t)g.n_elements * kThreads * sizeof(T) : 0;
  auto k = das_kernel<T, PW, LINEAR, UNIFORM, DSMEM, TZ>;
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return BM_ERR_CUDA;
  }
  dim3 grid(tiles, n_frames);
  k<<<grid, kThreads, smem, s>>>(a);
  return cuda_status();
}

template <typename T, bool PW, bool LINEAR, bool UNIFORM>
static int launch_d(const DasArgs& a, int n_frames, cudaStream_t s) {
  const size_t per_px = (size_t)a.g.n_elements * sizeof(T);
  if (sizeof(T) == 8 && per_px * kTileX <= 200 * 1024) {
    // f64: the TZ (1 or 2 rows of 32 pixels) with the most resident warps
    // per SM for this table size (227 KB of shared memory per SM)
    const size_t cap = 227 * 1024;
    const size_t w1 = std::min<size_t>(cap / (per_px * kTileX + 1024), 32);
    const size_t w2 = 2 * std::min<size_t>(cap / (per_px * 2 * kTileX + 1024), 16);
    const int otz = debug_override(BM_DBG_DAS_GENERIC_TZ);  // A/B override: 1 | 2 | 4
    const int tz = otz ? otz : (w2 >= w1 ? 2 : 1);
    if (tz == 1) return launch_t<T, PW, LINEAR, UNIFORM, true, 1>(a, n_frames, s);
    if (tz == 2) return launch_t<T, PW, LINEAR, UNIFORM, true, 2>(a, n_frames, s);
  }
  const size_t smem = per_px * kThreads;
  if (smem <= 200 * 1024) return launch_t<T, PW, LINEAR, UNIFORM, true>(a, n_frames, s);
  return launch_t<T, PW, LINEAR, UNIFORM, false>(a, n_frames, s);
}

template <typename T, bool PW>
static int launch_p(const DasArgs& a, int n_frames, cudaStream_t s) {
  const bool lin = a.g.interp == BM_LINEAR, uni = a.g.uniform != 0;
  if (lin) return uni ? launch_d<T, PW, true, true>(a, n_frames, s)
                      : launch_d<T, PW, true, false>(a, n_frames, s);
  return uni ? launch_d<T, PW, false, true>(a, n_frames, s)
             : launch_d<T, PW, false, false>(a, n_frames, s);
}

static int check_geometry(const bm_das_geometry* g) {
  if (!g) return BM_ERR_INVALID_ARGUMENT;
  if (g->dtype != BM_F32 && g->dtype != BM_F64) return BM_ERR_INVALID_ARGUMENT;
  if (g->scheme != BM_STA && g->scheme != BM_PW) return BM_ERR_INVALID_ARGUMENT;
  if (g->interp != BM_NEAREST && g->interp != BM_LINEAR) return BM_ERR_INVALID_ARGUMENT;
  if (g->window != BM_RECTANGULAR && g->window != BM_HANN) return BM_ERR_INVALID_ARGUMENT;
  if (g->n_tx < 1 || g->n_rx < 1 || g->n_samples < 1 || g->n_elements < 1 || g->n_z < 1 ||
      g->n_x < 1)
    return BM_ERR_INVALID_ARGUMENT;
  if (!g->elem_x || !g->x_pos || !g->z_pos || !g->rx_map || !g->t0_smp)
    return BM_ERR_INVALID_ARGUMENT;
  if (g->scheme == BM_STA && !g->tx_elements) return BM_ERR_INVALID_ARGUMENT;
  if (g->scheme == BM_PW && (!g->cos_a || !g->sin_a)) return BM_ERR_INVALID_ARGUMENT;
  if (!g->uniform && g->window == BM_HANN && !g->hann) return BM_ERR_INVALID_ARGUMENT;
  return BM_OK;
}

}  // namespace bm

extern "C" int bm_das_aperture_span(const bm_das_geometry* g, double f_number,
                                    int32_t* span_out, void* stream) {
  int rc = bm::check_geometry(g);
  if (rc) return rc;
  if (!span_out || !(f_number > 0.0)) return BM_ERR_INVALID_ARGUMENT;
  const int64_t n_px = (int64_t)g->n_z * g->n_x;
  int blocks = (int)((n_px + 255) / 256);
  if (blocks > 4 * bm::sm_count()) blocks = 4 * bm::sm_count();
  bm::span_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(*g, f_number, span_out);
  return bm::cuda_status();
}

extern "C" int bm_das_select(const bm_das_geometry* g, int64_t rf_frame_stride) {
  if (bm::check_geometry(g)) return -1;
  const int choice = bm::das_kernel_choice();
  if (choice == 0 && bm::das_tma_eligible(*g, rf_frame_stride)) return 5;
  if (choice == 0 && bm::das_tma64_eligible(*g, rf_frame_stride)) return 6;
  return 0;
}

extern "C" int bm_das_launch_shape(const bm_das_geometry* g, int64_t rf_frame_stride,
                                   int32_t n_frames, int32_t* shape) {
  if (!shape || bm::check_geometry(g)) return -1;
  const int choice = bm::das_kernel_choice();
  if (choice == 0 && bm::das_tma_eligible(*g, rf_frame_stride))
    return bm::das_tma_shape(*g, n_frames, shape);
  if (choice == 0 && bm::das_tma64_eligible(*g, rf_frame_stride))
    return bm::das_tma64_shape(*g, n_frames, shape);
  return -1;
}

extern "C" int bm_das_beamform_range(const bm_das_geometry* g, const void* rf,
                                     int64_t rf_frame_stride, void* out, int64_t out_frame_stride,
                                     int32_t n_frames, int32_t e_begin, int32_t e_end,
                                     int32_t accumulate, void* stream) {
  int rc = bm::check_geometry(g);
  if (rc) return rc;
  if (!rf || !out || n_frames < 0 || n_frames > 65535) return BM_ERR_INVALID_ARGUMENT;
  if (e_begin < 0 || e_end > g->n_tx || e_begin >= e_end) return BM_ERR_INVALID_ARGUMENT;
  if (n_frames == 0) return BM_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int choice = bm::das_kernel_choice();
  if (choice == 0 && bm::das_tma_eligible(*g, rf_frame_stride)) {
    rc = bm::das_tma_launch(*g, rf, rf_frame_stride, out, out_frame_stride, n_frames, e_begin,
                            e_end, accumulate, s);
    if (rc >= 0) return rc;  // -1: unaligned RF pointer etc. -> generic kernel
  }
  if (choice == 0 && bm::das_tma64_eligible(*g, rf_frame_stride)) {
    rc = bm::das_tma64_launch(*g, rf, rf_frame_stride, out, out_frame_stride, n_frames, e_begin,
                              e_end, accumulate, s);
    if (rc >= 0) return rc;
  }
  if (g->tx_ready) {
    // the generic kernel reads every transmit of the range from its first
    // CTA on: a one-warp kernel ahead of it on the stream holds it until the
    // copy side's counter covers the range (a wait inside the kernel body --
    // a barrier after one thread's spin -- cost the f64 nearest kernel 2x)
    bm::tx_wait_kernel<<<1, 32, 0, s>>>(g->tx_ready, g->tx_ready_base, e_end);
    if ((rc = bm::cuda_status()) != BM_OK) return rc;
  }
  bm::DasArgs a{*g, rf, rf_frame_stride, out, out_frame_stride, e_begin, e_end, accumulate};
  if (g->dtype == BM_F32)
    return g->scheme == BM_PW ? bm::launch_p<float, true>(a, n_frames, s)
                              : bm::launch_p<float, false>(a, n_frames, s);
  return g->scheme == BM_PW ? bm::launch_p<double, true>(a, n_frames, s)
                            : bm::launch_p<double, false>(a, n_frames, s);
}

extern "C" int bm_das_beamform(const bm_das_geometry* g, const void* rf, int64_t rf_frame_stride,
                               void* out, int64_t out_frame_stride, int32_t n_frames,
                               void* stream) {
  if (!g) return BM_ERR_INVALID_ARGUMENT;
  return bm_das_beamform_range(g, rf, rf_frame_stride, out, out_frame_stride, n_frames, 0,
                               g->n_tx, 0, stream);
}

// Copy n_traces traces of n_samples samples (row pitch src_pitch) into rows of
// dst_samples >= n_samples, zero-filling the tail: the TMA kernel's 16-B row
// pitch for trace lengths that are not a multiple of 4 f32 samples.  The
// padding reads as the zeros the reference's out-of-range sentinels stand
// for (beamform.py:127-137), so the result is unchanged.  Two DMA operations,
// no kernel.
extern "C" int bm_pad_traces(int32_t dtype, const void* src, int64_t src_pitch, int64_t n_traces,
                             int64_t n_samples, void* dst, int64_t dst_samples, void* stream) {
  if (!src || !dst || n_traces < 0 || n_samples < 1 || dst_samples < n_samples ||
      src_pitch < n_samples || (dtype != BM_F32 && dtype != BM_F64))
    return BM_ERR_INVALID_ARGUMENT;
  if (n_traces == 0) return BM_OK;
  const size_t eb = dtype == BM_F64 ? 8 : 4;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpy2DAsync(dst, dst_samples * eb, src, src_pitch * eb, n_samples * eb, n_traces,
                        cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return BM_ERR_CUDA;
  if (dst_samples > n_samples &&
      cudaMemset2DAsync((char*)dst + n_samples * eb, dst_samples * eb, 0,
                        (dst_samples - n_samples) * eb, n_traces, s) != cudaSuccess)
    return BM_ERR_CUDA;
  return BM_OK;
}
