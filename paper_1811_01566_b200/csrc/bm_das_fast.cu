// K1 fast path: shared-memory-staged, packed-f32x2 Delay-and-Sum (sm_100a).
//
// Same arithmetic as das_kernel (bm_das.cu) and therefore the same bits as
// the reference's f32 das_beamform (beamform.py:122-187 with the DasPlan
// delays of :211-228) -- every operator is rounded once, in the reference's
// order -- but organised for the B200's shared-memory crossbar and its
// packed FP32 pipe:
//
//  * CTA = 64 threads, tile = 8 rows x 16 columns; each thread owns the pixel
//    pair (r, c) / (r + 4, c) and evaluates both with FADD2/FMUL2 (f32x2), so
//    one instruction advances two pixels.  A warp's 32 "A" pixels form a 4 x 8
//    block: for every (e, j) their sample indices fall in one 32-word span, so
//    each gather is a single conflict-free shared-memory wavefront (measured
//    by tests/bankmodel in DESIGN.md).
//  * Receive delays of the tile, D[m][pair] = fs*(sqrt(dx^2+z^2)/c) for every
//    element m, are built once per CTA in shared memory and reused for every
//    transmit and every frame of the CTA's frame group.
//  * RF is staged per chunk of JC channels: for each (e, j) only the window of
//    samples the tile can reach ([tmin-3, tmax+4], from the tile rectangle's
//    nearest / farthest geometry) is copied with cp.async (16 B per copy,
//    src-size 0 zero fill for groups outside the trace, which reproduces
//    x_pad's zero sentinels, beamform.py:127-137, :273-274), double buffered
//    against the computation of the previous chunk.  (A TMA bulk-copy
//    variant, one cp.async.bulk per channel on an mbarrier, measured slower:
//    per-lane bulk copies serialise into a UBLKCP loop.)
//  * floor(t) and the integer sample index come from one FADD2.RM with the
//    1.5*2^23 magic constant (exact for |t| < 2^22, checked on the host by
//    bm_das_prepare); the index is the float's bit pattern, so no F2I.
#include <algorithm>
#include <cmath>
#include <vector>

#include "bm_f32x2.cuh"

namespace bm {

constexpr int FZ = 8, FX = 16, FTHREADS = 64, JC = 16;
struct FastArgs {
  bm_das_geometry g;
  const float* rf;
  int64_t rf_stride;
  float* out;
  int64_t out_stride;
  int n_frames;
  int frames_per_cta;
  int W;  // staged window capacity per channel (samples, multiple of 4)
};

// Per-transmit staging metadata, one int2 per receive channel j:
//   x = staged length (samples, multiple of 4, <= W)
//       | element m's D row byte offset (m * 64 threads * 8 B) << 13
//         (IDMAP: the D row of channel j is row j, known at compile time),
//   y = K, the shared-memory byte address of sample 0 of the channel's
//       window minus 4 * (1.5*2^23 bits): x[k] lives at bits(floor(t)+M)*4 + K.
// Ring of 2 transmits: meta(T + 1) is written at the first chunk of T.
template <bool PW, bool LINEAR, bool T0, bool IDMAP>
__global__ void __launch_bounds__(FTHREADS, 3) das_fast_kernel(const FastArgs a) {
  using O = R<float>;
  const bm_das_geometry& g = a.g;
  const int n_el = g.n_elements, n_tx = g.n_tx, n_rx = g.n_rx, n_s = g.n_samples;
  const int W = a.W;

  // shared memory carve-up (byte offsets from the shared base, so every
  // access below stays an LDS/STS)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int off_tmin = n_el * FTHREADS * 8;
  const int off_meta = (off_tmin + 8 * n_tx + 15) & ~15;
  const int off_win = (off_meta + 16 * n_rx + 15) & ~15;
  u64* D = reinterpret_cast<u64*>(smem_raw);                   // [n_el][64] pairs
  float* tmin = reinterpret_cast<float*>(smem_raw + off_tmin);  // [n_tx]
  float* tmax = tmin + n_tx;                                    // [n_tx]
  int2* meta = reinterpret_cast<int2*>(smem_raw + off_meta);    // [2][n_rx]
  float* win = reinterpret_cast<float*>(smem_raw + off_win);    // [2][JC][W]

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int tiles_x = (g.n_x + FX - 1) / FX;
  const int tz0 = (blockIdx.x / tiles_x) * FZ, tx0 = (blockIdx.x % tiles_x) * FX;
  const int col = tx0 + warp * 8 + (lane & 7);
  const int rowA = tz0 + (lane >> 3), rowB = rowA + 4;
  const int colc = min(col, g.n_x - 1);
  const int rAc = min(rowA, g.n_z - 1), rBc = min(rowB, g.n_z - 1);

  const float c = O::from_double(g.speed_of_sound);
  const float fs = O::from_double(g.sampling_frequency);
  const double px = g.x_pos[colc];
  const float pxd = O::from_double(px);
  const float pzA = O::from_double(g.z_pos[rAc]), pzB = O::from_double(g.z_pos[rBc]);
  const uint32_t win_s = (uint32_t)__cvta_generic_to_shared(win);

  // ---- per-CTA geometry: exact receive delays of the pixel pair, window bounds
  for (int m = 0; m < n_el; ++m) {
    const float dx = O::from_double(g.elem_x[m] - px);
    const float dA = O::mul(fs, O::div(O::sqrt(O::add(O::mul(dx, dx), O::mul(pzA, pzA))), c));
    const float dB = O::mul(fs, O::div(O::sqrt(O::add(O::mul(dx, dx), O::mul(pzB, pzB))), c));
    D[(size_t)m * FTHREADS + tid] = pk(dA, dB);
  }
  const double x0 = g.x_pos[tx0], x1 = g.x_pos[min(tx0 + FX, g.n_x) - 1];
  const double z0 = g.z_pos[tz0], z1 = g.z_pos[min(tz0 + FZ, g.n_z) - 1];
  const double k = g.sampling_frequency / g.speed_of_sound;
  // receive-path delay bounds of element m over the tile rectangle: nearest
  // and farthest point, in samples
  auto rx_bounds = [&](int m, float& lo, float& hi) {
    const double xm = g.elem_x[m];
    const double dmin = fmax(0.0, fmax(x0 - xm, xm - x1));
    const double dmax = fmax(fabs(x0 - xm), fabs(x1 - xm));
    lo = (float)(k * sqrt(dmin * dmin + z0 * z0));
    hi = (float)(k * sqrt(dmax * dmax + z1 * z1));
  };
  for (int e = tid; e < n_tx; e += FTHREADS) {
    if (PW) {
      const double ca = reinterpret_cast<const float*>(g.cos_a)[e];
      const double sa = reinterpret_cast<const float*>(g.sin_a)[e];
      const double v00 = z0 * ca + x0 * sa, v01 = z0 * ca + x1 * sa;
      const double v10 = z1 * ca + x0 * sa, v11 = z1 * ca + x1 * sa;
      tmin[e] = (float)(k * fmin(fmin(v00, v01), fmin(v10, v11)));
      tmax[e] = (float)(k * fmax(fmax(v00, v01), fmax(v10, v11)));
    } else {
      rx_bounds(g.tx_elements[e], tmin[e], tmax[e]);
    }
  }
  __syncthreads();

  const float* __restrict__ t0s = reinterpret_cast<const float*>(g.t0_smp);
  const int n_chunks = (n_rx + JC - 1) / JC;
  const int f_begin = blockIdx.y * a.frames_per_cta;
  const int f_count = min(a.frames_per_cta, a.n_frames - f_begin);
  const int Q = f_count * n_tx * n_chunks;
  const int n_T = f_count * n_tx;

  // staging metadata of running transmit T (all channels, all threads).
  // Chunk q of transmit T is q = T * n_chunks + cb, so its window buffer
  // (q & 1) -- and with it K -- is known here.
  auto make_meta = [&](int T) {
    const int e = T % n_tx;  // once per transmit, not per chunk
    int2* M = meta + (T & 1) * n_rx;
    const float t0 = t0s[e];
    const float lo_e = tmin[e] - t0, hi_e = tmax[e] - t0;
    const int* map = g.rx_map + (int64_t)e * n_rx;
    for (int j = tid; j < n_rx; j += FTHREADS) {
      const int m = IDMAP ? j : map[j];
      float rlo, rhi;
      rx_bounds(m, rlo, rhi);
      const int ws = ((int)floorf(lo_e + rlo) - 3) & ~3;
      const int hi = (int)floorf(hi_e + rhi) + 4;
      const int len = min((hi - ws + 3) & ~3, W);  // host guarantees <= W
      const int cb = j / JC, jj = j - cb * JC;
      const int buf = (T * n_chunks + cb) & 1;
      const uint32_t K = win_s + (uint32_t)((buf * JC + jj) * W) * 4u -
                         (uint32_t)(kMagicBits + ws) * 4u;
      M[j] = make_int2(len | ((m * FTHREADS * 8) << 13), (int)K);
    }
  };
  // cp.async staging of chunk q: 4 threads per channel, 16 B per copy,
  // zero fill (src-size 0) for 16 B groups outside the trace.  Thread tid
  // always serves channel jj = tid / 4 of a chunk and copy slots
  // o = 4*(tid % 4) + 16*i, i < ceil(W / 16) <= 4 (host guarantees W <= 64
  // for this kernel), so the per-chunk work is a few adds.
  const int ld_jj = tid >> 2, ld_o = 4 * (tid & 3);
  const int64_t ld_trace = (int64_t)ld_jj * n_s + ld_o;
  auto issue_loads = [&](int q, const Cursor& cu) {
    const int j = cu.cb * JC + ld_jj;
    if (j >= n_rx) return;
    const int2 mm = meta[(cu.T & 1) * n_rx + j];
    const int len = mm.x & 0x1fff;
    const uint32_t wb = win_s + (uint32_t)(((q & 1) * JC + ld_jj) * W + ld_o) * 4u;
    // K = wb0 - 4*(M_bits + ws) mod 2^32, so (wb0 - K)/4 = (M_bits + ws) mod 2^30
    const int ws = (int)((wb - (uint32_t)ld_o * 4u - (uint32_t)mm.y) >> 2) -
                   (kMagicBits & 0x3fffffff);
    const float* tr = a.rf + (int64_t)(f_begin + cu.fl) * a.rf_stride +
                      ((int64_t)cu.e * n_rx + cu.cb * JC) * n_s + ld_trace;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int o = ld_o + 16 * i;
      if (o < len) {
        const int s0 = ws + o;
        const bool in = (unsigned)s0 <= (unsigned)(n_s - 4);
        cp_async16(wb + 64u * i, tr + (in ? ws + 16 * i : -ld_o), in ? 16 : 0);
      }
    }
  };

  Cursor cur{0, 0, 0, 0}, nxt{0, 0, 0, 0};
  make_meta(0);
  __syncthreads();
  issue_loads(0, nxt);
  cp_async_commit();
  nxt.next(n_chunks, n_tx);

  const u64 M2 = pk(kMagic, kMagic);
  const u64 NM2 = pk(-kMagic, -kMagic);
  const u64 ONE2 = pk(1.0f, 1.0f);
  const u64 HALF2 = pk(0.5f, 0.5f);
  u64 acc = 0ull;  // (+0.0f, +0.0f)
  u64 txd = 0ull, t0e2 = 0ull;
  const unsigned char* Dbytes = reinterpret_cast<const unsigned char*>(D) + tid * 8;

  for (int q = 0; q < Q; ++q) {
    __syncthreads();  // compute(q-1) done everywhere: buffer (q+1)&1 may be refilled
    if (cur.cb == 0 && cur.T + 1 < n_T) {
      make_meta(cur.T + 1);  // ring slot of transmit T-1: all its loads/computes are done
      __syncthreads();
    }
    if (q + 1 < Q) issue_loads(q + 1, nxt);
    cp_async_commit();
    nxt.next(n_chunks, n_tx);
    if (cur.cb == 0) {
      if (PW) {
        const float ca = reinterpret_cast<const float*>(g.cos_a)[cur.e];
        const float sa = reinterpret_cast<const float*>(g.sin_a)[cur.e];
        const float xs = O::mul(pxd, sa);
        const float tA = O::mul(fs, O::div(O::add(O::mul(pzA, ca), xs), c));
        const float tB = O::mul(fs, O::div(O::add(O::mul(pzB, ca), xs), c));
        txd = pk(tA, tB);
      } else {
        txd = D[(size_t)g.tx_elements[cur.e] * FTHREADS + tid];
      }
      const float t0 = t0s[cur.e];
      t0e2 = pk(t0, t0);
    }
    cp_async_wait1();
    __syncthreads();  // chunk q staged and visible

    const int2* M = meta + (cur.T & 1) * n_rx + cur.cb * JC;
    const int jn = min(JC, n_rx - cur.cb * JC);
    const unsigned char* Dchunk = Dbytes + cur.cb * JC * FTHREADS * 8;
    auto contrib = [&](int jj) {
      const int2 mm = M[jj];
      const uint32_t K = (uint32_t)mm.y;
      const u64 rxd = IDMAP ? *reinterpret_cast<const u64*>(Dchunk + jj * FTHREADS * 8)
                            : *reinterpret_cast<const u64*>(Dbytes + ((unsigned)mm.x >> 13));
      u64 t = add2(txd, rxd);
      if (T0) t = sub2(t, t0e2);  // all-zero t0 skips it: x - 0 == x exactly
      if (LINEAR) {
        const u64 r = add2_rm(t, M2);   // floor(t) + 1.5*2^23, exactly
        const u64 k0f = add2(r, NM2);   // floor(t)
        const u64 fr = sub2(t, k0f);    // a = t - floor(t)
        const u64 om = sub2(ONE2, fr);  // 1 - a
        float rA, rB;
        unpk(r, rA, rB);
        const uint32_t aA = (uint32_t)__float_as_int(rA) * 4u + K;
        const uint32_t aB = (uint32_t)__float_as_int(rB) * 4u + K;
        const u64 x0 = pk(lds0(aA), lds0(aB));
        const u64 x1 = pk(lds1(aA), lds1(aB));
        acc = add2(acc, mul2(om, x0));  // acc = out + (1 - a) * x[k0]
        acc = add2(acc, mul2(fr, x1));  // out = acc + a * x[k1]
      } else {
        const u64 r = add2_rm(add2(t, HALF2), M2);  // floor(t + 0.5)
        float rA, rB;
        unpk(r, rA, rB);
        const uint32_t aA = (uint32_t)__float_as_int(rA) * 4u + K;
        const uint32_t aB = (uint32_t)__float_as_int(rB) * 4u + K;
        acc = add2(acc, pk(lds0(aA), lds0(aB)));
      }
    };
    // Full chunks run in groups of G channels, each stage issued for the whole
    // group before the next (delays, then floors and gather addresses, then
    // the shared-memory gathers, then the arithmetic and the in-order
    // accumulation), so every warp keeps G independent gathers in flight.
    constexpr int G = 8;
    auto group = [&](int j0) {
      u64 t[G], r[G], x0[G], x1[G];
      uint32_t aA[G], aB[G];
#pragma unroll
      for (int i = 0; i < G; ++i) {
        const int2 mm = M[j0 + i];
        const u64 rxd = IDMAP ? *reinterpret_cast<const u64*>(Dchunk + (j0 + i) * FTHREADS * 8)
                              : *reinterpret_cast<const u64*>(Dbytes + ((unsigned)mm.x >> 13));
        t[i] = add2(txd, rxd);
        if (T0) t[i] = sub2(t[i], t0e2);
        r[i] = LINEAR ? add2_rm(t[i], M2) : add2_rm(add2(t[i], HALF2), M2);
        float rA, rB;
        unpk(r[i], rA, rB);
        aA[i] = (uint32_t)__float_as_int(rA) * 4u + (uint32_t)mm.y;
        aB[i] = (uint32_t)__float_as_int(rB) * 4u + (uint32_t)mm.y;
      }
#pragma unroll
      for (int i = 0; i < G; ++i) {
        x0[i] = pk(lds0(aA[i]), lds0(aB[i]));
        if (LINEAR) x1[i] = pk(lds1(aA[i]), lds1(aB[i]));
      }
#pragma unroll
      for (int i = 0; i < G; ++i) {
        if (LINEAR) {
          const u64 fr = sub2(t[i], add2(r[i], NM2));  // a = t - floor(t)
          const u64 om = sub2(ONE2, fr);               // 1 - a
          acc = add2(acc, mul2(om, x0[i]));            // acc = out + (1 - a) * x[k0]
          acc = add2(acc, mul2(fr, x1[i]));            // out = acc + a * x[k1]
        } else {
          acc = add2(acc, x0[i]);
        }
      }
    };
    if (jn == JC) {
#pragma unroll
      for (int j0 = 0; j0 < JC; j0 += G) group(j0);
    } else {
      for (int jj = 0; jj < jn; ++jj) contrib(jj);
    }

    if (cur.e == n_tx - 1 && cur.cb == n_chunks - 1) {  // frame complete
      const int64_t fo = (int64_t)(f_begin + cur.fl) * a.out_stride;
      if (col < g.n_x) {
        if (rowA < g.n_z) a.out[fo + (int64_t)rowA * g.n_x + col] = lo_f(acc);
        if (rowB < g.n_z) a.out[fo + (int64_t)rowB * g.n_x + col] = hi_f(acc);
      }
      acc = 0ull;
    }
    cur.next(n_chunks, n_tx);
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

size_t fast_smem_bytes(const bm_das_geometry& g, int W) {
  size_t b = (size_t)g.n_elements * FTHREADS * 8 + (size_t)g.n_tx * 8;
  b = ((b + 15) & ~size_t(15)) + (size_t)g.n_rx * 16;
  b = (b + 15) & ~size_t(15);
  return b + (size_t)2 * JC * W * 4;
}

int das_fast_eligible(const bm_das_geometry& g, int64_t rf_stride) {
  if (g.dtype != BM_F32 || !g.uniform || g.window_hint <= 0) return 0;
  if (g.n_samples % 4 != 0 || rf_stride % 4 != 0) return 0;
  if (fast_smem_bytes(g, g.window_hint) > 200 * 1024) return 0;
  if (g.n_elements > 512) return 0;  // meta packing: D offset in 19 bits
  if (g.window_hint > 128) return 0;  // loader: <= 8 copies of 16 B per thread
  return 1;
}

int das_fast_launch(const bm_das_geometry& g, const void* rf, int64_t rf_stride, void* out,
                    int64_t out_stride, int n_frames, cudaStream_t s) {
  FastArgs a{g, (const float*)rf, rf_stride, (float*)out, out_stride, n_frames, 1, g.window_hint};
  const int tiles = ((g.n_z + FZ - 1) / FZ) * ((g.n_x + FX - 1) / FX);
  // frames per CTA: amortise the per-CTA delay build over a frame group while
  // keeping >= ~8 waves of CTAs for load balance
  int fpc = 1;
  while (fpc < 8 && fpc * 2 <= n_frames && (int64_t)tiles * ((n_frames + fpc * 2 - 1) / (fpc * 2)) >=
                                               8LL * 3 * sm_count())
    fpc *= 2;
  a.frames_per_cta = fpc;
  const size_t smem = fast_smem_bytes(g, a.W);
  const bool pw = g.scheme == BM_PW, lin = g.interp == BM_LINEAR;
  typedef void (*kfn)(const FastArgs);
  // [pw][lin][t0][idmap]
  static const kfn table[16] = {
      das_fast_kernel<false, false, false, false>, das_fast_kernel<false, false, false, true>,
      das_fast_kernel<false, false, true, false>,  das_fast_kernel<false, false, true, true>,
      das_fast_kernel<false, true, false, false>,  das_fast_kernel<false, true, false, true>,
      das_fast_kernel<false, true, true, false>,   das_fast_kernel<false, true, true, true>,
      das_fast_kernel<true, false, false, false>,  das_fast_kernel<true, false, false, true>,
      das_fast_kernel<true, false, true, false>,   das_fast_kernel<true, false, true, true>,
      das_fast_kernel<true, true, false, false>,   das_fast_kernel<true, true, false, true>,
      das_fast_kernel<true, true, true, false>,    das_fast_kernel<true, true, true, true>};
  const kfn k = table[(pw ? 8 : 0) | (lin ? 4 : 0) | (g.t0_nonzero ? 2 : 0) |
                      (g.rx_identity ? 1 : 0)];
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return BM_ERR_CUDA;
  dim3 grid(tiles, (n_frames + fpc - 1) / fpc);
  k<<<grid, FTHREADS, smem, s>>>(a);
  return cuda_status();
}

}  // namespace bm

// Host-only: the largest window a 16 x 16 tile needs for 4 adjacent elements,
// evaluated per tile with the device's own bound arithmetic (das_tma_kernel:
// tmin/tmax of the transmit path, rmin/rmax of each element):
//   need <= max_e (tmax_e - tmin_e) + max_group (max rmax - min rmin) + 12
// where 12 covers the -3 / align-to-4 / +4 window margins and the float
// rounding of the device's sums and floors.  Returns 0 if the transmit
// geometry cannot be read back.
static int g4_window_bound(const bm_das_geometry* g, const double* elem_x, const double* x,
                           const double* z, int TZ = 16, int TX = 16) {
  const int n_el = g->n_elements, n_tx = g->n_tx;
  std::vector<float> ca(n_tx), sa(n_tx);
  std::vector<int> te(n_tx);
  const bool pw = g->scheme == BM_PW;
  if (pw) {
    const size_t es = g->dtype == BM_F64 ? 8 : 4;
    std::vector<unsigned char> bc(es * n_tx), bs(es * n_tx);
    if (!g->cos_a || !g->sin_a ||
        cudaMemcpy(bc.data(), g->cos_a, es * n_tx, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(bs.data(), g->sin_a, es * n_tx, cudaMemcpyDeviceToHost) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    for (int e = 0; e < n_tx; ++e) {
      ca[e] = es == 8 ? (float)reinterpret_cast<double*>(bc.data())[e]
                      : reinterpret_cast<float*>(bc.data())[e];
      sa[e] = es == 8 ? (float)reinterpret_cast<double*>(bs.data())[e]
                      : reinterpret_cast<float*>(bs.data())[e];
    }
  } else {
    if (!g->tx_elements ||
        cudaMemcpy(te.data(), g->tx_elements, sizeof(int) * n_tx, cudaMemcpyDeviceToHost) !=
            cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
  }
  const double k = g->sampling_frequency / g->speed_of_sound;
  const float kf = (float)k;
  std::vector<float> rmin(n_el), rmax(n_el);
  double need = 0.0;
  for (int tz0 = 0; tz0 < g->n_z; tz0 += TZ)
    for (int tx0 = 0; tx0 < g->n_x; tx0 += TX) {
      const double x0 = x[tx0], x1 = x[std::min(tx0 + TX, g->n_x) - 1];
      const double z0 = z[tz0], z1 = z[std::min(tz0 + TZ, g->n_z) - 1];
      const float x0f = (float)x0, x1f = (float)x1, z0f = (float)z0, z1f = (float)z1;
      for (int m = 0; m < n_el; ++m) {
        const float xm = (float)elem_x[m];
        const float dmin = std::max(0.0f, std::max(x0f - xm, xm - x1f));
        const float dmax = std::max(std::fabs(x0f - xm), std::fabs(x1f - xm));
        rmin[m] = kf * std::sqrt(dmin * dmin + z0f * z0f);
        rmax[m] = kf * std::sqrt(dmax * dmax + z1f * z1f);
      }
      double txr = 0.0;
      for (int e = 0; e < n_tx; ++e) {
        if (pw) {
          const double c = ca[e], s = sa[e];
          const double v00 = z0 * c + x0 * s, v01 = z0 * c + x1 * s;
          const double v10 = z1 * c + x0 * s, v11 = z1 * c + x1 * s;
          const float lo = (float)(k * std::min(std::min(v00, v01), std::min(v10, v11)));
          const float hi = (float)(k * std::max(std::max(v00, v01), std::max(v10, v11)));
          txr = std::max(txr, (double)hi - (double)lo);
        } else {
          const int m = te[e];
          if (m >= 0 && m < n_el) txr = std::max(txr, (double)rmax[m] - (double)rmin[m]);
        }
      }
      // groups of 4 consecutive elements: aligned for identity maps, every
      // start for the per-acquisition runs of a contiguous map
      const int gstep = g->rx_identity ? 4 : 1;
      double grp = 0.0;
      for (int m0 = 0; m0 < n_el; m0 += gstep) {
        float lo = rmin[m0], hi = rmax[m0];
        for (int m = m0 + 1; m < std::min(m0 + 4, n_el); ++m) {
          lo = std::min(lo, rmin[m]);
          hi = std::max(hi, rmax[m]);
        }
        grp = std::max(grp, (double)hi - (double)lo);
      }
      need = std::max(need, txr + grp);
    }
  const int w = (int)std::ceil(need) + 12;
  return (w + 7) & ~7;
}

// Host-only: bound the fast kernel's per-(e, j) sample window over all tiles.
extern "C" int bm_das_prepare(bm_das_geometry* g, const double* elem_x, const double* x,
                              const double* z, const double* t0_smp, const int32_t* rx_map) {
  if (!g || !elem_x || !x || !z || !t0_smp || !rx_map) return BM_ERR_INVALID_ARGUMENT;
  g->window_hint = 0;
  g->window_hint_wide = 0;
  g->window_hint_g4 = 0;
  g->t0_nonzero = 1;
  g->rx_identity = 0;
  g->rx_contig = 0;
  g->tile_ls = 3;
  if (g->n_z < 1 || g->n_x < 1 || g->n_elements < 1 || g->n_tx < 1) return BM_ERR_INVALID_ARGUMENT;
  // window bound of a tz x tx-pixel tile: tx delay range + rx delay range
  // (each <= k * tile diagonal) + margins
  const double k = g->sampling_frequency / g->speed_of_sound;
  auto bound = [&](int tz, int tx) {
    double zext = 0.0, xext = 0.0;
    for (int i = 0; i < g->n_z; i += tz) {
      const int l = (i + tz < g->n_z ? i + tz : g->n_z) - 1;
      zext = fmax(zext, z[l] - z[i]);
    }
    for (int i = 0; i < g->n_x; i += tx) {
      const int l = (i + tx < g->n_x ? i + tx : g->n_x) - 1;
      xext = fmax(xext, x[l] - x[i]);
    }
    const int w = (int)ceil(2.0 * k * sqrt(zext * zext + xext * xext) + 16.0);
    return (w + 3) & ~3;
  };
  int W = bound(16, 16);
  const int W_wide = bound(16, 24);
  // largest |t|: every delay is <= k * (farthest grid corner from any element
  // or from the origin) per path
  double dmax = 0.0;
  const double cx[2] = {x[0], x[g->n_x - 1]}, cz[2] = {z[0], z[g->n_z - 1]};
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      dmax = fmax(dmax, sqrt(cx[a] * cx[a] + cz[b] * cz[b]));
      for (int m = 0; m < g->n_elements; m += (g->n_elements > 1 ? g->n_elements - 1 : 1)) {
        const double dx = cx[a] - elem_x[m];
        dmax = fmax(dmax, sqrt(dx * dx + cz[b] * cz[b]));
      }
    }
  double t0max = 0.0;
  g->t0_nonzero = 0;
  for (int e = 0; e < g->n_tx; ++e) {
    t0max = fmax(t0max, fabs(t0_smp[e]));
    if (t0_smp[e] != 0.0) g->t0_nonzero = 1;
  }
  const double tabs = 2.0 * k * dmax + t0max + 16.0 + W;
  int ident = g->n_rx <= g->n_elements;
  for (int64_t i = 0; ident && i < (int64_t)g->n_tx * g->n_rx; ++i)
    if (rx_map[i] != (int)(i % g->n_rx)) ident = 0;
  g->rx_identity = ident;
  int contig = g->n_rx <= g->n_elements;
  for (int e = 0; contig && e < g->n_tx; ++e) {
    const int32_t* r = rx_map + (int64_t)e * g->n_rx;
    if (r[0] < 0 || r[0] + g->n_rx > g->n_elements) contig = 0;
    for (int j = 1; contig && j < g->n_rx; ++j)
      if (r[j] != r[0] + j) contig = 0;
  }
  g->rx_contig = contig;
  // 4 adjacent elements share one window (a 4-row TMA box): rx delays are
  // k-Lipschitz in the element position, so the union spans at most
  // W + k * (x[m+3] - x[m]); rounded to 8 samples (128-B aligned box rows)
  // and tightened by the per-tile evaluation where the geometry can be read.
  // Per TMA tile shape ls: lane blocks of (32 >> ls) x (1 << ls) pixels,
  // tiles of 4 (32 >> ls) x 2 (1 << ls).
  double ext = 0.0;
  for (int m = 0; m + 3 < g->n_elements; ++m) ext = fmax(ext, fabs(elem_x[m + 3] - elem_x[m]));
  auto g4_for = [&](int ls) {
    const int TZ = 4 * (32 >> ls), TX = 2 << ls;
    const int wg = ((int)ceil(bound(TZ, TX) + k * ext + 4.0) + 7) & ~7;
    const int exact = g4_window_bound(g, elem_x, x, z, TZ, TX);
    return exact > 0 && exact < wg ? exact : wg;
  };
  // contiguous maps pick the tile whose staged window is smallest; another
  // shape than 16 x 16 only for a >= 20 % smaller window (measured: sta-paper
  // 64 x 4 tiles W 96 vs 192, 0.77 -> 0.53 ms/frame; cfg1 8 x 32 W 128 vs 152
  // is 2 % slower)
  int ls = 3, wbest = g->n_elements >= 4 ? g4_for(3) : 0;
  if (contig && g->n_elements >= 4) {
    const char* e = getenv("BM_DAS_TILE");  // override: 1 (64 x 4) .. 4 (8 x 32)
    const int force = e ? atoi(e) : 0;
    if (force >= 1 && force <= 4) {
      ls = force;
      wbest = g4_for(ls);
    } else {
      for (int c : {1, 2, 4}) {
        const int w = g4_for(c);
        if (w * 5 <= wbest * 4 && w < wbest) {
          ls = c;
          wbest = w;
        }
      }
    }
  }
  g->tile_ls = ls;
  if (!(tabs - W + (wbest > W ? wbest : W) < 4194304.0)) return BM_OK;  // outside the exact magic-number range
  if (W_wide > 4096) return BM_OK;
  g->window_hint = W;
  g->window_hint_wide = W_wide;
  if (g->n_elements >= 4) g->window_hint_g4 = wbest;
  return BM_OK;
}
