// K1, warp-specialised: TMA-fed RF windows, receive delays in TENSOR MEMORY.
//
// Same arithmetic -- and therefore the same bits -- as the generic kernel
// (bm_das.cu) and the reference's f32 das_beamform (beamform.py:122-187 with
// the DasPlan delays of :211-228).  What changes is who moves the data (the
// round-1 predecessor, where every warp issued its share of cp.async window
// copies and met the others at one __syncthreads per chunk, spent ~35 % of its
// warp samples outside the gather loop, profiles/r01_das_tmem_ncu.txt):
//
//  * a PRODUCER warp owns all of it: per stage of TJC receive channels
//    it computes each 4-channel group's window start, publishes the gather
//    bases K, and issues one cp.async.bulk.tensor (TMA) box {W samples, 4
//    traces, frames of the pass} per group (one trace per box for general
//    receive maps).  TMA's out-of-bounds fill writes exact zeros for samples
//    outside [0, n_s) -- the reference's sentinel semantics
//    (beamform.py:127-137) without a slow path.  The CONSUMER warps (4 x FP)
//    only wait on the stage's full barrier, gather and interpolate, and
//    release the stage through its empty barrier: no CTA-wide barrier in the
//    loop.
//
// Tile and lane layout: 2 x 2 warp blocks per CTA; thread (warp w, lane l)
// owns pixels A (row l >> ls, col l & (2^ls - 1) of its block) and B (A +
// 32 >> ls rows), ls = 3 giving 16 x 16 tiles of 8 x 8 blocks (tile_ls picks
// 32 x 8, 64 x 4 or 8 x 32 for other grids).  TMEM lane 32 (w & 3) + l holds
// the pair's delays to element m in columns 2m, 2m+1.
// Several frames per pass (FP warp groups x FT frames per thread) share the
// table and the frame-independent work; see the kernel's comment.
#include <cuda.h>  // CUtensorMap
#include <algorithm>
#include <type_traits>
#include <stdio.h>

#include "bm_tma.cuh"

namespace bm {

constexpr int kTmaMaxStages = 8;

struct TmaArgs {
  bm_das_geometry g;
  float* out;
  int64_t out_stride;
  int n_frames;
  int e_begin, e_end;  // transmits of this launch (the whole scheme by default)
  int accumulate;      // 1: continue the sums already in `out` (a later transmit range)
  int frames_per_cta;
  int W;          // samples per channel window (multiple of 32: 128-B aligned rows)
  int nst;        // pipeline stages (2 .. kTmaMaxStages)
  int tmem_cols;  // allocated TMEM columns (power of two >= 2 * n_elements)
  int ls;         // tile shape: lane blocks of (32 >> ls) x (1 << ls) pixels
  int prefetch;   // with a plan delay table: tiles ahead whose table to prefetch into L2
  int early_producer;  // 1: the RF pipeline fills while the consumers build their delays
};

// shared-memory carve (bytes), identical on host and device
struct TmaLayout {
  int tmin, rmin, metaK, metaM, txd, win, total;
  __host__ __device__ TmaLayout(int n_tx, int n_el, int tjc, int nst, int W, bool pw, int fp) {
    tmin = 256;  // [0,16) TMEM base, [16,24) active element span, [64,128) full
                 // barriers, [128,192) empty barriers
    rmin = (tmin + 28 * n_tx + 15) & ~15;
    metaK = (rmin + 8 * n_el + 15) & ~15;
    metaM = metaK + 4 * tjc * nst * fp;
    txd = metaM + 4 * tjc * nst;
    win = (txd + (pw ? n_tx * 128 * 8 : 0) + 127) & ~127;
    total = win + nst * tjc * fp * W * 4;
  }
};

// exact receive delays fs*(sqrt(dx*dx + z*z)/c) of element m for a pixel
// pair at (px, pzA) / (px, pzB), dx = T(elem_x - px) (beamform.py:211-216)
__device__ __forceinline__ float2 rx_delay_pair(const bm_das_geometry& g, int m, double px,
                                                float pzA, float pzB, float c, float fs) {
  using O = R<float>;
  const float dx = O::from_double(g.elem_x[m] - px);
  const float dA = O::mul(fs, O::div(O::sqrt(O::add(O::mul(dx, dx), O::mul(pzA, pzA))), c));
  const float dB = O::mul(fs, O::div(O::sqrt(O::add(O::mul(dx, dx), O::mul(pzB, pzB))), c));
  return make_float2(dA, dB);
}

// bm_das_build_table: table[tile][m][ctid] = delays of the thread's pair
__global__ void __launch_bounds__(128) das_table_kernel(const bm_das_geometry g, int ls,
                                                        float2* __restrict__ table) {
  using O = R<float>;
  const PairPos pp(g, ls, blockIdx.x, threadIdx.x);
  const int colc = min(pp.col, g.n_x - 1);
  const int rAc = min(pp.rowA, g.n_z - 1), rBc = min(pp.rowB, g.n_z - 1);
  const float c = O::from_double(g.speed_of_sound);
  const float fs = O::from_double(g.sampling_frequency);
  const double px = g.x_pos[colc];
  const float pzA = O::from_double(g.z_pos[rAc]), pzB = O::from_double(g.z_pos[rBc]);
  float2* tb = table + (int64_t)blockIdx.x * g.n_elements * 128 + threadIdx.x;
  for (int m = blockIdx.y; m < g.n_elements; m += gridDim.y)
    tb[(int64_t)m * 128] = rx_delay_pair(g, m, px, pzA, pzB, c, fs);
}

// WT: non-uniform receive apodisation (Hann and/or F-number gate): a
// contribution is acc + (w*(1-a))*x0 + (w*a)*x1 exactly as beamform.py:175-187
// rounds it, with the weight w[m] of each pixel formed in registers per
// 4-channel group -- the Hann element row (no F-number: the same row for
// every pixel), 1 / 0 from the pixel's active span (rectangular +
// F-number), or the span's Hann row, both rows read through L1 -- so the
// delay table alone fills TMEM (2 columns per element) and two CTAs share an
// SM.
//
// FP = 2: two frames per pass.  Consumer warps w and w + 4 own the same pixel
// pairs (the same TMEM lane quarter, so they share one delay table) but
// accumulate different frames; each TMA box carries both frames' windows
// ({W, G, 2}).  Twice the warps per SM for the same TMEM, so twice the
// independent instruction streams to hide the FP32 / shared-memory latencies.
//
// FT = 2: two frames per THREAD.  The delay t, the sample index, a and 1 - a
// of a (pixel, channel) do not depend on the frame, so a thread that
// accumulates two frames computes them once: 13 FP32 instructions per pixel
// pair, channel and two frames instead of 18, and the per-frame gathers of
// the second frame reuse the first frame's addresses plus the frame-plane
// offset of the staged box.  A pass then covers FP * FT frames (box
// {W, G, FP * FT}); each accumulator keeps the reference's e -> j order.
// WM (weighted kernels): the weight mode fixed at compile time -- 1 rectangular
// with an F-number gate, 2 Hann without, 3 Hann with (reading g.weight_pad)
// -- or 0, read from the geometry at run time
template <bool PW, bool LINEAR, bool T0, bool IDMAP, int TJC, bool WT = false, int FP = 1,
          int FT = 1, int WI = 0, int WM = 0>
__global__ void __launch_bounds__(32 * (4 * FP + 1), 2)
    das_tma_kernel(const __grid_constant__ CUtensorMap rf_map, const TmaArgs a) {
  using O = R<float>;
  using L = Lane<true>;
  typedef u64 VT;
  constexpr int NTH = 32 * (4 * FP + 1), NC = 128;  // threads, pixel-pair threads
  constexpr int NCW = 4 * FP;                        // consumer warps
  constexpr int FPP = FP * FT;                       // frames per pass
  // tile = 2 x 2 warp blocks; a warp block = pixel rows A (lane / CA) and B
  // (A + RA) of a RA x CA lane block (ls = 3: 16 x 16 tiles of 8 x 8 blocks)
  const int CA = 1 << a.ls, RA = 32 >> a.ls;
  const int TZk = 4 * RA, TXk = 2 * CA;
  constexpr int G = IDMAP ? 4 : 1;  // receive channels per TMA box (rows of W samples)
  const bm_das_geometry& g = a.g;
  const int n_el = g.n_elements, n_tx = g.n_tx, n_rx = g.n_rx;
  // WI > 0: the window width is a compile-time constant, so the frame-plane
  // offsets of frames 1..FT-1 become LDS immediates (no address adds)
  const int W = WI > 0 ? WI : a.W, nst = a.nst;
  const TmaLayout lay(n_tx, n_el, TJC, nst, W, PW, FPP);

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw);
  const uint32_t smem_s = (uint32_t)__cvta_generic_to_shared(smem_raw);
  const uint32_t full_s = smem_s + 64, empty_s = smem_s + 128;  // + 8 * stage
  float* tmin = reinterpret_cast<float*>(smem_raw + lay.tmin);  // [n_tx]
  float* tmax = tmin + n_tx;                                    // [n_tx]
  float* t0v = tmax + n_tx;                                     // [n_tx] fs*t0
  int* txe = reinterpret_cast<int*>(t0v + n_tx);                // [n_tx] STA tx element
  int* rxb = txe + n_tx;  // [n_tx] first receive element of each transmit (IDMAP: run rxb + j)
  int* cblo = rxb + n_tx;  // [n_tx] SKIP: first / last stage chunk of each transmit
  int* cbhi = cblo + n_tx;
  int* espan = reinterpret_cast<int*>(smem_raw + 16);  // SKIP: union of the tile's active spans
  float* rmin = reinterpret_cast<float*>(smem_raw + lay.rmin);  // [n_el]
  float* rmax = rmin + n_el;                                    // [n_el]
  int* metaK = reinterpret_cast<int*>(smem_raw + lay.metaK);    // [nst][FPP][TJC] gather base K
  int* metaM = reinterpret_cast<int*>(smem_raw + lay.metaM);    // [nst][TJC] element m
  u64* txd_s = reinterpret_cast<u64*>(smem_raw + lay.txd);      // PW: [n_tx][128]
  const uint32_t win_s = smem_s + (uint32_t)lay.win;            // [nst][TJC/G][FPP][G][W] f32

  // SKIP: with an F-number gate (g.span) every element outside the union of
  // the tile's active spans has weight 0 for all its pixels, so its terms
  // are exact zeros (x is finite, acc never -0: acc + (+-0) == acc) and the
  // stages of channels outside it are neither loaded nor computed
  // (no F-number gate, WM = 2: nothing to skip -- the skip code is compiled out)
  constexpr bool SKIP = WT && IDMAP && WM != 2;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const bool producer = warp == NCW;
  const int slot = (warp >> 2) & (FP - 1);  // consumer: frame slot of the pass
  const int ctid = tid & (NC - 1);          // consumer: pixel-pair thread index
  const int tiles_x = (g.n_x + TXk - 1) / TXk;
  const int tz0 = (blockIdx.x / tiles_x) * TZk, tx0 = (blockIdx.x % tiles_x) * TXk;
  const int col = tx0 + (warp & 1) * CA + (lane & (CA - 1));
  const int rowA = tz0 + ((warp >> 1) & 1) * 2 * RA + (lane >> a.ls), rowB = rowA + RA;
  const int colc = min(col, g.n_x - 1);
  const int rAc = min(rowA, g.n_z - 1), rBc = min(rowB, g.n_z - 1);

  const float c = O::from_double(g.speed_of_sound);
  const float fs = O::from_double(g.sampling_frequency);
  const double px = g.x_pos[colc];
  const float pxd = O::from_double(px);
  const float pzA = O::from_double(g.z_pos[rAc]), pzB = O::from_double(g.z_pos[rBc]);

  // ---- TMEM allocation (warp 0), barrier init (producer lane 0)
  if (warp == 0) {
    tm_alloc(smem_s, (uint32_t)a.tmem_cols);
    tm_relinquish();
  }
  if (SKIP && tid == 0) {  // without an F-number every element is active
    espan[0] = g.span ? n_el : 0;
    espan[1] = g.span ? -1 : n_el - 1;
  }
  if (producer && lane == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(full_s + 8 * s, 32);  // the producer's 32 lanes (one carries expect_tx)
      mbar_init(empty_s + 8 * s, NCW);  // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&rf_map)) : "memory");
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t tlane = tbase + ((uint32_t)((warp & 3) * 32) << 16);  // this warp's lane quarter

  // SKIP: union of the active spans of this warp's 64 pixels (warp-uniform)
  int wlo = 0, whi = n_el - 1;
  // WT: the pair's active element spans (all elements without an F-number)
  int i0A = 0, i1A = n_el - 1, i0B = 0, i1B = n_el - 1;
  // ---- exact receive delays of the consumer thread's pixel pair -> TMEM
  auto load_delays = [&]() {
    if (g.rx_table) {
      // precomputed per plan (bm_das_build_table, the same bits): 32 loads
      // in flight per thread (a CTA's 128 KB arrives at ~HBM latency x 4, not
      // x 16), streamed past L2 (the RF windows want it).  Evaluating part of
      // the elements while the loads fly instead was slower at every split
      // tried (cfg2 one frame: 2/16 of the elements 0.177 ms, 8/16 0.211,
      // against 0.165 ms reading them all)
      const float2* tb =
          reinterpret_cast<const float2*>(g.rx_table) + (int64_t)blockIdx.x * n_el * NC + ctid;
      int m = slot;
      for (; m + 31 * FP < n_el; m += 32 * FP) {
        float2 d[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) d[u] = __ldcs(tb + (int64_t)(m + u * FP) * NC);
#pragma unroll
        for (int u = 0; u < 32; ++u) tm_st2(tlane + 2 * (m + u * FP), d[u].x, d[u].y);
      }
      for (; m < n_el; m += FP) {
        const float2 d = __ldcs(tb + (int64_t)m * NC);
        tm_st2(tlane + 2 * m, d.x, d.y);
      }
    } else {
      // the FP warps sharing a lane quarter split the elements
      for (int m = slot; m < n_el; m += FP) {
        const float2 d = rx_delay_pair(g, m, px, pzA, pzB, c, fs);
        tm_st2(tlane + 2 * m, d.x, d.y);
      }
    }
    if (WT && g.span) {
      // receive apodisation (beamform.py:84-109): weight of element m is
      // window[m - i0] inside the pixel's active span [i0, i1], 0 outside
      const int64_t pA = (int64_t)rAc * g.n_x + colc, pB = (int64_t)rBc * g.n_x + colc;
      i0A = g.span[2 * pA];
      i1A = g.span[2 * pA + 1];
      i0B = g.span[2 * pB];
      i1B = g.span[2 * pB + 1];
      int lo = n_el, hi = -1;
      if (i0A <= i1A) lo = min(lo, i0A), hi = max(hi, i1A);
      if (i0B <= i1B) lo = min(lo, i0B), hi = max(hi, i1B);
      lo = max(lo, 0);
      hi = min(hi, n_el - 1);
      if (slot == 0 && hi >= 0) {
        if (SKIP) {
          atomicMin(&espan[0], lo);
          atomicMax(&espan[1], hi);
        }
      }
      if (SKIP) {
        wlo = __reduce_min_sync(0xffffffffu, lo);
        whi = (int)__reduce_max_sync(0xffffffffu, (unsigned)(hi + 1)) - 1;
      }
    }
    if (PW && slot == 0) {
      // exact transmit delays fs*((z cos + x sin)/c) of the pixel pair for every
      // angle (beamform.py:218-225), once per CTA
      for (int e = 0; e < n_tx; ++e) {
        const float ca = reinterpret_cast<const float*>(g.cos_a)[e];
        const float sa = reinterpret_cast<const float*>(g.sin_a)[e];
        const float xs = O::mul(pxd, sa);
        const float tA = O::mul(fs, O::div(O::add(O::mul(pzA, ca), xs), c));
        const float tB = O::mul(fs, O::div(O::add(O::mul(pzB, ca), xs), c));
        txd_s[e * NC + ctid] = pk(tA, tB);
      }
    }
    tm_wait_st();
  };
  // SKIP needs every warp's span before the stage ranges exist; otherwise the
  // producer starts filling the RF pipeline while the consumers build their
  // delays (the consumers then meet at a barrier of their own)
  const bool early = !SKIP && a.early_producer;
  if (!producer && !early) load_delays();

  const int zl = min(tz0 + TZk, g.n_z) - 1;
  const double x0 = g.x_pos[tx0], x1 = g.x_pos[min(tx0 + TXk, g.n_x) - 1];
  const double z0 = g.z_pos[tz0], z1 = g.z_pos[zl];
  const double k = g.sampling_frequency / g.speed_of_sound;
  // receive-path delay bounds of element m over the tile rectangle (samples);
  // float arithmetic: the window margins of 3-4 samples absorb its error
  const float kf = (float)k, x0f = (float)x0, x1f = (float)x1, z0f = (float)z0, z1f = (float)z1;
  auto rx_bounds = [&](int m, float& lo, float& hi) {
    const float xm = (float)g.elem_x[m];
    const float dmin = fmaxf(0.0f, fmaxf(x0f - xm, xm - x1f));
    const float dmax = fmaxf(fabsf(x0f - xm), fabsf(x1f - xm));
    lo = kf * sqrtf(dmin * dmin + z0f * z0f);
    hi = kf * sqrtf(dmax * dmax + z1f * z1f);
  };
  for (int m = tid; m < n_el; m += NTH) rx_bounds(m, rmin[m], rmax[m]);
  for (int e = tid; e < n_tx; e += NTH) {
    t0v[e] = reinterpret_cast<const float*>(g.t0_smp)[e];
    if (!PW) txe[e] = g.tx_elements[e];
    rxb[e] = IDMAP ? g.rx_map[(int64_t)e * n_rx] : 0;
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
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  if (!producer && early) {
    load_delays();
    // the consumers' own barrier: TMEM columns and transmit delays written by
    // the other warps of the lane quarter / of slot 0
    tm_fence_before();
    asm volatile("bar.sync 1, %0;" ::"r"(32 * NCW) : "memory");
    tm_fence_after();
  }

  // WT: the Hann rows (beamform.py:48-63) are read through L1 from the
  // plan's table: the element row without an F-number (one row for every
  // pixel), else the row of each pixel's span width -- a tile's pixels use a
  // handful of rows, so they stay L1-resident
  const float* hglob = reinterpret_cast<const float*>(g.hann);
  const bool hann = WT && (WM ? WM >= 2 : g.window == BM_HANN);
  const bool gated = WM ? WM != 2 : g.span != nullptr;  // an F-number span per pixel
  auto hann_row = [&](int i0, int i1) -> const float* {
    const int cnt = gated ? max(0, min(i1 - i0 + 1, n_el)) : n_el;
    return hglob + (int64_t)cnt * n_el;
  };
  const float* hrA = hann ? hann_row(i0A, i1A) : nullptr;
  const float* hrB = hann ? hann_row(i0B, i1B) : nullptr;
  // WM = 3 (Hann + F-number): the Hann rows by span width zero-padded by n_el
  // on both sides (g.weight_pad), so a pixel's weight of element m is one read
  // at m - i0 + n_el, zero outside its span -- no span tests or selects per
  // channel.  (The same rows of ones for the rectangular window measured
  // slower than its two compares: 0.53 vs 0.58 of the gather roof.)
  constexpr bool PADW = WM == 3;
  const float* hpA = nullptr;
  const float* hpB = nullptr;
  if (PADW) {
    const float* hp = reinterpret_cast<const float*>(g.weight_pad);
    const int cA = max(0, min(i1A - i0A + 1, n_el)), cB = max(0, min(i1B - i0B + 1, n_el));
    hpA = hp + (int64_t)cA * 3 * n_el + n_el - i0A;
    hpB = hp + (int64_t)cB * 3 * n_el + n_el - i0B;
  }
  // receive weights (w_A, w_B) of element m (beamform.py:84-109)
  auto weight_pair = [&](int m) -> u64 {
    if (PADW) return L::make(__ldg(hpA + m), __ldg(hpB + m));
    if (hann && !gated) return L::splat(__ldg(hrA + m));
    const bool inA = m >= i0A && m <= i1A, inB = m >= i0B && m <= i1B;
    const float wA = inA ? (hann ? __ldg(hrA + (m - i0A)) : 1.0f) : 0.0f;
    const float wB = inB ? (hann ? __ldg(hrB + (m - i0B)) : 1.0f) : 0.0f;
    return L::make(wA, wB);
  };

  const int n_chunks = (n_rx + TJC - 1) / TJC;
  const int f_begin = blockIdx.y * a.frames_per_cta;
  const int f_count = min(a.frames_per_cta, a.n_frames - f_begin);
  const int n_pass = (f_count + FPP - 1) / FPP;
  const int e_lo = a.e_begin, e_hi = a.e_end;
  int Q = n_pass * (e_hi - e_lo) * n_chunks;  // passes x transmits x stages
  int e_first = e_lo, e_last = e_hi - 1;
  if (SKIP) {
    // per-transmit stage range over the active channels; an all-zero tile
    // still runs its first transmit's first stage (its terms are zeros)
    const int elo = espan[0], ehi = espan[1];
    for (int e = e_lo + tid; e < e_hi; e += NTH) {
      const int jlo = max(0, elo - rxb[e]), jhi = min(n_rx - 1, ehi - rxb[e]);
      cblo[e] = jlo <= jhi ? jlo / TJC : 1;
      cbhi[e] = jlo <= jhi ? jhi / TJC : 0;
    }
    __syncthreads();
    int tot = 0;
    e_first = -1;
    for (int e = e_lo; e < e_hi; ++e)
      if (cblo[e] <= cbhi[e]) {
        tot += cbhi[e] - cblo[e] + 1;
        if (e_first < 0) e_first = e;
        e_last = e;
      }
    if (e_first < 0) {
      __syncthreads();
      if (tid == 0) cblo[e_lo] = cbhi[e_lo] = 0;
      __syncthreads();
      e_first = e_last = e_lo;
      tot = 1;
    }
    Q = n_pass * tot;
  }
  // stage cursor: (pass, transmit, chunk); SKIP walks each transmit's range
  auto advance = [&](Cursor& c) {
    if (!SKIP) {
      c.next(n_chunks, e_lo, e_hi);
      return;
    }
    if (++c.cb > cbhi[c.e]) {
      do {
        if (++c.e == e_hi) {
          c.e = e_lo;
          ++c.fl;
        }
      } while (cblo[c.e] > cbhi[c.e]);
      c.cb = cblo[c.e];
    }
  };
  const Cursor c0{0, e_first, SKIP ? cblo[e_first] : 0, 0};

  if (producer) {
    // ================= producer warp: window starts + TMA issue
    if (g.rx_table && a.prefetch > 0 && lane == 0) {
      // the CTA that will take this one's place on the SM (about `prefetch`
      // tiles ahead; modulo the grid, so the last wave warms the next
      // launch's first) finds its delay table in L2
      const int nt = gridDim.x;
      const char* nxt = reinterpret_cast<const char*>(g.rx_table) +
                        (int64_t)((blockIdx.x + a.prefetch) % nt) * n_el * NC * 8;
      const uint32_t bytes = (uint32_t)n_el * NC * 8;
      for (uint32_t o = 0; o < bytes; o += 16384)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nxt + o),
                     "r"(min(16384u, bytes - o))
                     : "memory");
    }
    Cursor cu = c0;
    int s = 0, r = 0;  // stage, round (q = r * nst + s)
    int landed = 0;    // transmits known copied in (g.tx_ready launches)
    for (int q = 0; q < Q; ++q) {
      // round r >= 1 reuses stage s: wait for the consumers' release of round r-1
      if (r > 0) mbar_wait_sleep(empty_s + 8 * s, (uint32_t)(r - 1) & 1u);
      const int e = cu.e;
      if (g.tx_ready && e >= landed) {  // this transmit's RF may still be in flight
        landed = wait_tx_ready(g.tx_ready, g.tx_ready_base, e + 1);
        asm volatile("fence.proxy.async.global;" ::: "memory");  // TMA reads after the acquire
      }
      const float t0 = t0v[e];
      const float lo_e = tmin[e] - t0;
      const int jb = cu.cb * TJC;
      const int jn = min(TJC, n_rx - jb);
      const int row0 = e * n_rx + jb;
      const int fr = f_begin + cu.fl * FPP;  // first frame of the pass
      const uint32_t bar = full_s + 8 * s;
      const int ngr = (jn + G - 1) / G;  // boxes this chunk
#pragma unroll
      for (int u = 0; u < (TJC / G + 31) / 32; ++u) {
        const int gi = lane + 32 * u;
        if (gi < ngr) {
          const int jj0 = gi * G;
          int m = (IDMAP ? rxb[e] : 0) + jb + jj0;
          float rlo = rmin[m];
          if (IDMAP) {  // G adjacent elements share the window
#pragma unroll
            for (int i = 1; i < G; ++i)
              if (jj0 + i < jn) rlo = fminf(rlo, rmin[m + i]);
          } else {
            m = g.rx_map[(int64_t)e * n_rx + jb + jj0];
            rlo = rmin[m];
            metaM[s * TJC + jj0] = m;
          }
          const int ws = ((int)floorf(lo_e + rlo) - 3) & ~3;
          // box = [FPP frames][G traces][W samples]
          const uint32_t dst = win_s + (uint32_t)((s * TJC + jj0) * FPP * W) * 4u;
#pragma unroll
          for (int f = 0; f < FPP; ++f) {
            const uint32_t K0 = dst + (uint32_t)(f * G * W) * 4u - (uint32_t)(kMagicBits + ws) * 4u;
            int* mk = metaK + (s * FPP + f) * TJC + jj0;
            if (G == 4) {
              const uint32_t rs = (uint32_t)W * 4u;
              *reinterpret_cast<int4*>(mk) =
                  make_int4((int)K0, (int)(K0 + rs), (int)(K0 + 2 * rs), (int)(K0 + 3 * rs));
            } else {
              *mk = (int)K0;
            }
          }
          tma_load_3d(dst, &rf_map, ws, row0 + jj0, fr, bar);
        }
      }
      if (lane == 0)
        mbar_arrive_tx(bar, (uint32_t)(ngr * G * FPP * W * 4));
      else
        mbar_arrive(bar);
      advance(cu);
      if (++s == nst) {
        s = 0;
        ++r;
      }
    }
  } else {
    // ================= consumer warps: gather + interpolate + accumulate
    const VT M2 = L::splat(kMagic), NM2 = L::splat(-kMagic);
    const VT ONE2 = L::splat(1.0f), HALF2 = L::splat(0.5f);
    VT acc[FT];
    // sums start at +0, or -- for a later transmit range of the same frames --
    // at the values the previous launch stored (exact: the same f32 sums
    // continue in the same e -> j order)
    auto start_acc = [&](int fl_pass) {
#pragma unroll
      for (int i = 0; i < FT; ++i) {
        acc[i] = L::splat(0.0f);  // +0.0f
        const int fl = fl_pass * FPP + slot * FT + i;
        if (a.accumulate && col < g.n_x && fl < f_count) {
          const float* fo = a.out + (int64_t)(f_begin + fl) * a.out_stride;
          const float oA = rowA < g.n_z ? fo[(int64_t)rowA * g.n_x + col] : 0.0f;
          const float oB = rowB < g.n_z ? fo[(int64_t)rowB * g.n_x + col] : 0.0f;
          acc[i] = L::make(oA, oB);
        }
      }
    };
    start_acc(0);
    VT txd = acc[0], t0e2 = acc[0];
    // the thread's frame i > 0 sits i frame planes ({G, W} floats) after frame 0
    const uint32_t FOFF = (uint32_t)(G * W) * 4u;
    Cursor cur = c0;
    int s = 0;
    uint32_t ph = 0;
    for (int q = 0; q < Q; ++q) {
      mbar_wait(full_s + 8 * s, ph);
      if (cur.cb == (SKIP ? cblo[cur.e] : 0)) {  // first stage of a transmit
        if (PW)
          txd = (VT)txd_s[cur.e * NC + ctid];
        else
          txd = (VT)tm_ld2(tlane + 2 * txe[cur.e]);
        t0e2 = L::splat(t0v[cur.e]);
      }
      const int* MKc = metaK + (s * FPP + slot * FT) * TJC;
      const int* MMc = metaM + s * TJC;
      const int4* MK4 = reinterpret_cast<const int4*>(MKc);  // 4 gather bases per LDS.128
      const int jn = min(TJC, n_rx - cur.cb * TJC);

      // one channel: rxd = receive delays of the pair, K = gather address base
      auto channel = [&](VT rxd, VT wgt, uint32_t K) {
        VT t = L::add(txd, rxd);
        if (T0) t = L::sub(t, t0e2);  // all-zero t0 skips it: x - 0 == x exactly
        const VT r = LINEAR ? L::add_rm(t, M2) : L::add_rm(L::add(t, HALF2), M2);
        float rA, rB;
        unpk((u64)r, rA, rB);
        const uint32_t aA = (uint32_t)__float_as_int(rA) * 4u + K;
        const uint32_t aB = (uint32_t)__float_as_int(rB) * 4u + K;
        if (LINEAR) {
          const VT fr = L::sub(t, L::add(r, NM2));  // a = t - floor(t)
          const VT om = L::sub(ONE2, fr);           // 1 - a
          VT wom = om, wfr = fr;
          if (WT) {
            wom = L::mul(wgt, om);  // w * (1 - a)
            wfr = L::mul(wgt, fr);  // w * a
          }
#pragma unroll
          for (int i = 0; i < FT; ++i) {
            const uint32_t fA = aA + i * FOFF, fB = aB + i * FOFF;
            const VT x0 = L::make(lds0(fA), lds0(fB));
            const VT x1 = L::make(lds1(fA), lds1(fB));
            acc[i] = L::add(acc[i], L::mul(wom, x0));  // acc = out + (w*(1-a)) * x[k0]
            acc[i] = L::add(acc[i], L::mul(wfr, x1));  // out = acc + (w*a) * x[k1]
          }
        } else {
#pragma unroll
          for (int i = 0; i < FT; ++i) {
            const VT x = L::make(lds0(aA + i * FOFF), lds0(aB + i * FOFF));
            acc[i] = L::add(acc[i], WT ? L::mul(wgt, x) : x);
          }
        }
      };
      if (IDMAP && jn == TJC) {
        // identity map: channel j is element j -- one tcgen05.ld.x32 fetches
        // the delay pairs of 16 consecutive channels
        // m0: element of the group's first channel (weights formed 4 at a time)
        auto group = [&](const uint32_t(&r)[32], int m0, int h, auto check) {
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            // SKIP: 4 channels outside every pixel's aperture of this warp are
            // exact zeros (warp-uniform; tested only on groups that straddle
            // the aperture's edge, so the common case keeps one schedule)
            if (decltype(check)::value && (m0 + i > whi || m0 + i + 3 < wlo)) continue;
            const int4 k4 = MK4[(h + i) >> 2];
#define BM_PAIR(R, q) (((u64)R[2 * (i + q) + 1] << 32) | R[2 * (i + q)])
#define BM_W(q) (WT ? weight_pair(m0 + i + q) : 0ull)
            channel(BM_PAIR(r, 0), BM_W(0), (uint32_t)k4.x);
            channel(BM_PAIR(r, 1), BM_W(1), (uint32_t)k4.y);
            channel(BM_PAIR(r, 2), BM_W(2), (uint32_t)k4.z);
            channel(BM_PAIR(r, 3), BM_W(3), (uint32_t)k4.w);
#undef BM_W
#undef BM_PAIR
          }
        };
        const uint32_t tc = tlane + 2 * (rxb[cur.e] + cur.cb * TJC);
#pragma unroll
        for (int h = 0; h < TJC; h += 16) {
          if (SKIP) {  // 16 channels outside every pixel's aperture of this warp: zeros
            const int m0 = rxb[cur.e] + cur.cb * TJC + h;
            if (m0 > whi || m0 + 15 < wlo) continue;
          }
          uint32_t r[32];
          tm_ld32_issue(tc + 2 * h, r);
          tm_wait_regs(r);
          const int m0 = rxb[cur.e] + cur.cb * TJC + h;
          if (SKIP && (m0 < wlo || m0 + 15 > whi))
            group(r, m0, h, std::true_type{});
          else
            group(r, m0, h, std::false_type{});
        }
      } else {
        for (int jj = 0; jj < jn; ++jj) {
          const int m = IDMAP ? rxb[cur.e] + cur.cb * TJC + jj : MMc[jj];
          channel((VT)tm_ld2(tlane + 2 * m), WT ? (VT)weight_pair(m) : 0ull, (uint32_t)MKc[jj]);
        }
      }
      // every gathered sample feeds acc: pinning acc before the arrive keeps
      // the (non-volatile) shared loads of this stage ahead of its release
#pragma unroll
      for (int i = 0; i < FT; ++i) asm volatile("" ::"l"(acc[i]));
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_s + 8 * s);  // stage s may be refilled

      if (cur.e == e_last && cur.cb == (SKIP ? cbhi[e_last] : n_chunks - 1)) {  // pass complete
#pragma unroll
        for (int i = 0; i < FT; ++i) {
          const int fl = cur.fl * FPP + slot * FT + i;  // this thread's frame in the CTA's group
          const int64_t fo = (int64_t)(f_begin + fl) * a.out_stride;
          if (col < g.n_x && fl < f_count) {
            float oA, oB;
            unpk((u64)acc[i], oA, oB);
            if (rowA < g.n_z) a.out[fo + (int64_t)rowA * g.n_x + col] = oA;
            if (rowB < g.n_z) a.out[fo + (int64_t)rowB * g.n_x + col] = oB;
          }
        }
        start_acc(cur.fl + 1);
      }
      advance(cur);
      if (++s == nst) {
        s = 0;
        ph ^= 1;
      }
    }
  }

  // ---- release TMEM (the allocating warp)
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  if (warp == 0) tm_dealloc(tbase, (uint32_t)a.tmem_cols);
}

// ---------------------------------------------------------------- host side

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

// row stride of the staged windows: one channel per box (128-B aligned rows)
// or 4 adjacent channels per box sharing one window start
// nearest-interpolation launches without a delay table may take their own
// tile shape (bm_das_prepare: tile_ls_nearest)
static bool tma_nearest_tile(const bm_das_geometry& g) {
  return g.interp == BM_NEAREST && !g.rx_table && g.rx_contig && g.tile_ls_nearest >= 1 &&
         g.tile_ls_nearest <= 4 && g.window_hint_g4_nearest > 0;
}

int tma_window(const bm_das_geometry& g) {
  const int w = tma_nearest_tile(g) ? g.window_hint_g4_nearest
                : g.rx_contig && g.window_hint_g4 > 0 ? g.window_hint_g4
                                                      : (g.window_hint + 31) & ~31;
  // within 8 samples below a multiple of 32 (up to 192): round up, so a
  // kernel with a compile-time window (WI = 96 .. 192) covers it; larger
  // roundings would cost stages of shared memory
  const int r = (w + 31) & ~31;
  return w <= 192 && r - w <= 8 ? r : w;
}

// tile shape of a launch: contiguous maps use the prepared shape, other maps
// the 16 x 16 tiles window_hint bounds
int tma_ls(const bm_das_geometry& g) {
  if (tma_nearest_tile(g)) return g.tile_ls_nearest;
  return g.rx_contig && g.tile_ls >= 1 && g.tile_ls <= 4 ? g.tile_ls : 3;
}
int tma_tiles(const bm_das_geometry& g) {
  const int ls = tma_ls(g), TZ = 4 * (32 >> ls), TX = 2 << ls;
  return ((g.n_z + TZ - 1) / TZ) * ((g.n_x + TX - 1) / TX);
}

// TMEM columns of one CTA: delay pairs (2 per element) plus, with
// non-uniform apodisation, weight pairs (2 more per element)
static int tma_cols(const bm_das_geometry& g) {
  const int need = 2 * g.n_elements;
  return need <= 256 ? 256 : 512;
}

// 128-channel stages exist for the uniform linear identity-map no-t0 kernels
// (the BASELINE configurations): one stage boundary per 128 channels
static bool tma_has128(const bm_das_geometry& g) {
  return g.uniform && g.interp == BM_LINEAR && !g.t0_nonzero && g.rx_contig;
}

// channels per stage and stage count for the shared-memory share of one CTA
// (fp frames per pass: every stage holds fp frames' windows)
static bool tma_plan(const bm_das_geometry& g, int fp, int& tjc, int& nst, size_t& smem,
                     int max_t = 128) {
  if (fp > 8) return false;
  const int W = tma_window(g);
  const int per_sm = 512 / tma_cols(g);
  const size_t cap = (size_t)(227 * 1024) / per_sm - 1024;
  const bool pw = g.scheme == BM_PW;
  const int only = debug_override(BM_DBG_DAS_TJC);  // tuning override: 32 | 64 | 128
  for (int t : {128, 64, 32, 16}) {
    if (t > g.n_rx && t > 32) continue;
    // 128-channel stages (one-frame launches: the only ones with fp == 1
    // left): one stage boundary per 128 channels pays on launches of many
    // waves (cfg3 / cfg5: 3.13 -> 3.08 / 24.3 -> 23.6 ms); a few-wave launch
    // fills its pipeline sooner with 64 x 4 stages (cfg2 0.174 -> 0.168 ms)
    if (t == 128 && (!tma_has128(g) || fp != 1 || (only != 128 && tma_tiles(g) < 1800)))
      continue;
    if (t == 16 && fp < 4) continue;  // 16-channel stages: four frames per pass only
    if (t > max_t) continue;          // no kernel instantiated for this stage size
    if (only && t != only) continue;
    int n = kTmaMaxStages;
    while (n >= 2 &&
           (size_t)TmaLayout(g.n_tx, g.n_elements, t, n, W, pw, fp).total > cap)
      --n;
    if (n >= (t == 64 && fp == 1 ? 3 : 2)) {
      tjc = t;
      nst = n;
      smem = cap;
      return true;
    }
  }
  return false;
}

int das_tma_eligible(const bm_das_geometry& g, int64_t rf_stride) {
  if (g.dtype != BM_F32 || g.window_hint <= 0 || tma_window(g) > 256) return 0;
  if (!g.uniform && g.window == BM_HANN && !g.hann) return 0;
  if (g.rx_contig && g.window_hint_g4 <= 0) return 0;  // 4-channel boxes need the bound
  if (g.n_samples % 4 != 0 || rf_stride % 4 != 0) return 0;  // 16-B TMA strides
  if (2 * g.n_elements > 512) return 0;                       // pair layout in TMEM
  if ((int64_t)g.n_tx * g.n_rx > 0x7fffffffLL) return 0;
  int tjc, nst;
  size_t smem;
  if (!tma_plan(g, 1, tjc, nst, smem)) return 0;
  return encode_tiled() != nullptr;
}

// Launch shape of a TMA DAS launch over n_frames frames: frames per CTA, the
// pass shape (fp warp groups sharing one delay table x ft frames per thread)
// and the stage plan.  False when the TMA kernel cannot run this geometry.
struct TmaChoice {
  int fpc, fp, ft, tjc, nst;
  size_t smem;
};
static bool tma_choose(const bm_das_geometry& g, int n_frames, TmaChoice& c) {
  if (!tma_plan(g, 1, c.tjc, c.nst, c.smem)) return false;
  const int tiles = tma_tiles(g);
  const int per_sm = 512 / tma_cols(g);
  // frames per CTA: amortise the per-CTA delay-table build over a frame
  // group while keeping >= 4 waves of CTAs for load balance
  int fpc = 1;
  while (fpc < 16 && fpc * 2 <= n_frames &&
         (int64_t)tiles * ((n_frames + fpc * 2 - 1) / (fpc * 2)) >= 4LL * per_sm * sm_count())
    fpc *= 2;
  if (const int want = debug_override(BM_DBG_DAS_FPC); want >= 1)  // test hook
    fpc = want < n_frames ? want : n_frames;
  c.fpc = fpc;
  // several frames per pass for identity-map apertures whenever a CTA owns
  // enough frames: fp consumer warp groups share one delay table (FP), each
  // thread accumulates ft frames (FT)
  c.fp = c.ft = 1;
  if (g.rx_contig) {
    const int ofp = debug_override(BM_DBG_DAS_FP);  // tuning override: 1 | 2
    const int oft = debug_override(BM_DBG_DAS_FT);  // tuning override: 1 | 2 | 4 (the most tried)
    const int want_fp = ofp == 1 ? 1 : 2;
    const int want_ft = oft ? (oft >= 4 ? 4 : oft == 2 ? 2 : 1) : 4;
    // several frames per thread: all-zero t0; non-uniform apodisation (its
    // w*(1-a), w*a shared by the frames too) with four frames per thread
    const bool ftn_ok = !g.t0_nonzero;
    // most frames per pass first; FP = 2 before FP = 1 at equal FT
    const int cand[6][2] = {{want_fp, 4}, {1, 4}, {want_fp, 2}, {1, 2}, {want_fp, 1}, {1, 1}};
    for (const auto& cd : cand) {
      const int f = cd[0], t = cd[1];
      if (t > want_ft || f * t == 1 || (t > 1 && !ftn_ok) || fpc < f * t) continue;
      if (t == 2 && !g.uniform) continue;  // not instantiated
      int t2, n2;
      size_t s2;
      if (tma_plan(g, f * t, t2, n2, s2, t == 4 ? 32 : 64)) {
        c.fp = f;
        c.ft = t;
        c.tjc = t2;
        c.nst = n2;
        c.smem = s2;
        break;
      }
    }
  }
  return true;
}

int das_tma_shape(const bm_das_geometry& g, int n_frames, int32_t* shape) {
  TmaChoice c;
  if (n_frames < 1 || !tma_choose(g, n_frames, c)) return -1;
  shape[0] = c.fpc;
  shape[1] = c.fp;
  shape[2] = c.ft;
  shape[3] = c.tjc;
  shape[4] = c.nst;
  shape[5] = tma_window(g);
  return 0;
}

int das_tma_launch(const bm_das_geometry& g, const void* rf, int64_t rf_stride, void* out,
                   int64_t out_stride, int n_frames, int e_begin, int e_end, int accumulate,
                   cudaStream_t s) {
  if (((uintptr_t)rf & 15) != 0) return -1;  // caller falls back
  TmaChoice c;
  if (!tma_choose(g, n_frames, c)) return -1;
  const int W = tma_window(g);
  const int tiles = tma_tiles(g);
  const int fpc = c.fpc, fp = c.fp, ft = c.ft, tjc = c.tjc, nst = c.nst;
  const size_t smem = c.smem;
  // RF as a 3-D tensor: samples x (transmit, channel) rows x frames
  CUtensorMap map;
  const int64_t fstride = n_frames > 1 ? rf_stride : (int64_t)g.n_tx * g.n_rx * g.n_samples;
  cuuint64_t dims[3] = {(cuuint64_t)g.n_samples, (cuuint64_t)g.n_tx * g.n_rx,
                        (cuuint64_t)n_frames};
  cuuint64_t strides[2] = {(cuuint64_t)g.n_samples * 4, (cuuint64_t)fstride * 4};
  cuuint32_t box[3] = {(cuuint32_t)W, g.rx_contig ? 4u : 1u, (cuuint32_t)(fp * ft)};
  cuuint32_t estr[3] = {1, 1, 1};
  if (encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(rf), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  TmaArgs a{g,   (float*)out, out_stride, n_frames,    e_begin,   e_end,
            accumulate, fpc,  W,    nst,        tma_cols(g), tma_ls(g), 0};
  // tiles between a CTA and its successor on an SM: the co-resident CTAs
  a.prefetch = debug_override(BM_DBG_DAS_PREFETCH) < 0 ? 0 : (512 / tma_cols(g)) * sm_count();
  a.early_producer = debug_override(BM_DBG_DAS_LATE_PRODUCER) == 1 ? 0 : 1;
  const bool pw = g.scheme == BM_PW, lin = g.interp == BM_LINEAR;
  typedef void (*kfn)(const CUtensorMap, const TmaArgs);
#define BM_TMA_ROW(J, WT)                                                                  \
  das_tma_kernel<false, false, false, false, J, WT>,                                        \
      das_tma_kernel<false, false, false, true, J, WT>,                                     \
      das_tma_kernel<false, false, true, false, J, WT>,                                     \
      das_tma_kernel<false, false, true, true, J, WT>,                                      \
      das_tma_kernel<false, true, false, false, J, WT>,                                     \
      das_tma_kernel<false, true, false, true, J, WT>,                                      \
      das_tma_kernel<false, true, true, false, J, WT>,                                      \
      das_tma_kernel<false, true, true, true, J, WT>,                                       \
      das_tma_kernel<true, false, false, false, J, WT>,                                     \
      das_tma_kernel<true, false, false, true, J, WT>,                                      \
      das_tma_kernel<true, false, true, false, J, WT>,                                      \
      das_tma_kernel<true, false, true, true, J, WT>,                                       \
      das_tma_kernel<true, true, false, false, J, WT>,                                      \
      das_tma_kernel<true, true, false, true, J, WT>,                                       \
      das_tma_kernel<true, true, true, false, J, WT>, das_tma_kernel<true, true, true, true, J, WT>
  // rows: uniform/32, uniform/64, weighted/32, weighted/64
  static const kfn table[64] = {BM_TMA_ROW(32, false), BM_TMA_ROW(64, false),
                                BM_TMA_ROW(32, true), BM_TMA_ROW(64, true)};
#undef BM_TMA_ROW
  kfn k = table[(g.uniform ? 0 : 32) + (tjc >= 64 ? 16 : 0) +
                ((pw ? 8 : 0) | (lin ? 4 : 0) | (g.t0_nonzero ? 2 : 0) | (g.rx_contig ? 1 : 0))];
  if (tjc == 128) {
    if (!tma_has128(g)) return -1;
    k = pw ? das_tma_kernel<true, true, false, true, 128> : das_tma_kernel<false, true, false, true, 128>;
  }
  if (!g.uniform && fp == 1 && ft == 1 && g.rx_contig && !g.t0_nonzero && (tjc == 32 || tjc == 64)) {
    // one-frame weighted launches (the drop-in path with Hann / F-number
    // receive weights): the weight mode compiled in, as for the batched
    // kernels -- the run-time form is 2.2x the uniform kernel's time there
    // (branches, span tests, and an instruction footprint that misses the
    // instruction cache)
    const int wm = g.window == BM_HANN ? (g.span ? 3 : 2) : 1;
    if (wm != 3 || g.weight_pad) {
#define BM_TMA_W1(J, M)                                                                    \
  das_tma_kernel<false, false, false, true, J, true, 1, 1, 0, M>,                          \
      das_tma_kernel<true, false, false, true, J, true, 1, 1, 0, M>,                       \
      das_tma_kernel<false, true, false, true, J, true, 1, 1, 0, M>,                       \
      das_tma_kernel<true, true, false, true, J, true, 1, 1, 0, M>
      static const kfn table9[24] = {BM_TMA_W1(32, 1), BM_TMA_W1(64, 1), BM_TMA_W1(32, 2),
                                     BM_TMA_W1(64, 2), BM_TMA_W1(32, 3), BM_TMA_W1(64, 3)};
#undef BM_TMA_W1
      k = table9[(wm - 1) * 8 + (tjc == 64 ? 4 : 0) + (lin ? 2 : 0) + (pw ? 1 : 0)];
    }
  }
  if (fp == 2) {
#define BM_TMA_FP2(J, WT)                                                                   \
  das_tma_kernel<false, false, false, true, J, WT, 2>,                                      \
      das_tma_kernel<false, false, true, true, J, WT, 2>,                                   \
      das_tma_kernel<false, true, false, true, J, WT, 2>,                                   \
      das_tma_kernel<false, true, true, true, J, WT, 2>,                                    \
      das_tma_kernel<true, false, false, true, J, WT, 2>,                                   \
      das_tma_kernel<true, false, true, true, J, WT, 2>,                                    \
      das_tma_kernel<true, true, false, true, J, WT, 2>,                                    \
      das_tma_kernel<true, true, true, true, J, WT, 2>
    // identity map only; rows: uniform/32, uniform/64, weighted/32, weighted/64
    static const kfn table2[32] = {BM_TMA_FP2(32, false), BM_TMA_FP2(64, false),
                                   BM_TMA_FP2(32, true), BM_TMA_FP2(64, true)};
#undef BM_TMA_FP2
    k = table2[(g.uniform ? 0 : 16) + (tjc >= 64 ? 8 : 0) +
               ((pw ? 4 : 0) | (lin ? 2 : 0) | (g.t0_nonzero ? 1 : 0))];
  }
  if (ft == 2) {
    // uniform identity-map no-t0 apertures (the BASELINE configurations),
    // linear and nearest; rows: FP = 1 / 2 x 16 / 32 / 64-channel stages (16
    // only with four frames per pass)
#define BM_TMA_FT2(J, F)                                                                   \
  das_tma_kernel<false, false, false, true, J, false, F, 2>,                               \
      das_tma_kernel<true, false, false, true, J, false, F, 2>,                            \
      das_tma_kernel<false, true, false, true, J, false, F, 2>,                            \
      das_tma_kernel<true, true, false, true, J, false, F, 2>
    static const kfn table3[24] = {nullptr,           nullptr, nullptr, nullptr,
                                   BM_TMA_FT2(32, 1), BM_TMA_FT2(64, 1),
                                   BM_TMA_FT2(16, 2), BM_TMA_FT2(32, 2), BM_TMA_FT2(64, 2)};
#undef BM_TMA_FT2
    if (tjc > 64) return -1;
    k = table3[(fp == 2 ? 12 : 0) + (tjc == 64 ? 8 : tjc == 32 ? 4 : 0) + (lin ? 2 : 0) +
               (pw ? 1 : 0)];
    if (!k) return -1;
  }
  if (ft == 4) {
    // four frames per thread, contiguous maps, no t0, uniform and weighted;
    // rows: uniform / weighted x FP = 1 / 2 x 16 / 32-channel stages
    // (weighted: the weight mode compiled in -- rectangular + F, Hann, Hann
    // + F over g.weight_pad; without the padded rows Hann + F takes the
    // generic kernel)
#define BM_TMA_FT4(J, F, WT, M)                                                            \
  das_tma_kernel<false, false, false, true, J, WT, F, 4, 0, M>,                            \
      das_tma_kernel<true, false, false, true, J, WT, F, 4, 0, M>,                         \
      das_tma_kernel<false, true, false, true, J, WT, F, 4, 0, M>,                         \
      das_tma_kernel<true, true, false, true, J, WT, F, 4, 0, M>
#define BM_TMA_FT4W(M)                                                                     \
  BM_TMA_FT4(16, 1, true, M), BM_TMA_FT4(32, 1, true, M), BM_TMA_FT4(16, 2, true, M),      \
      BM_TMA_FT4(32, 2, true, M)
    static const kfn table4[64] = {
        BM_TMA_FT4(16, 1, false, 0), BM_TMA_FT4(32, 1, false, 0), BM_TMA_FT4(16, 2, false, 0),
        BM_TMA_FT4(32, 2, false, 0), BM_TMA_FT4W(1), BM_TMA_FT4W(2), BM_TMA_FT4W(3)};
#undef BM_TMA_FT4W
#undef BM_TMA_FT4
    if (tjc > 32) return -1;
    const int wm4 = g.uniform ? 0 : g.window == BM_HANN ? (g.span ? 3 : 2) : 1;
    if (wm4 == 3 && !g.weight_pad) return -1;
    k = table4[wm4 * 16 + (fp == 2 ? 8 : 0) + (tjc == 32 ? 4 : 0) + (lin ? 2 : 0) +
               (pw ? 1 : 0)];
    // compile-time window widths for the uniform 16-channel kernels: the
    // frame-plane offsets of frames 1..3 become LDS immediates (cfg2: 12 %
    // fewer instructions in the gather loop, +3 % frames/s)
    const bool rt_w = debug_override(BM_DBG_DAS_RUNTIME_W) > 0;  // A/B override
    const int wi = W == 96 ? 0 : W == 128 ? 1 : W == 160 ? 2 : W == 192 ? 3 : -1;
    if (wi >= 0 && g.uniform && tjc == 16 && !rt_w) {
#define BM_TMA_WI(F, WV)                                                                   \
  das_tma_kernel<false, false, false, true, 16, false, F, 4, WV>,                          \
      das_tma_kernel<true, false, false, true, 16, false, F, 4, WV>,                       \
      das_tma_kernel<false, true, false, true, 16, false, F, 4, WV>,                       \
      das_tma_kernel<true, true, false, true, 16, false, F, 4, WV>
      static const kfn table7[32] = {
          BM_TMA_WI(1, 96),  BM_TMA_WI(1, 128), BM_TMA_WI(1, 160), BM_TMA_WI(1, 192),
          BM_TMA_WI(2, 96),  BM_TMA_WI(2, 128), BM_TMA_WI(2, 160), BM_TMA_WI(2, 192)};
#undef BM_TMA_WI
      k = table7[(fp == 2 ? 16 : 0) + wi * 4 + (lin ? 2 : 0) + (pw ? 1 : 0)];
    }
    if (W == 96 && !g.uniform && fp == 2 && !rt_w) {
      // weighted (Hann / F-number), 96-sample windows: 16 / 32-channel stages
      // ... with the weight mode compiled in (rectangular + F, Hann, Hann + F)
#define BM_TMA_WIW(J, M)                                                                   \
  das_tma_kernel<false, false, false, true, J, true, 2, 4, 96, M>,                         \
      das_tma_kernel<true, false, false, true, J, true, 2, 4, 96, M>,                      \
      das_tma_kernel<false, true, false, true, J, true, 2, 4, 96, M>,                      \
      das_tma_kernel<true, true, false, true, J, true, 2, 4, 96, M>
      static const kfn table8[24] = {BM_TMA_WIW(16, 1), BM_TMA_WIW(32, 1), BM_TMA_WIW(16, 2),
                                     BM_TMA_WIW(32, 2), BM_TMA_WIW(16, 3), BM_TMA_WIW(32, 3)};
#undef BM_TMA_WIW
      // (Hann + F without the padded rows already left for the generic kernel)
      const int wm = g.window == BM_HANN ? (g.span ? 3 : 2) : 1;
      if (wm != 3 || g.weight_pad)
        k = table8[(wm - 1) * 8 + (tjc == 32 ? 4 : 0) + (lin ? 2 : 0) + (pw ? 1 : 0)];
    }
  }
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return BM_ERR_CUDA;
  dim3 grid(tiles, (n_frames + fpc - 1) / fpc);
  if (debug_override(BM_DBG_DAS_VERBOSE) > 0)
    fprintf(stderr, "das_tma: fp=%d ft=%d tjc=%d nst=%d W=%d fpc=%d smem=%zu\n", fp, ft, tjc, nst, W, fpc, smem);
  k<<<grid, 32 * (4 * fp + 1), smem, s>>>(map, a);
  return cuda_status();
}

}  // namespace bm

extern "C" int64_t bm_das_table_bytes(const bm_das_geometry* g) {
  if (!g || g->n_elements < 1 || g->n_z < 1 || g->n_x < 1) return 0;
  if (g->dtype == BM_F64)  // f64 delays of each consumer thread's pixel
    return (int64_t)bm::tma_tiles(*g) * g->n_elements * 256 * 8;
  if (g->dtype != BM_F32) return 0;
  return (int64_t)bm::tma_tiles(*g) * g->n_elements * 128 * 8;
}

extern "C" int bm_das_build_table(const bm_das_geometry* g, float* table, void* stream) {
  if (!g || !table || !g->elem_x || !g->x_pos || !g->z_pos) return BM_ERR_INVALID_ARGUMENT;
  if (bm_das_table_bytes(g) <= 0) return BM_ERR_UNSUPPORTED;
  if (g->dtype == BM_F64)
    return bm::das_table64_build(*g, reinterpret_cast<double*>(table), (cudaStream_t)stream);
  const dim3 grid((unsigned)bm::tma_tiles(*g), (unsigned)std::min(g->n_elements, 16));
  bm::das_table_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(*g, bm::tma_ls(*g),
                                                               reinterpret_cast<float2*>(table));
  return bm::cuda_status();
}
