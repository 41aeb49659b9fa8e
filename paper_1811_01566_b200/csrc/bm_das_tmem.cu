// K1 fast path with the receive-delay table in TENSOR MEMORY (sm_100a).
//
// Same arithmetic (and therefore the same bits) as das_fast_kernel and the
// reference's f32 das_beamform (beamform.py:122-187 with the DasPlan delays
// of :211-228).  The difference is where the per-tile delay table
// D[m][pixel] = fs*(sqrt(dx^2+z^2)/c) lives:
//
//  * The shared-memory kernel keeps D in SMEM (n_el x 8 B per thread), which
//    caps residency at 3 CTAs x 2 warps per SM and costs one LDS.64 and one
//    shared-memory wavefront per channel.
//  * Here D lives in TMEM, the 256 KB per-SM tensor memory that no other part
//    of this kernel uses: thread (warp w, lane l) owns TMEM lane 32w + l and
//    the two columns 2m, 2m+1 hold its pixel pair's delays to element m.  A
//    chunk of 16 channels is ONE tcgen05.ld.32x32b.x32 into registers, and
//    shared memory is left to the RF windows -- 2 CTAs x 4 warps per SM.
//
// CTA = 128 threads, tile = 16 rows x 16 columns; warp w covers an 8 x 8
// block (columns 8*(w&1).., rows 8*(w>>1)..), lane l the pixel pair
// (row l/8, col l%8) / (row l/8 + 4, col l%8), so each gather of a warp is a
// 4 x 8 pixel block (conflict-free, see das_fast_kernel).  RF windows are
// staged per chunk of 32 channels with cp.async exactly as in
// das_fast_kernel.
#include "bm_tmem.cuh"

namespace bm {

constexpr int TX = 16, NST = 3;  // channels per chunk (32 or 64) is a launch argument

struct TmemArgs {
  bm_das_geometry g;
  const float* rf;
  int64_t rf_stride;
  float* out;
  int64_t out_stride;
  int n_frames;
  int frames_per_cta;
  int W;          // staged window capacity per channel (samples, multiple of 4)
  int tmem_cols;  // allocated TMEM columns (power of two >= 2 * n_elements)
  int jc;         // receive channels per staged chunk: 32 or 64
};

// PAIR: tile 16 x 16, thread = pixel pair (r, c) / (r + 4, c), TMEM columns 2m, 2m+1.
// !PAIR: tile 8 x 16, thread = one pixel, TMEM column m, 4 CTAs per SM fit in TMEM.
// Either way a warp's 32 gathers of one channel cover a 4 x 8 pixel block.
// HYB (pair only): a 6-warp CTA whose warps 4-5 keep their delay table in
// SHARED memory next to the four TMEM warps -- TMEM caps the SM at 8 warps,
// TMEM + SMEM together hold 12.  Tile 16 x 24 (warps 4-5: columns 16-23).
template <bool PAIR, bool PW, bool LINEAR, bool T0, bool IDMAP, bool HYB, int TJC>
__global__ void __launch_bounds__(HYB ? 192 : 128, PAIR ? 2 : 4) das_tmem_kernel(const TmemArgs a) {
  using O = R<float>;
  using L = Lane<PAIR>;
  typedef typename L::T VT;
  constexpr int NTH = HYB ? 192 : 128;
  constexpr int TXk = HYB ? 24 : TX;
  constexpr bool TXD_SMEM = PW && !HYB;  // precomputed PW transmit delays
  constexpr int TZk = PAIR ? 16 : 8;
  constexpr int CPE = PAIR ? 2 : 1;  // TMEM columns per element
  const bm_das_geometry& g = a.g;
  const int n_el = g.n_elements, n_tx = g.n_tx, n_rx = g.n_rx, n_s = g.n_samples;
  const int W = a.W;

  // shared memory: [tmem base][tmin|tmax][meta ring][windows]
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // [tmem base][tmin|tmax|t0|tx sel][rmin|rmax][meta ring][PW tx delays][windows]
  const int off_tmin = 16;
  const int off_rmin = (off_tmin + 16 * n_tx + 15) & ~15;
  const int off_meta = (off_rmin + 8 * n_el + 15) & ~15;
  const int nrp = (n_rx + 3) & ~3;  // meta row stride (16 B aligned rows)
  const int off_txd = off_meta + 24 * nrp;
  const int off_dsm = off_txd + (TXD_SMEM ? n_tx * NTH * (int)sizeof(u64) : 0);
  const int off_win = off_dsm + (HYB ? n_el * 64 * (int)sizeof(u64) : 0);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw);
  float* tmin = reinterpret_cast<float*>(smem_raw + off_tmin);  // [n_tx]
  float* tmax = tmin + n_tx;                                    // [n_tx]
  float* t0v = tmax + n_tx;                                     // [n_tx] fs*t0
  int* txe = reinterpret_cast<int*>(t0v + n_tx);                // [n_tx] STA tx element
  float* rmin = reinterpret_cast<float*>(smem_raw + off_rmin);  // [n_el]
  float* rmax = rmin + n_el;                                    // [n_el]
  int* metaX = reinterpret_cast<int*>(smem_raw + off_meta);     // [3][nrp] len | m << 13
  int* metaK = metaX + 3 * nrp;                                 // [3][nrp] gather base K
  u64* txd_s = reinterpret_cast<u64*>(smem_raw + off_txd);      // PW: [n_tx][NTH]
  u64* dsm = reinterpret_cast<u64*>(smem_raw + off_dsm);        // HYB: [n_el][64] pairs
  float* win = reinterpret_cast<float*>(smem_raw + off_win);    // [NST][TJC][W]

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int tiles_x = (g.n_x + TXk - 1) / TXk;
  const int tz0 = (blockIdx.x / tiles_x) * TZk, tx0 = (blockIdx.x % tiles_x) * TXk;
  const bool tm_warp = !HYB || warp < 4;  // delay table in TMEM (else shared memory)
  const int wcol = tm_warp ? (warp & 1) * 8 : 16;
  const int wrow = tm_warp ? (warp >> 1) * (PAIR ? 8 : 4) : (warp - 4) * 8;
  const int col = tx0 + wcol + (lane & 7);
  const int rowA = tz0 + wrow + (lane >> 3), rowB = rowA + 4;
  const int dtid = tid - 128;  // HYB warps 4-5: row of the shared-memory table
  const int colc = min(col, g.n_x - 1);
  const int rAc = min(rowA, g.n_z - 1), rBc = min(rowB, g.n_z - 1);

  const float c = O::from_double(g.speed_of_sound);
  const float fs = O::from_double(g.sampling_frequency);
  const double px = g.x_pos[colc];
  const float pxd = O::from_double(px);
  const float pzA = O::from_double(g.z_pos[rAc]), pzB = O::from_double(g.z_pos[rBc]);
  const uint32_t win_s = (uint32_t)__cvta_generic_to_shared(win);

  // ---- TMEM allocation (warp 0), address broadcast through shared memory
  if (warp == 0) {
    tm_alloc((uint32_t)__cvta_generic_to_shared(tmem_slot), (uint32_t)a.tmem_cols);
    tm_relinquish();
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t tlane = tbase + ((uint32_t)((warp & 3) * 32) << 16);  // this warp's lane quarter

  // ---- exact receive delays of the thread's pixel(s) -> TMEM
  for (int m = 0; m < n_el; ++m) {
    const float dx = O::from_double(g.elem_x[m] - px);
    const float dA = O::mul(fs, O::div(O::sqrt(O::add(O::mul(dx, dx), O::mul(pzA, pzA))), c));
    if (PAIR) {
      const float dB = O::mul(fs, O::div(O::sqrt(O::add(O::mul(dx, dx), O::mul(pzB, pzB))), c));
      if (tm_warp)
        tm_st2(tlane + 2 * m, dA, dB);
      else
        dsm[m * 64 + dtid] = pk(dA, dB);
    } else {
      tm_st1(tlane + m, dA);
    }
  }
  if (tm_warp) tm_wait_st();

  const int zl = min(tz0 + TZk, g.n_z) - 1;
  const double x0 = g.x_pos[tx0], x1 = g.x_pos[min(tx0 + TXk, g.n_x) - 1];
  const double z0 = g.z_pos[tz0], z1 = g.z_pos[zl];
  const double k = g.sampling_frequency / g.speed_of_sound;
  // receive-path delay bounds of element m over the tile rectangle (samples)
  // (float arithmetic: the window margins of 3-4 samples absorb its error)
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
  auto pw_txd = [&](int e) -> VT {  // fs*((z cos + x sin)/c), beamform.py:218-225
    const float ca = reinterpret_cast<const float*>(g.cos_a)[e];
    const float sa = reinterpret_cast<const float*>(g.sin_a)[e];
    const float xs = O::mul(pxd, sa);
    const float tA = O::mul(fs, O::div(O::add(O::mul(pzA, ca), xs), c));
    const float tB = PAIR ? O::mul(fs, O::div(O::add(O::mul(pzB, ca), xs), c)) : tA;
    return L::make(tA, tB);
  };
  if (TXD_SMEM) {
    // exact transmit delays of the thread's pixels for every angle, once per CTA
    for (int e = 0; e < n_tx; ++e) {
      const float ca = reinterpret_cast<const float*>(g.cos_a)[e];
      const float sa = reinterpret_cast<const float*>(g.sin_a)[e];
      const float xs = O::mul(pxd, sa);
      const float tA = O::mul(fs, O::div(O::add(O::mul(pzA, ca), xs), c));
      const float tB = PAIR ? O::mul(fs, O::div(O::add(O::mul(pzB, ca), xs), c)) : tA;
      txd_s[e * NTH + tid] = pk(tA, tB);
    }
  }
  __syncthreads();

  const float* __restrict__ t0s = t0v;
  const int n_chunks = (n_rx + TJC - 1) / TJC;
  const int f_begin = blockIdx.y * a.frames_per_cta;
  const int f_count = min(a.frames_per_cta, a.n_frames - f_begin);
  const int Q = f_count * n_tx * n_chunks;
  const int n_T = f_count * n_tx;

  // staging metadata of running transmit T: per channel
  //   x = staged length | element m << 13,  y = K (gather address base)
  auto make_meta = [&](int T) {
    const int e = T % n_tx;
    int* MX = metaX + (T % 3) * nrp;
    int* MK = metaK + (T % 3) * nrp;
    const float t0 = t0s[e];
    const float lo_e = tmin[e] - t0, hi_e = tmax[e] - t0;
    const int* map = g.rx_map + (int64_t)e * n_rx;
    for (int j = tid; j < n_rx; j += NTH) {
      const int m = IDMAP ? j : map[j];
      const float rlo = rmin[m], rhi = rmax[m];
      const int ws = ((int)floorf(lo_e + rlo) - 3) & ~3;
      const int hi = (int)floorf(hi_e + rhi) + 4;
      const int len = min((hi - ws + 3) & ~3, W);  // host guarantees <= W
      const int cb = j / TJC, jj = j - cb * TJC;
      const int buf = (T * n_chunks + cb) % NST;
      const uint32_t K = win_s + (uint32_t)((buf * TJC + jj) * W) * 4u -
                         (uint32_t)(kMagicBits + ws) * 4u;
      MX[j] = len | (m << 13);
      MK[j] = (int)K;
    }
  };
  // cp.async staging: 4 threads per channel, 16 B copies at fixed slots
  // o = 4*(tid % 4) + 16*i, i < ceil(W / 16) <= 16
  const int ld_o = 4 * (tid & 3);  // channel jj = tid / 4 (+ 32 per sub-chunk)
  // returns the fast path's source pointer, which the caller keeps live
  // until the end of the iteration so that no instruction overwrites a
  // register an in-flight cp.async still reads (a write-after-read stall)
  auto issue_loads = [&](int slot, int tslot, const Cursor& cu, int ld_jj) -> const float* {
    const int64_t ld_trace = (int64_t)ld_jj * n_s + ld_o;
    const int j = cu.cb * TJC + ld_jj;
    if ((HYB && tid >= 128) || j >= n_rx) return nullptr;
    const int2 mm = make_int2(metaX[tslot * nrp + j], metaK[tslot * nrp + j]);
    const int len = mm.x & 0x1fff;
    const uint32_t wb = win_s + (uint32_t)((slot * TJC + ld_jj) * W + ld_o) * 4u;
    // K = wb0 - 4*(M_bits + ws) mod 2^32, so (wb0 - K)/4 = (M_bits + ws) mod 2^30
    const int ws = (int)((wb - (uint32_t)ld_o * 4u - (uint32_t)mm.y) >> 2) -
                   (kMagicBits & 0x3fffffff);
    const float* tr = a.rf + (int64_t)(f_begin + cu.fl) * a.rf_stride +
                      ((int64_t)cu.e * n_rx + cu.cb * TJC) * n_s + ld_trace;
    if (ws >= 0 && ws + len <= n_s) {
      // whole window inside the trace (the common case): one source pointer,
      // copies at immediate +64 B steps
      const float* p = tr + ws;
      const int nc = (len - ld_o + 15) >> 4;  // this thread's copies
      asm volatile(
          "{\n .reg .pred q<8>;\n"
          " setp.gt.s32 q0, %2, 0;\n setp.gt.s32 q1, %2, 1;\n setp.gt.s32 q2, %2, 2;\n"
          " setp.gt.s32 q3, %2, 3;\n setp.gt.s32 q4, %2, 4;\n setp.gt.s32 q5, %2, 5;\n"
          " setp.gt.s32 q6, %2, 6;\n setp.gt.s32 q7, %2, 7;\n"
          " @q0 cp.async.cg.shared.global [%0], [%1], 16;\n"
          " @q1 cp.async.cg.shared.global [%0+64], [%1+64], 16;\n"
          " @q2 cp.async.cg.shared.global [%0+128], [%1+128], 16;\n"
          " @q3 cp.async.cg.shared.global [%0+192], [%1+192], 16;\n"
          " @q4 cp.async.cg.shared.global [%0+256], [%1+256], 16;\n"
          " @q5 cp.async.cg.shared.global [%0+320], [%1+320], 16;\n"
          " @q6 cp.async.cg.shared.global [%0+384], [%1+384], 16;\n"
          " @q7 cp.async.cg.shared.global [%0+448], [%1+448], 16;\n}\n" ::"r"(wb),
          "l"(p), "r"(nc)
          : "memory");
      if (nc > 8)  // windows of 129-256 samples
        asm volatile(
            "{\n .reg .pred q<8>;\n"
            " setp.gt.s32 q0, %2, 8;\n setp.gt.s32 q1, %2, 9;\n setp.gt.s32 q2, %2, 10;\n"
            " setp.gt.s32 q3, %2, 11;\n setp.gt.s32 q4, %2, 12;\n setp.gt.s32 q5, %2, 13;\n"
            " setp.gt.s32 q6, %2, 14;\n setp.gt.s32 q7, %2, 15;\n"
            " @q0 cp.async.cg.shared.global [%0+512], [%1+512], 16;\n"
            " @q1 cp.async.cg.shared.global [%0+576], [%1+576], 16;\n"
            " @q2 cp.async.cg.shared.global [%0+640], [%1+640], 16;\n"
            " @q3 cp.async.cg.shared.global [%0+704], [%1+704], 16;\n"
            " @q4 cp.async.cg.shared.global [%0+768], [%1+768], 16;\n"
            " @q5 cp.async.cg.shared.global [%0+832], [%1+832], 16;\n"
            " @q6 cp.async.cg.shared.global [%0+896], [%1+896], 16;\n"
            " @q7 cp.async.cg.shared.global [%0+960], [%1+960], 16;\n}\n" ::"r"(wb),
            "l"(p), "r"(nc)
            : "memory");
      return p;
    }
    // window crosses a trace end (rare): per-copy source and zero fill; the
    // copies of each 8-block use distinct address registers
    for (int i0 = 0; i0 < 16 && ld_o + 16 * i0 < len; i0 += 8) {
      const float* src[8];
      int nb[8], act[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = i0 + k;
        const int o = ld_o + 16 * i;
        const bool in = (unsigned)(ws + o) <= (unsigned)(n_s - 4);
        src[k] = tr + (in ? ws + 16 * i : -ld_o);
        nb[k] = in ? 16 : 0;
        act[k] = o < len;
      }
      const uint32_t wbi = wb + 64u * i0;
#pragma unroll
      for (int h = 0; h < 8; h += 4)
        asm volatile(
            "{\n .reg .pred q0, q1, q2, q3;\n"
            " setp.ne.b32 q0, %12, 0;\n setp.ne.b32 q1, %13, 0;\n"
            " setp.ne.b32 q2, %14, 0;\n setp.ne.b32 q3, %15, 0;\n"
            " @q0 cp.async.cg.shared.global [%0], [%4], 16, %8;\n"
            " @q1 cp.async.cg.shared.global [%1], [%5], 16, %9;\n"
            " @q2 cp.async.cg.shared.global [%2], [%6], 16, %10;\n"
            " @q3 cp.async.cg.shared.global [%3], [%7], 16, %11;\n}\n" ::"r"(wbi + 64u * h),
            "r"(wbi + 64u * (h + 1)), "r"(wbi + 64u * (h + 2)), "r"(wbi + 64u * (h + 3)),
            "l"(src[h]), "l"(src[h + 1]), "l"(src[h + 2]), "l"(src[h + 3]), "r"(nb[h]),
            "r"(nb[h + 1]), "r"(nb[h + 2]), "r"(nb[h + 3]), "r"(act[h]), "r"(act[h + 1]),
            "r"(act[h + 2]), "r"(act[h + 3])
            : "memory");
    }
    return nullptr;
  };

  // 3-stage cp.async pipeline, one barrier per chunk: at iteration q the
  // barrier both publishes chunk q and retires chunk q-1, whose buffer
  // ((q+2) % 3) is then refilled with chunk q+2.
  Cursor cur{0, 0, 0, 0}, nx2{0, 0, 0, 0};
  int slot_cur = 0, slot_ld = 0, tslot_cur = 0, tslot_ld = 0;  // q, q+2 and their T, mod 3
  auto bump3 = [](int& x) { x = x == 2 ? 0 : x + 1; };
  auto advance = [&](Cursor& cu, int& slot, int& tslot) {
    const int t_prev = cu.T;
    cu.next(n_chunks, n_tx);
    bump3(slot);
    if (cu.T != t_prev) bump3(tslot);
  };
  make_meta(0);
  if (n_T > 1) make_meta(1);
  __syncthreads();
  for (int p = 0; p < 2; ++p) {
    if (p < Q)
      for (int sub = 0; sub < TJC / 32; ++sub)
        issue_loads(slot_ld, tslot_ld, nx2, (tid >> 2) + 32 * sub);
    cp_async_commit();
    advance(nx2, slot_ld, tslot_ld);
  }

  const VT M2 = L::splat(kMagic), NM2 = L::splat(-kMagic);
  const VT ONE2 = L::splat(1.0f), HALF2 = L::splat(0.5f);
  VT acc = L::splat(0.0f);  // +0.0f
  VT txd = acc, t0e2 = acc;

  for (int q = 0; q < Q; ++q) {
    cp_async_wait1();  // this thread's copies of chunk q have landed
    __syncthreads();   // chunk q visible; compute(q-1) retired everywhere
    if (cur.cb == 0 && cur.T + 2 < n_T) {
      make_meta(cur.T + 2);  // ring slot of transmit T-1: retired
      if (n_chunks < 2) __syncthreads();  // first used by this iteration's loads
    }
    const float* keep = nullptr;
    const float* keep2 = nullptr;
    if (q + 2 < Q) {
      keep = issue_loads(slot_ld, tslot_ld, nx2, tid >> 2);
      if (TJC > 32) keep2 = issue_loads(slot_ld, tslot_ld, nx2, (tid >> 2) + 32);
    }
    cp_async_commit();
    advance(nx2, slot_ld, tslot_ld);
    if (cur.cb == 0) {
      if (TXD_SMEM) {
        const u64 tt = txd_s[cur.e * NTH + tid];
        txd = PAIR ? (VT)tt : L::make(lo_f(tt), 0.0f);
      } else if (PW) {
        txd = pw_txd(cur.e);
      } else if (PAIR) {
        if (tm_warp)
          txd = (VT)tm_ld2(tlane + 2 * txe[cur.e]);
        else
          txd = (VT)dsm[txe[cur.e] * 64 + dtid];
      } else {
        txd = L::make(tm_ld1(tlane + txe[cur.e]), 0.0f);
      }
      t0e2 = L::splat(t0s[cur.e]);
    }
    const int* MXc = metaX + tslot_cur * nrp + cur.cb * TJC;
    const int* MKc = metaK + tslot_cur * nrp + cur.cb * TJC;
    const int4* MK4 = reinterpret_cast<const int4*>(MKc);  // 4 gather bases per LDS.128
    const int jn = min(TJC, n_rx - cur.cb * TJC);

    // one channel: rxd = receive delay(s), K = gather address base
    auto channel = [&](VT rxd, uint32_t K) {
      VT t = L::add(txd, rxd);
      if (T0) t = L::sub(t, t0e2);  // all-zero t0 skips it: x - 0 == x exactly
      const VT r = LINEAR ? L::add_rm(t, M2) : L::add_rm(L::add(t, HALF2), M2);
      float rA, rB;
      if (PAIR) {
        unpk((u64)r, rA, rB);
      } else {
        rA = (float)r;
        rB = rA;
      }
      const uint32_t aA = (uint32_t)__float_as_int(rA) * 4u + K;
      const uint32_t aB = (uint32_t)__float_as_int(rB) * 4u + K;
      if (LINEAR) {
        const VT x0 = L::make(lds0(aA), PAIR ? lds0(aB) : 0.0f);
        const VT x1 = L::make(lds1(aA), PAIR ? lds1(aB) : 0.0f);
        const VT fr = L::sub(t, L::add(r, NM2));  // a = t - floor(t)
        const VT om = L::sub(ONE2, fr);           // 1 - a
        acc = L::add(acc, L::mul(om, x0));        // acc = out + (1 - a) * x[k0]
        acc = L::add(acc, L::mul(fr, x1));        // out = acc + a * x[k1]
      } else {
        acc = L::add(acc, L::make(lds0(aA), PAIR ? lds0(aB) : 0.0f));
      }
    };
    if (IDMAP && jn == TJC) {
      // identity map: channels cb*32 .. cb*32+31 are elements of the same
      // index -- tcgen05.ld.x32 fetches 16 delay pairs (PAIR) or 32 delays
      if (PAIR) {
#pragma unroll
        for (int h = 0; h < TJC; h += 16) {
          u64 d[16];
          if (tm_warp) {
            tm_ld32(tlane + 2 * (cur.cb * TJC + h), d);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) d[i] = dsm[(cur.cb * TJC + h + i) * 64 + dtid];
          }
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            const int4 k4 = MK4[(h + i) >> 2];
            channel((VT)d[i], (uint32_t)k4.x);
            channel((VT)d[i + 1], (uint32_t)k4.y);
            channel((VT)d[i + 2], (uint32_t)k4.z);
            channel((VT)d[i + 3], (uint32_t)k4.w);
          }
        }
      } else {
        for (int h = 0; h < TJC; h += 32) {
          float d[32];
          tm_ld32f(tlane + cur.cb * TJC + h, d);
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const int4 k4 = MK4[(h + i) >> 2];
            channel(L::make(d[i], 0.0f), (uint32_t)k4.x);
            channel(L::make(d[i + 1], 0.0f), (uint32_t)k4.y);
            channel(L::make(d[i + 2], 0.0f), (uint32_t)k4.z);
            channel(L::make(d[i + 3], 0.0f), (uint32_t)k4.w);
          }
        }
      }
    } else {
      for (int jj = 0; jj < jn; ++jj) {
        const int2 mm = make_int2(MXc[jj], MKc[jj]);
        const uint32_t col_m = CPE * ((unsigned)mm.x >> 13);
        VT rxd;
        if (!tm_warp)
          rxd = (VT)dsm[((unsigned)mm.x >> 13) * 64 + dtid];
        else
          rxd = PAIR ? (VT)tm_ld2(tlane + col_m) : L::make(tm_ld1(tlane + col_m), 0.0f);
        channel(rxd, (uint32_t)mm.y);
      }
    }

    if (cur.e == n_tx - 1 && cur.cb == n_chunks - 1) {  // frame complete
      const int64_t fo = (int64_t)(f_begin + cur.fl) * a.out_stride;
      if (col < g.n_x) {
        float oA, oB;
        if (PAIR) {
          unpk((u64)acc, oA, oB);
        } else {
          oA = (float)acc;
          oB = 0.0f;
        }
        if (rowA < g.n_z) a.out[fo + (int64_t)rowA * g.n_x + col] = oA;
        if (PAIR && rowB < g.n_z) a.out[fo + (int64_t)rowB * g.n_x + col] = oB;
      }
      acc = L::splat(0.0f);
    }
    advance(cur, slot_cur, tslot_cur);
    asm volatile("" ::"l"(keep), "l"(keep2));
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");

  // ---- release TMEM (the allocating warp)
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  if (warp == 0) tm_dealloc(tbase, (uint32_t)a.tmem_cols);
}

// variant of the TMEM kernel a launch uses
enum TmemVariant { kScalar = 0, kPair = 1, kHybrid = 2 };

static size_t tmem_smem_bytes(const bm_das_geometry& g, int W, int variant, int jc = 32) {
  const int nth = variant == kHybrid ? 192 : 128;
  size_t b = 16 + (size_t)g.n_tx * 16;
  b = ((b + 15) & ~size_t(15)) + (size_t)g.n_elements * 8;
  b = ((b + 15) & ~size_t(15)) + (size_t)((g.n_rx + 3) & ~3) * 24;
  if (g.scheme == BM_PW && variant != kHybrid) b += (size_t)g.n_tx * nth * 8;
  if (variant == kHybrid) b += (size_t)g.n_elements * 64 * 8;
  return b + (size_t)NST * jc * W * 4;
}

static int tmem_cols_for(int n_el, bool pair) {
  int cols = 32;
  while (cols < (pair ? 2 : 1) * n_el) cols *= 2;
  return cols;
}

// BM_DAS_LANES = pair (default) | hybrid | scalar.  Measured on cfg2 (32
// frames): pair 6.37 ms, hybrid 6.68 ms, scalar 7.82 ms.
static int tmem_variant(const bm_das_geometry& g) {
  const char* e = getenv("BM_DAS_LANES");
  const bool pair_ok = 2 * g.n_elements <= 512;
  const bool hyb_ok = 2 * g.n_elements <= 256 && g.window_hint_wide > 0 &&
                      g.window_hint_wide <= 256 &&
                      tmem_smem_bytes(g, g.window_hint_wide, kHybrid) + 1024 <= (227 * 1024) / 2;
  if (e && !strcmp(e, "scalar")) return kScalar;
  if (e && !strcmp(e, "hybrid") && hyb_ok) return kHybrid;
  return pair_ok ? kPair : kScalar;
}

int das_tmem_variant(const bm_das_geometry& g) { return tmem_variant(g); }

int das_tmem_eligible(const bm_das_geometry& g, int64_t rf_stride) {
  if (g.dtype != BM_F32 || !g.uniform || g.window_hint <= 0) return 0;
  if (g.n_samples % 4 != 0 || rf_stride % 4 != 0) return 0;
  if (g.window_hint > 256) return 0;             // loader: <= 16 copies of 16 B per thread
  if (g.n_elements > 512) return 0;              // one TMEM column per element (scalar)
  if (tmem_smem_bytes(g, g.window_hint, tmem_variant(g)) > 110 * 1024) return 0;
  return 1;
}

int das_tmem_launch(const bm_das_geometry& g, const void* rf, int64_t rf_stride, void* out,
                    int64_t out_stride, int n_frames, cudaStream_t s) {
  const int variant = tmem_variant(g);
  const bool pair = variant != kScalar, hyb = variant == kHybrid;
  TmemArgs a{g, (const float*)rf, rf_stride, (float*)out, out_stride, n_frames, 1,
             hyb ? g.window_hint_wide : g.window_hint, tmem_cols_for(g.n_elements, pair), 32};
  const int tz = pair ? 16 : 8, tx = hyb ? 24 : TX, nth = hyb ? 192 : 128;
  const int tiles = ((g.n_z + tz - 1) / tz) * ((g.n_x + tx - 1) / tx);
  // CTAs per SM are limited to what TMEM holds (512 columns): request enough
  // shared memory that no extra CTA is scheduled to spin in tcgen05.alloc
  int per_sm = 512 / a.tmem_cols;
  if (per_sm > 4) per_sm = 4;
  const size_t cap = (size_t)(227 * 1024) / per_sm - 1024;
  // 64-channel chunks halve the per-chunk overhead (cfg2: 5.87 vs 6.30 ms
  // per 32 frames) when their windows still fit the SMEM share of a CTA
  if (variant == kPair && g.n_rx >= 64 && tmem_smem_bytes(g, a.W, variant, 64) <= cap) a.jc = 64;
  size_t smem = tmem_smem_bytes(g, a.W, variant, a.jc);
  if (smem < cap) smem = cap;
  // frames per CTA: amortise the per-CTA delay-table build over a frame
  // group while keeping >= 4 waves of CTAs for load balance
  int fpc = 1;
  while (fpc < 16 && fpc * 2 <= n_frames &&
         (int64_t)tiles * ((n_frames + fpc * 2 - 1) / (fpc * 2)) >= 4LL * per_sm * sm_count())
    fpc *= 2;
  a.frames_per_cta = fpc;
  const bool pw = g.scheme == BM_PW, lin = g.interp == BM_LINEAR;
  typedef void (*kfn)(const TmemArgs);
#define BM_TMEM_ROW(P, H, J)                                                                 \
  das_tmem_kernel<P, false, false, false, false, H, J>,                                     \
      das_tmem_kernel<P, false, false, false, true, H, J>,                                  \
      das_tmem_kernel<P, false, false, true, false, H, J>,                                  \
      das_tmem_kernel<P, false, false, true, true, H, J>,                                   \
      das_tmem_kernel<P, false, true, false, false, H, J>,                                  \
      das_tmem_kernel<P, false, true, false, true, H, J>,                                   \
      das_tmem_kernel<P, false, true, true, false, H, J>,                                   \
      das_tmem_kernel<P, false, true, true, true, H, J>,                                    \
      das_tmem_kernel<P, true, false, false, false, H, J>,                                  \
      das_tmem_kernel<P, true, false, false, true, H, J>,                                   \
      das_tmem_kernel<P, true, false, true, false, H, J>,                                   \
      das_tmem_kernel<P, true, false, true, true, H, J>,                                    \
      das_tmem_kernel<P, true, true, false, false, H, J>,                                   \
      das_tmem_kernel<P, true, true, false, true, H, J>,                                    \
      das_tmem_kernel<P, true, true, true, false, H, J>,                                    \
      das_tmem_kernel<P, true, true, true, true, H, J>
  // rows: scalar/32, pair/32, hybrid/32, pair/64
  static const kfn table[64] = {BM_TMEM_ROW(false, false, 32), BM_TMEM_ROW(true, false, 32),
                                BM_TMEM_ROW(true, true, 32), BM_TMEM_ROW(true, false, 64)};
#undef BM_TMEM_ROW
  const int row = (variant == kPair && a.jc == 64) ? 3 : variant;
  const kfn k = table[16 * row + ((pw ? 8 : 0) | (lin ? 4 : 0) | (g.t0_nonzero ? 2 : 0) |
                                  (g.rx_identity ? 1 : 0))];
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return BM_ERR_CUDA;
  dim3 grid(tiles, (n_frames + fpc - 1) / fpc);
  k<<<grid, nth, smem, s>>>(a);
  return cuda_status();
}

}  // namespace bm
