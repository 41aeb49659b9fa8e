// K1 for f64 frames (the reference's oracle precision, and the precision of
// the paper's Titan X runs): the warp-specialised TMA design of
// bm_das_tma.cu with one pixel per thread in double precision.
//
// Same arithmetic as the generic kernel and the reference's f64 das_beamform
// (beamform.py:122-187 with the DasPlan delays of :211-228): every operator
// rounded once (__dadd_rn / __dmul_rn / __dsqrt_rn / __ddiv_rn, no FMA), the
// same e -> j order, floor(t) from one add.rm with M = 1.5 * 2^52 (exact for
// |t| < 2^51; the sample index is the low word of the result).
//
// CTA = 8 consumer warps + 1 producer warp over the f32 kernel's tile (the
// same tile shapes and window bounds, bm_das_prepare): consumer warp w and
// w + 4 own pixels A and B of the f32 kernel's pixel pair, so both read the
// same TMEM lane quarter -- A's f64 delays in columns [0, 2 n_el), B's in
// [2 n_el, 4 n_el) (128 elements fill the 512 columns of an SM).  The
// producer stages each 4-channel group's window with one TMA box {W, 4 traces}
// of f64 samples per 16-channel stage into an mbarrier ring; consumers gather
// with LDS.64 and interpolate.  Frames of a CTA's frame group are passes that
// reuse the delay table.
#include <algorithm>

#include "bm_tma.cuh"

namespace bm {

constexpr int kJ64 = 16;  // receive channels per stage
constexpr int kT64MaxStages = 12;
constexpr double kMagic64 = 6755399441055744.0;  // 1.5 * 2^52

struct Tma64Args {
  bm_das_geometry g;
  double* out;
  int64_t out_stride;
  int n_frames;
  int e_begin, e_end, accumulate;
  int frames_per_cta;
  int W, nst, ls;
};

struct Tma64Layout {  // shared-memory carve (bytes), identical on host and device
  int tmin, rmin, metaK, metaM, txd, win, total;
  __host__ __device__ Tma64Layout(int n_tx, int n_el, int nst, int W, bool pw) {
    tmin = 256;  // [0,16) TMEM base, [16,24) active element span, [64,160) full
                 // barriers, [160,256) empty barriers
    // tmin, tmax (f32), t0 (f64), txe, rxb, cblo, cbhi (int) per transmit
    rmin = (tmin + 8 * n_tx + 8 * n_tx + 16 * n_tx + 15) & ~15;
    metaK = (rmin + 8 * n_el + 15) & ~15;
    metaM = metaK + 4 * kJ64 * nst;
    txd = (metaM + 4 * kJ64 * nst + 15) & ~15;
    win = (txd + (pw ? n_tx * 256 * 8 : 0) + 127) & ~127;
    total = win + nst * kJ64 * W * 8;
  }
};

__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void tm_st_f64(uint32_t taddr, double d) {
  tm_st2(taddr, __int_as_float(__double2loint(d)), __int_as_float(__double2hiint(d)));
}
__device__ __forceinline__ double words_f64(uint32_t lo, uint32_t hi) {
  return __hiloint2double((int)hi, (int)lo);
}

// exact f64 receive delay fs*(sqrt(dx*dx + z*z)/c) of element m (beamform.py:211-216)
__device__ __forceinline__ double rx_delay64(const bm_das_geometry& g, int m, double px,
                                             double pz) {
  using O = R<double>;
  const double dx = g.elem_x[m] - px;
  return O::mul(g.sampling_frequency,
                O::div(O::sqrt(O::add(O::mul(dx, dx), O::mul(pz, pz))), g.speed_of_sound));
}

// f64 plan table: table[tile][m][i], i = consumer thread (i < 128: pixel A of
// pair i, else pixel B of pair i - 128)
__global__ void __launch_bounds__(256) das_table64_kernel(const bm_das_geometry g, int ls,
                                                          double* __restrict__ table) {
  const int i = threadIdx.x;
  const PairPos pp(g, ls, blockIdx.x, i & 127);
  const int row = (i >> 7) ? pp.rowB : pp.rowA;
  const double px = g.x_pos[min(pp.col, g.n_x - 1)], pz = g.z_pos[min(row, g.n_z - 1)];
  double* tb = table + (int64_t)blockIdx.x * g.n_elements * 256 + i;
  for (int m = blockIdx.y; m < g.n_elements; m += gridDim.y)
    tb[(int64_t)m * 256] = rx_delay64(g, m, px, pz);
}

int das_table64_build(const bm_das_geometry& g, double* table, cudaStream_t s) {
  const dim3 grid((unsigned)tma_tiles(g), (unsigned)std::min(g.n_elements, 16));
  das_table64_kernel<<<grid, 256, 0, s>>>(g, tma_ls(g), table);
  return cuda_status();
}

// WM (weighted kernels): the weight mode compiled in -- 1 rectangular with an
// F-number gate, 2 Hann without, 3 Hann with -- or 0, read at run time (as in
// the f32 kernel: the run-time form costs branches and instruction-cache
// misses on every channel)
template <bool PW, bool LINEAR, bool T0, bool IDMAP, bool WT, int WM = 0>
__global__ void __launch_bounds__(288, 1)
    das_tma64_kernel(const __grid_constant__ CUtensorMap rf_map, const Tma64Args a) {
  using O = R<double>;
  constexpr int NTH = 288, NCW = 8, NC = 256;  // threads, consumer warps, consumer threads
  constexpr int G = IDMAP ? 4 : 1;           // traces per TMA box
  constexpr bool SKIP = WT && IDMAP && WM != 2;  // nothing to skip without an F-number
  const bm_das_geometry& g = a.g;
  const int n_el = g.n_elements, n_tx = g.n_tx, n_rx = g.n_rx;
  const int W = a.W, nst = a.nst;
  const Tma64Layout lay(n_tx, n_el, nst, W, PW);
  const int CA = 1 << a.ls, RA = 32 >> a.ls, TZk = 4 * RA, TXk = 2 * CA;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw);
  const uint32_t smem_s = (uint32_t)__cvta_generic_to_shared(smem_raw);
  const uint32_t full_s = smem_s + 64, empty_s = smem_s + 160;  // + 8 * stage
  float* tmin = reinterpret_cast<float*>(smem_raw + lay.tmin);
  float* tmax = tmin + n_tx;
  double* t0v = reinterpret_cast<double*>(tmax + n_tx);
  int* txe = reinterpret_cast<int*>(t0v + n_tx);
  int* rxb = txe + n_tx;
  int* cblo = rxb + n_tx;
  int* cbhi = cblo + n_tx;
  int* espan = reinterpret_cast<int*>(smem_raw + 16);
  float* rmin = reinterpret_cast<float*>(smem_raw + lay.rmin);
  float* rmax = rmin + n_el;
  int* metaK = reinterpret_cast<int*>(smem_raw + lay.metaK);  // [nst][16] gather base
  int* metaM = reinterpret_cast<int*>(smem_raw + lay.metaM);  // [nst][16] element
  double* txd_s = reinterpret_cast<double*>(smem_raw + lay.txd);  // PW: [n_tx][256]
  const uint32_t win_s = smem_s + (uint32_t)lay.win;              // [nst][16 / G][G][W] f64

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool producer = warp == NCW;
  const int half = (warp >> 2) & 1;  // 0: pixel A of the pair, 1: pixel B
  const int ctid = tid & 127, cidx = tid & (NC - 1);
  const int tiles_x = (g.n_x + TXk - 1) / TXk;
  const int tz0 = (blockIdx.x / tiles_x) * TZk, tx0 = (blockIdx.x % tiles_x) * TXk;
  const PairPos pp(g, a.ls, blockIdx.x, ctid);
  const int col = pp.col, row = half ? pp.rowB : pp.rowA;
  const int colc = min(col, g.n_x - 1), rowc = min(row, g.n_z - 1);
  const double c = g.speed_of_sound, fs = g.sampling_frequency;
  const double px = g.x_pos[colc], pz = g.z_pos[rowc];

  if (warp == 0) {
    tm_alloc(smem_s, 512u);
    tm_relinquish();
  }
  if (SKIP && tid == 0) {
    espan[0] = g.span ? n_el : 0;
    espan[1] = g.span ? -1 : n_el - 1;
  }
  if (producer && lane == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(full_s + 8 * s, 32);
      mbar_init(empty_s + 8 * s, NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&rf_map)) : "memory");
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t tlane = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (half ? 2 * n_el : 0);

  int wlo = 0, whi = n_el - 1;
  int i0 = 0, i1 = n_el - 1;  // WT: the pixel's active span
  if (!producer) {
    if (g.rx_table) {
      // the plan's table (bm_das_build_table): [tile][m][256 consumer threads]
      const double* tb = reinterpret_cast<const double*>(g.rx_table) +
                         (int64_t)blockIdx.x * n_el * NC + cidx;
      int m = 0;
      for (; m + 15 < n_el; m += 16) {
        double d[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) d[u] = __ldcs(tb + (int64_t)(m + u) * NC);
#pragma unroll
        for (int u = 0; u < 16; ++u) tm_st_f64(tlane + 2 * (m + u), d[u]);
      }
      for (; m < n_el; ++m) tm_st_f64(tlane + 2 * m, __ldcs(tb + (int64_t)m * NC));
    } else {
      // exact receive delays of the pixel (beamform.py:211-216) -> TMEM
      for (int m = 0; m < n_el; ++m) tm_st_f64(tlane + 2 * m, rx_delay64(g, m, px, pz));
    }
    if (WT && g.span) {
      const int64_t p = (int64_t)rowc * g.n_x + colc;
      i0 = g.span[2 * p];
      i1 = g.span[2 * p + 1];
      const int lo = max(i0 <= i1 ? i0 : n_el, 0), hi = min(i0 <= i1 ? i1 : -1, n_el - 1);
      if (SKIP) {
        if (hi >= 0) {
          atomicMin(&espan[0], lo);
          atomicMax(&espan[1], hi);
        }
        wlo = __reduce_min_sync(0xffffffffu, lo);
        whi = (int)__reduce_max_sync(0xffffffffu, (unsigned)(hi + 1)) - 1;
      }
    }
    tm_wait_st();
  }

  const int zl = min(tz0 + TZk, g.n_z) - 1;
  const double x0 = g.x_pos[tx0], x1 = g.x_pos[min(tx0 + TXk, g.n_x) - 1];
  const double z0 = g.z_pos[tz0], z1 = g.z_pos[zl];
  const double k = g.sampling_frequency / g.speed_of_sound;
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
    t0v[e] = reinterpret_cast<const double*>(g.t0_smp)[e];
    if (!PW) txe[e] = g.tx_elements[e];
    rxb[e] = IDMAP ? g.rx_map[(int64_t)e * n_rx] : 0;
    if (PW) {
      const double ca = reinterpret_cast<const double*>(g.cos_a)[e];
      const double sa = reinterpret_cast<const double*>(g.sin_a)[e];
      const double v00 = z0 * ca + x0 * sa, v01 = z0 * ca + x1 * sa;
      const double v10 = z1 * ca + x0 * sa, v11 = z1 * ca + x1 * sa;
      tmin[e] = (float)(k * fmin(fmin(v00, v01), fmin(v10, v11)));
      tmax[e] = (float)(k * fmax(fmax(v00, v01), fmax(v10, v11)));
    } else {
      rx_bounds(g.tx_elements[e], tmin[e], tmax[e]);
    }
  }
  if (PW && !producer) {
    // exact transmit delays fs*((z cos + x sin)/c) (beamform.py:218-225)
    for (int e = 0; e < n_tx; ++e) {
      const double ca = reinterpret_cast<const double*>(g.cos_a)[e];
      const double sa = reinterpret_cast<const double*>(g.sin_a)[e];
      txd_s[e * NC + cidx] = O::mul(fs, O::div(O::add(O::mul(pz, ca), O::mul(px, sa)), c));
    }
  }
  __syncthreads();

  const double* hglob = reinterpret_cast<const double*>(g.hann);
  const bool hann = WT && (WM ? WM >= 2 : g.window == BM_HANN);
  const bool gated = WM ? WM != 2 : g.span != nullptr;
  const double* hrow =
      hann ? hglob + (int64_t)(gated ? max(0, min(i1 - i0 + 1, n_el)) : n_el) * n_el : nullptr;
  auto weight = [&](int m) -> double {
    if (hann && !gated) return __ldg(hrow + m);
    if (m < i0 || m > i1) return 0.0;
    return hann ? __ldg(hrow + (m - i0)) : 1.0;
  };

  const int n_chunks = (n_rx + kJ64 - 1) / kJ64;
  const int f_begin = blockIdx.y * a.frames_per_cta;
  const int f_count = min(a.frames_per_cta, a.n_frames - f_begin);
  const int e_lo = a.e_begin, e_hi = a.e_end;
  int Q = f_count * (e_hi - e_lo) * n_chunks;
  int e_first = e_lo, e_last = e_hi - 1;
  if (SKIP) {
    const int elo = espan[0], ehi = espan[1];
    for (int e = e_lo + tid; e < e_hi; e += NTH) {
      const int jlo = max(0, elo - rxb[e]), jhi = min(n_rx - 1, ehi - rxb[e]);
      cblo[e] = jlo <= jhi ? jlo / kJ64 : 1;
      cbhi[e] = jlo <= jhi ? jhi / kJ64 : 0;
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
    Q = f_count * tot;
  }
  auto advance = [&](Cursor& cu) {
    if (!SKIP) {
      cu.next(n_chunks, e_lo, e_hi);
      return;
    }
    if (++cu.cb > cbhi[cu.e]) {
      do {
        if (++cu.e == e_hi) {
          cu.e = e_lo;
          ++cu.fl;
        }
      } while (cblo[cu.e] > cbhi[cu.e]);
      cu.cb = cblo[cu.e];
    }
  };
  const Cursor c0{0, e_first, SKIP ? cblo[e_first] : 0, 0};

  if (producer) {
    Cursor cu = c0;
    int s = 0, r = 0;
    int landed = 0;  // transmits known copied in (g.tx_ready launches)
    for (int q = 0; q < Q; ++q) {
      if (r > 0) mbar_wait_sleep(empty_s + 8 * s, (uint32_t)(r - 1) & 1u);
      const int e = cu.e;
      if (g.tx_ready && e >= landed) {
        landed = wait_tx_ready(g.tx_ready, g.tx_ready_base, e + 1);
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      const float lo_e = tmin[e] - (float)t0v[e];
      const int jb = cu.cb * kJ64, jn = min(kJ64, n_rx - jb);
      const int ngr = (jn + G - 1) / G;
      const uint32_t bar = full_s + 8 * s;
      if (lane < ngr) {
        const int jj0 = lane * G;
        int m = (IDMAP ? rxb[e] : 0) + jb + jj0;
        float rlo = rmin[m];
        if (IDMAP) {
#pragma unroll
          for (int i = 1; i < G; ++i)
            if (jj0 + i < jn) rlo = fminf(rlo, rmin[m + i]);
        } else {
          m = g.rx_map[(int64_t)e * n_rx + jb + jj0];
          rlo = rmin[m];
          metaM[s * kJ64 + jj0] = m;
        }
        const int ws = ((int)floorf(lo_e + rlo) - 3) & ~1;
        const uint32_t dst = win_s + (uint32_t)((s * kJ64 + jj0) * W) * 8u;
#pragma unroll
        for (int i = 0; i < G; ++i)  // gather base of each trace: dst - 8 ws (+ row)
          metaK[s * kJ64 + jj0 + i] = (int)(dst + (uint32_t)(i * W) * 8u - (uint32_t)ws * 8u);
        tma_load_3d(dst, &rf_map, ws, e * n_rx + jb + jj0, f_begin + cu.fl, bar);
      }
      if (lane == 0)
        mbar_arrive_tx(bar, (uint32_t)(ngr * G * W * 8));
      else
        mbar_arrive(bar);
      advance(cu);
      if (++s == nst) {
        s = 0;
        ++r;
      }
    }
  } else {
    auto start_acc = [&](int fl) -> double {
      if (a.accumulate && fl < f_count && col < g.n_x && row < g.n_z)
        return a.out[(int64_t)(f_begin + fl) * a.out_stride + (int64_t)row * g.n_x + col];
      return 0.0;
    };
    double acc = start_acc(0);
    double txd = 0.0, t0e = 0.0;
    Cursor cur = c0;
    int s = 0;
    uint32_t ph = 0;
    auto channel = [&](double rxd, double w, uint32_t K) {
      double t = O::add(txd, rxd);
      if (T0) t = O::sub(t, t0e);
      if (LINEAR) {
        const double r = __dadd_rd(t, kMagic64);  // kMagic64 + floor(t)
        const uint32_t ad = K + (uint32_t)__double2loint(r) * 8u;
        const double fr = O::sub(t, O::sub(r, kMagic64));  // a = t - floor(t)
        const double om = O::sub(1.0, fr);
        const double x0v = lds_f64(ad), x1v = lds_f64(ad + 8u);
        if (WT) {
          const double s0 = O::add(acc, O::mul(O::mul(w, om), x0v));
          acc = O::add(s0, O::mul(O::mul(w, fr), x1v));
        } else {
          const double s0 = O::add(acc, O::mul(om, x0v));
          acc = O::add(s0, O::mul(fr, x1v));
        }
      } else {
        const double r = __dadd_rd(O::add(t, 0.5), kMagic64);
        const double xv = lds_f64(K + (uint32_t)__double2loint(r) * 8u);
        acc = O::add(acc, WT ? O::mul(w, xv) : xv);
      }
    };
    for (int q = 0; q < Q; ++q) {
      mbar_wait(full_s + 8 * s, ph);
      if (cur.cb == (SKIP ? cblo[cur.e] : 0)) {  // first stage of a transmit
        if (PW) {
          txd = txd_s[cur.e * NC + cidx];
        } else {
          const u64 v = tm_ld2(tlane + 2 * txe[cur.e]);
          txd = words_f64((uint32_t)v, (uint32_t)(v >> 32));
        }
        t0e = t0v[cur.e];
      }
      const int* MK = metaK + s * kJ64;
      const int jn = min(kJ64, n_rx - cur.cb * kJ64);
      const int m0 = rxb[cur.e] + cur.cb * kJ64;
      if (IDMAP && jn == kJ64 && !(SKIP && (m0 > whi || m0 + 15 < wlo))) {
        // 16 consecutive elements: one tcgen05.ld.x32 of 16 f64 delays
        uint32_t rr[32];
        tm_ld32_issue(tlane + 2 * m0, rr);
        tm_wait_regs(rr);
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
          const int4 k4 = reinterpret_cast<const int4*>(MK)[i >> 2];
          channel(words_f64(rr[2 * i], rr[2 * i + 1]), WT ? weight(m0 + i) : 1.0, (uint32_t)k4.x);
          channel(words_f64(rr[2 * i + 2], rr[2 * i + 3]), WT ? weight(m0 + i + 1) : 1.0,
                  (uint32_t)k4.y);
          channel(words_f64(rr[2 * i + 4], rr[2 * i + 5]), WT ? weight(m0 + i + 2) : 1.0,
                  (uint32_t)k4.z);
          channel(words_f64(rr[2 * i + 6], rr[2 * i + 7]), WT ? weight(m0 + i + 3) : 1.0,
                  (uint32_t)k4.w);
        }
      } else if (!(SKIP && (m0 > whi || m0 + jn - 1 < wlo))) {
        for (int jj = 0; jj < jn; ++jj) {
          const int m = IDMAP ? m0 + jj : metaM[s * kJ64 + jj];
          const u64 v = tm_ld2(tlane + 2 * m);
          channel(words_f64((uint32_t)v, (uint32_t)(v >> 32)), WT ? weight(m) : 1.0,
                  (uint32_t)MK[jj]);
        }
      }
      asm volatile("" ::"d"(acc));
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_s + 8 * s);
      if (cur.e == e_last && cur.cb == (SKIP ? cbhi[e_last] : n_chunks - 1)) {  // frame done
        if (col < g.n_x && row < g.n_z && cur.fl < f_count)
          a.out[(int64_t)(f_begin + cur.fl) * a.out_stride + (int64_t)row * g.n_x + col] = acc;
        acc = start_acc(cur.fl + 1);
      }
      advance(cur);
      if (++s == nst) {
        s = 0;
        ph ^= 1;
      }
    }
  }

  tm_fence_before();
  __syncthreads();
  tm_fence_after();
  if (warp == 0) tm_dealloc(tbase, 512u);
}

// ---------------------------------------------------------------- host side
static size_t tma64_cap() { return (size_t)(227 * 1024) - 1024; }

static int tma64_stages(const bm_das_geometry& g, int W) {
  int n = kT64MaxStages;
  while (n >= 2 && (size_t)Tma64Layout(g.n_tx, g.n_elements, n, W, g.scheme == BM_PW).total >
                       tma64_cap())
    --n;
  return n;
}

int das_tma64_eligible(const bm_das_geometry& g, int64_t rf_stride) {
  if (g.dtype != BM_F64 || g.window_hint <= 0) return 0;
  if (g.rx_contig && g.window_hint_g4 <= 0) return 0;
  const int W = tma_window(g);
  if (W > 256 || 4 * g.n_elements > 512) return 0;
  if (!g.uniform && g.window == BM_HANN && !g.hann) return 0;
  if (g.n_samples % 2 != 0 || rf_stride % 2 != 0) return 0;  // 16-B TMA row strides
  if ((int64_t)g.n_tx * g.n_rx > 0x7fffffffLL) return 0;
  if (tma64_stages(g, W) < 2) return 0;
  return encode_tiled() != nullptr;
}

static int tma64_fpc(const bm_das_geometry& g, int n_frames) {
  const int tiles = tma_tiles(g);
  int fpc = 1;
  while (fpc < 16 && fpc * 2 <= n_frames &&
         (int64_t)tiles * ((n_frames + fpc * 2 - 1) / (fpc * 2)) >= 4LL * sm_count())
    fpc *= 2;
  if (const int want = debug_override(BM_DBG_DAS_FPC); want >= 1)
    fpc = want < n_frames ? want : n_frames;
  return fpc;
}

int das_tma64_shape(const bm_das_geometry& g, int n_frames, int32_t* shape) {
  if (n_frames < 1) return -1;
  const int W = tma_window(g);
  shape[0] = tma64_fpc(g, n_frames);
  shape[1] = 1;
  shape[2] = 1;
  shape[3] = kJ64;
  shape[4] = tma64_stages(g, W);
  shape[5] = W;
  return 0;
}

int das_tma64_launch(const bm_das_geometry& g, const void* rf, int64_t rf_stride, void* out,
                     int64_t out_stride, int n_frames, int e_begin, int e_end, int accumulate,
                     cudaStream_t s) {
  if (((uintptr_t)rf & 15) != 0) return -1;
  const int W = tma_window(g), nst = tma64_stages(g, W), fpc = tma64_fpc(g, n_frames);
  const size_t smem = tma64_cap();
  CUtensorMap map;
  const int64_t fstride = n_frames > 1 ? rf_stride : (int64_t)g.n_tx * g.n_rx * g.n_samples;
  cuuint64_t dims[3] = {(cuuint64_t)g.n_samples, (cuuint64_t)g.n_tx * g.n_rx,
                        (cuuint64_t)n_frames};
  cuuint64_t strides[2] = {(cuuint64_t)g.n_samples * 8, (cuuint64_t)fstride * 8};
  cuuint32_t box[3] = {(cuuint32_t)W, g.rx_contig ? 4u : 1u, 1u};
  cuuint32_t estr[3] = {1, 1, 1};
  if (encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(rf), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -1;
  Tma64Args a{g,     (double*)out, out_stride, n_frames, e_begin, e_end, accumulate,
              fpc,   W,            nst,        tma_ls(g)};
  typedef void (*kfn)(const CUtensorMap, const Tma64Args);
#define BM_T64(WT)                                                                        \
  das_tma64_kernel<false, false, false, false, WT>, das_tma64_kernel<false, false, false, true, WT>, \
      das_tma64_kernel<false, false, true, false, WT>,                                      \
      das_tma64_kernel<false, false, true, true, WT>,                                       \
      das_tma64_kernel<false, true, false, false, WT>,                                      \
      das_tma64_kernel<false, true, false, true, WT>,                                       \
      das_tma64_kernel<false, true, true, false, WT>,                                       \
      das_tma64_kernel<false, true, true, true, WT>,                                        \
      das_tma64_kernel<true, false, false, false, WT>,                                      \
      das_tma64_kernel<true, false, false, true, WT>,                                       \
      das_tma64_kernel<true, false, true, false, WT>,                                       \
      das_tma64_kernel<true, false, true, true, WT>,                                        \
      das_tma64_kernel<true, true, false, false, WT>,                                       \
      das_tma64_kernel<true, true, false, true, WT>,                                        \
      das_tma64_kernel<true, true, true, false, WT>, das_tma64_kernel<true, true, true, true, WT>
  static const kfn table[32] = {BM_T64(false), BM_T64(true)};
#undef BM_T64
  kfn k = table[(g.uniform ? 0 : 16) + (g.scheme == BM_PW ? 8 : 0) +
                (g.interp == BM_LINEAR ? 4 : 0) + (g.t0_nonzero ? 2 : 0) + (g.rx_contig ? 1 : 0)];
  if (!g.uniform && g.rx_contig && !g.t0_nonzero) {
    // weighted, contiguous maps, no t0: the weight mode compiled in
#define BM_T64W(M)                                                                          \
  das_tma64_kernel<false, false, false, true, true, M>,                                     \
      das_tma64_kernel<false, true, false, true, true, M>,                                  \
      das_tma64_kernel<true, false, false, true, true, M>,                                  \
      das_tma64_kernel<true, true, false, true, true, M>
    static const kfn tablew[12] = {BM_T64W(1), BM_T64W(2), BM_T64W(3)};
#undef BM_T64W
    const int wm = g.window == BM_HANN ? (g.span ? 3 : 2) : 1;
    k = tablew[(wm - 1) * 4 + (g.scheme == BM_PW ? 2 : 0) + (g.interp == BM_LINEAR ? 1 : 0)];
  }
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return BM_ERR_CUDA;
  dim3 grid(tma_tiles(g), (n_frames + fpc - 1) / fpc);
  k<<<grid, 288, smem, s>>>(map, a);
  return cuda_status();
}

}  // namespace bm
