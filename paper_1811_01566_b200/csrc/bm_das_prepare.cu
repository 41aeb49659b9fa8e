// Host-side preparation of the TMA DAS kernel (bm_das_prepare): the sample
// window a tile can reach, the exact-index range check of the kernel's
// magic-number floor, and the receive-map classification (identity /
// contiguous runs, echopipe's centered_rx_map, types.py:319-333).  Pure host
// code except for reading back the transmit geometry (a few hundred bytes).
#include <algorithm>
#include <cmath>
#include <vector>

#include "bm_common.cuh"

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
  g->tile_ls_nearest = 0;
  g->window_hint_g4_nearest = 0;
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
  int ls_near = 0, w_near = 0;
  if (contig && g->n_elements >= 4) {
    const int force = bm::debug_override(BM_DBG_DAS_TILE);  // override: 1 (64 x 4) .. 4 (8 x 32)
    if (force >= 1 && force <= 4) {
      ls = force;
      wbest = g4_for(ls);
    } else {
      int wc[5] = {0, 0, 0, wbest, 0};
      for (int c : {1, 2, 4}) {
        const int w = wc[c] = g4_for(c);
        if (w * 5 <= wbest * 4 && w < wbest) {
          ls = c;
          wbest = w;
        }
      }
      // nearest interpolation gathers one sample per contribution: a smaller
      // window (more stages) pays at any margin (cfg1: 8 x 32 tiles, W 128 vs
      // 152: 0.65 vs 0.59 of the gather roof; linear 3 % slower there)
      w_near = wbest;
      for (int c : {1, 2, 3, 4})
        if (wc[c] > 0 && wc[c] < w_near) {
          ls_near = c;
          w_near = wc[c];
        }
      if (ls_near == ls) ls_near = 0;
    }
  }
  g->tile_ls = ls;
  if (!(tabs - W + (wbest > W ? wbest : W) < 4194304.0)) return BM_OK;  // outside the exact magic-number range
  if (W_wide > 4096) return BM_OK;
  g->window_hint = W;
  g->window_hint_wide = W_wide;
  if (g->n_elements >= 4) g->window_hint_g4 = wbest;
  if (ls_near) {
    g->tile_ls_nearest = ls_near;
    g->window_hint_g4_nearest = w_near;
  }
  return BM_OK;
}
