// On-device RF simulator: environment.simulate_rf
// (environment.py:91-129) -- the synthetic cine source of the benchmarks.
//
// Sample k of acquisition e records time k/fs + t0_e; scatterer s adds
//   amp_s * p((k/fs + t0_e) - tau_s),   p(t) = cos(2 pi fc t) * 0.5 (1 + cos(2 pi t / T))
// for |t| <= T/2 and the `span` samples from k0 = ceil((tau - T/2 - t0) fs),
// tau = (d_tx + d_rx) / c the exact two-way flight time.  Everything is f64
// with the reference's operation order; sums run over scatterers in order,
// as np.add.at applies them.  Only cos() differs from the host's libm (CUDA's
// f64 cos is within 2 ulp; the plane-wave angles' cos/sin come from the host),
// so f64 frames agree to ~1e-16 relative and f32
// frames -- one rounding of that -- agree bit for bit except with
// probability ~1e-8 per sample.
//
// One CTA per trace (e, j): the CTA computes every scatterer's (tau, k0) into
// shared memory (256 at a time), then each thread sums its samples.
#include "bm_common.cuh"

namespace bm {

constexpr int kSimThreads = 256, kSimPerThread = 16;  // samples per thread kept in registers

struct SimArgs {
  int scheme, n_tx, n_rx, n_s, n_scat;
  double c, fs, fc, T, half, two_pi_fc, two_pi;
  int span;
  const double* elem_x;      // [n_el]
  const int32_t* tx_el;      // STA: [n_tx]
  const double* cos_a;       // PW: [n_tx] cos(angle), evaluated on the host (math.cos)
  const double* sin_a;       // PW: [n_tx] sin(angle)
  const int32_t* rx_map;     // [n_tx][n_rx] element of each channel
  const double* t0;          // [n_tx] seconds
  const double* scat;        // [n_scat][3] x, z, amplitude
};

__device__ __forceinline__ double pulse(const SimArgs& a, double t) {
  if (!(fabs(t) <= a.half)) return 0.0;
  const double carrier = cos(__dmul_rn(a.two_pi_fc, t));
  const double window = __dmul_rn(0.5, __dadd_rn(1.0, cos(__ddiv_rn(__dmul_rn(a.two_pi, t), a.T))));
  return __dmul_rn(carrier, window);
}

template <typename TO>
__global__ void __launch_bounds__(kSimThreads) sim_kernel(const SimArgs a, TO* __restrict__ out,
                                                          int64_t chunk0) {
  __shared__ double s_tau[kSimThreads], s_amp[kSimThreads];
  __shared__ long long s_k0[kSimThreads];
  const int64_t trace = (int64_t)blockIdx.x;
  const int e = (int)(trace / a.n_rx), j = (int)(trace % a.n_rx);
  const int m = a.rx_map[(int64_t)e * a.n_rx + j];
  const double rx_x = a.elem_x[m];
  const double t0 = a.t0[e];
  const int64_t kbase = chunk0 + (int64_t)threadIdx.x * kSimPerThread;
  double acc[kSimPerThread];
#pragma unroll
  for (int q = 0; q < kSimPerThread; ++q) acc[q] = 0.0;
  for (int s0 = 0; s0 < a.n_scat; s0 += kSimThreads) {
    const int s = s0 + threadIdx.x;
    if (s < a.n_scat) {
      const double x = a.scat[3 * s], z = a.scat[3 * s + 1];
      const double dxr = __dsub_rn(x, rx_x);
      const double d_rx = __dsqrt_rn(__dadd_rn(__dmul_rn(dxr, dxr), __dmul_rn(z, z)));
      double d_tx;
      if (a.scheme == BM_PW) {
        d_tx = __dadd_rn(__dmul_rn(z, a.cos_a[e]), __dmul_rn(x, a.sin_a[e]));
      } else {
        const double dxt = __dsub_rn(x, a.elem_x[a.tx_el[e]]);
        d_tx = __dsqrt_rn(__dadd_rn(__dmul_rn(dxt, dxt), __dmul_rn(z, z)));
      }
      const double tau = __ddiv_rn(__dadd_rn(d_tx, d_rx), a.c);
      s_tau[threadIdx.x] = tau;
      s_k0[threadIdx.x] = (long long)ceil(__dmul_rn(__dsub_rn(__dsub_rn(tau, a.half), t0), a.fs));
      s_amp[threadIdx.x] = a.scat[3 * s + 2];
    }
    __syncthreads();
    const int ns = min(kSimThreads, a.n_scat - s0);
    for (int i = 0; i < ns; ++i) {
      const long long k0 = s_k0[i];
      const long long first = k0 > kbase ? k0 : kbase;
      const long long last = min(k0 + a.span, (long long)(kbase + kSimPerThread));
      if (first >= last) continue;  // no sample of this thread in the burst
      const double tau = s_tau[i], amp = s_amp[i];
#pragma unroll
      for (int q = 0; q < kSimPerThread; ++q) {
        const long long k = kbase + q;
        if (k >= first && k < last) {
          const double t = __dsub_rn(__dadd_rn(__ddiv_rn((double)k, a.fs), t0), tau);
          acc[q] = __dadd_rn(acc[q], __dmul_rn(amp, pulse(a, t)));
        }
      }
    }
    __syncthreads();
  }
  TO* o = out + trace * (int64_t)a.n_s;
#pragma unroll
  for (int q = 0; q < kSimPerThread; ++q) {
    const int64_t k = kbase + q;
    if (k < a.n_s) o[k] = (TO)acc[q];
  }
}

}  // namespace bm

extern "C" int bm_simulate_rf(int32_t scheme, int32_t n_tx, int32_t n_rx, int32_t n_samples,
                              const double* elem_x, const int32_t* tx_elements,
                              const double* cos_a, const double* sin_a, const int32_t* rx_map,
                              const double* t0,
                              double c, double fs, double center_frequency, double n_cycles,
                              const double* scatterers, int32_t n_scatterers, int32_t out_dtype,
                              void* out, void* stream) {
  using namespace bm;
  if (n_tx < 1 || n_rx < 1 || n_samples < 1 || n_scatterers < 0 || !elem_x || !rx_map || !t0 ||
      !out || (n_scatterers > 0 && !scatterers))
    return BM_ERR_INVALID_ARGUMENT;
  if ((scheme == BM_PW && (!cos_a || !sin_a)) || (scheme == BM_STA && !tx_elements) ||
      (scheme != BM_PW && scheme != BM_STA))
    return BM_ERR_INVALID_ARGUMENT;
  if (!(c > 0) || !(fs > 0) || !(center_frequency > 0) || !(n_cycles > 0))
    return BM_ERR_INVALID_ARGUMENT;
  if (out_dtype != BM_F32 && out_dtype != BM_F64) return BM_ERR_INVALID_ARGUMENT;
  SimArgs a;
  a.scheme = scheme;
  a.n_tx = n_tx;
  a.n_rx = n_rx;
  a.n_s = n_samples;
  a.n_scat = n_scatterers;
  a.c = c;
  a.fs = fs;
  a.fc = center_frequency;
  a.T = n_cycles / center_frequency;           // burst_duration
  a.half = a.T / 2.0;
  a.two_pi = 2.0 * 3.141592653589793;          // 2.0 * np.pi
  a.two_pi_fc = a.two_pi * center_frequency;   // (2.0 * np.pi) * fc
  a.span = (int)floor(a.T * fs) + 2;
  a.elem_x = elem_x;
  a.tx_el = tx_elements;
  a.cos_a = cos_a;
  a.sin_a = sin_a;
  a.rx_map = rx_map;
  a.t0 = t0;
  a.scat = scatterers;
  const int64_t traces = (int64_t)n_tx * n_rx;
  if (traces > 0x7fffffffLL) return BM_ERR_UNSUPPORTED;
  cudaStream_t s = (cudaStream_t)stream;
  for (int64_t k0 = 0; k0 < n_samples; k0 += (int64_t)kSimThreads * kSimPerThread) {
    // each launch covers 4096 samples of every trace
    if (out_dtype == BM_F32)
      sim_kernel<float><<<(unsigned)traces, kSimThreads, 0, s>>>(a, (float*)out, k0);
    else
      sim_kernel<double><<<(unsigned)traces, kSimThreads, 0, s>>>(a, (double*)out, k0);
  }
  return cuda_status();
}
