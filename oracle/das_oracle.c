/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the DAS hot path.
 *
 * Plain-C restatement of echopipe's numba kernel `_das_kernel`
 * (/root/reference/pkg/src/echopipe/beamform.py:122-187).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library; the product path (paper_1811_01566_b200) never does.
 *
 * Semantics mirrored line by line (beamform.py file:line):
 *   - x_pad carries one zero sentinel sample at each end of every trace
 *     (:127-137, filled by das_beamform :273-274); out-of-range indices clamp
 *     onto a sentinel and add an exact zero.
 *   - per pixel p, ascending e (:146) then ascending j (:149):
 *       t  = (tx_row[p] + d_row[p]) - t0e                       (:156, :171)
 *     nearest (:154-166):  k = clamp(floor(t + 0.5), -1, n_s) + 1
 *                          out += x[k]            (uniform)
 *                          out += w * x[k]        (weighted)
 *     linear (:167-187):   k0f = floor(t); a = t - k0f
 *                          k0 = clamp(k0f, -1, n_s) + 1; k1 = clamp(k0f + 1, -1, n_s) + 1
 *                          acc = out + (1 - a) * x[k0];  out = acc + a * x[k1]       (uniform)
 *                          acc = out + (w*(1 - a)) * x[k0]; out = acc + (w*a) * x[k1] (weighted)
 *   - one IEEE rounding per operator, no FMA contraction (numba compiles the
 *     kernel without fastmath; the Makefile passes -ffp-contract=off).
 *
 * Parallelism: pthreads over 4096-pixel blocks (static round-robin).  Each
 * pixel is owned by exactly one thread and keeps the fixed (e, j) order, so
 * the bits are independent of the thread count (same argument as
 * beamform.py:1-11).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <unistd.h>

#define BLOCK 4096

typedef struct {
  const void *x_pad, *tx_rows, *d_rx, *weights, *t0_smp;
  const int64_t *te_idx, *rx_map;
  void* out;
  int nearest, uniform;
  int64_t n_tx, n_rx, n_samples, n_px;
  int tid, n_threads;
} job_t;

#define DEFINE_WORKER(NAME, T, FLOOR)                                            \
  static void* NAME(void* arg) {                                                 \
    const job_t* a = (const job_t*)arg;                                          \
    const T* x_pad = (const T*)a->x_pad;                                         \
    const T* tx_rows = (const T*)a->tx_rows;                                     \
    const T* d_rx = (const T*)a->d_rx;                                           \
    const T* weights = (const T*)a->weights;                                     \
    const T* t0_smp = (const T*)a->t0_smp;                                       \
    T* out = (T*)a->out;                                                         \
    const int64_t n_px = a->n_px, n_tx = a->n_tx, n_rx = a->n_rx;                \
    const int64_t ns_pad = a->n_samples + 2;                                     \
    const T one = (T)1.0, half = (T)0.5;                                         \
    const T lo = -one, hi = (T)a->n_samples;                                     \
    const int64_t n_blocks = (n_px + BLOCK - 1) / BLOCK;                         \
    for (int64_t b = a->tid; b < n_blocks; b += a->n_threads) {                  \
      const int64_t p_lo = b * BLOCK;                                            \
      const int64_t p_hi = (p_lo + BLOCK < n_px) ? p_lo + BLOCK : n_px;          \
      for (int64_t p = p_lo; p < p_hi; ++p) out[p] = (T)0.0;                     \
      for (int64_t e = 0; e < n_tx; ++e) {                                       \
        const T* tx_row = tx_rows + a->te_idx[e] * n_px;                         \
        const T t0e = t0_smp[e];                                                 \
        for (int64_t j = 0; j < n_rx; ++j) {                                     \
          const int64_t m = a->rx_map[e * n_rx + j];                             \
          const T* d_row = d_rx + m * n_px;                                      \
          const T* w_row = weights + m * n_px;                                   \
          const T* x_row = x_pad + (e * n_rx + j) * ns_pad;                      \
          for (int64_t p = p_lo; p < p_hi; ++p) {                                \
            const T t = (tx_row[p] + d_row[p]) - t0e;                            \
            if (a->nearest) {                                                    \
              T kf = FLOOR(t + half);                                            \
              kf = kf < lo ? lo : kf;                                            \
              kf = kf > hi ? hi : kf;                                            \
              const int64_t k0 = (int64_t)(kf + one);                           \
              if (a->uniform) out[p] += x_row[k0];                               \
              else out[p] += w_row[p] * x_row[k0];                               \
            } else {                                                             \
              const T k0f = FLOOR(t);                                            \
              const T fr = t - k0f;                                              \
              T c0 = k0f < lo ? lo : k0f;                                        \
              c0 = c0 > hi ? hi : c0;                                            \
              T c1 = k0f + one;                                                  \
              c1 = c1 < lo ? lo : c1;                                            \
              c1 = c1 > hi ? hi : c1;                                            \
              const int64_t k0 = (int64_t)(c0 + one);                           \
              const int64_t k1 = (int64_t)(c1 + one);                           \
              if (a->uniform) {                                                  \
                const T acc = out[p] + (one - fr) * x_row[k0];                   \
                out[p] = acc + fr * x_row[k1];                                   \
              } else {                                                           \
                const T w = w_row[p];                                            \
                const T acc = out[p] + (w * (one - fr)) * x_row[k0];             \
                out[p] = acc + (w * fr) * x_row[k1];                             \
              }                                                                  \
            }                                                                    \
          }                                                                      \
        }                                                                        \
      }                                                                          \
    }                                                                            \
    return 0;                                                                    \
  }

DEFINE_WORKER(worker_f32, float, floorf)
DEFINE_WORKER(worker_f64, double, floor)

static void run(void* (*worker)(void*), job_t base, int n_threads) {
  if (n_threads < 1) n_threads = 1;
  if (n_threads > 512) n_threads = 512;
  pthread_t th[512];
  job_t jobs[512];
  for (int i = 0; i < n_threads; ++i) {
    jobs[i] = base;
    jobs[i].tid = i;
    jobs[i].n_threads = n_threads;
  }
  int started = 0;
  for (int i = 1; i < n_threads; ++i)
    if (pthread_create(&th[i], 0, worker, &jobs[i]) == 0) started = i;
    else break;
  if (started < n_threads - 1) { /* could not spawn all: fall back to serial */
    for (int i = 1; i <= started; ++i) pthread_join(th[i], 0);
    jobs[0].tid = 0;
    jobs[0].n_threads = 1;
    worker(&jobs[0]);
    return;
  }
  worker(&jobs[0]);
  for (int i = 1; i < n_threads; ++i) pthread_join(th[i], 0);
}

/* Argument order follows _das_kernel(x_pad, tx_rows, te_idx, d_rx, weights,
 * rx_map, t0_smp, half, one, nearest, uniform, out) (beamform.py:122-126);
 * half/one are implied by the dtype, sizes are explicit. */
#define DEFINE_ENTRY(NAME, T, WORKER)                                            \
  void NAME(const T* x_pad, const T* tx_rows, const int64_t* te_idx,             \
            const T* d_rx, const T* weights, const int64_t* rx_map,              \
            const T* t0_smp, int nearest, int uniform, T* out, int64_t n_tx,     \
            int64_t n_rx, int64_t n_samples, int64_t n_px, int n_threads) {      \
    job_t j = {x_pad, tx_rows, d_rx, weights, t0_smp, te_idx, rx_map, out,       \
               nearest, uniform, n_tx, n_rx, n_samples, n_px, 0, 1};             \
    run(WORKER, j, n_threads);                                                   \
  }

DEFINE_ENTRY(das_oracle_f32, float, worker_f32)
DEFINE_ENTRY(das_oracle_f64, double, worker_f64)

int das_oracle_max_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n < 1 ? 1 : (int)n;
}
