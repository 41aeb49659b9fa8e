/*
 * bmode200 -- C ABI of the B200 (sm_100a) B-mode reconstruction hot path.
 *
 * Every entry point is stream-ordered, stateless and re-entrant: it enqueues
 * work on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 * stream) and returns immediately.  No entry point allocates memory; all
 * buffers are caller-owned and device-accessible (device memory, or pinned
 * host memory a kernel may write over the bus -- the display of a host-origin
 * chain); bm_host_upload alone reads a pageable host frame.  Inputs are never
 * written.
 * Return value: BM_OK (0) or a BM_ERR_* code (see bm_error_string()).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/echopipe):
 *   bm_das_beamform        <- _das_kernel(x_pad, tx_rows, te_idx, d_rx, weights,
 *                             rx_map, t0_smp, half, one, nearest, uniform, out)
 *                             beamform.py:122-187, called by das_beamform
 *                             beamform.py:248-296 (which also builds x_pad and
 *                             zeroes `out`, :270-274 -- both folded in here)
 *   bm_das_aperture_span   <- _aperture_span beamform.py:66-81 (the gate half of
 *                             aperture_weight_table :84-109, evaluated in f64)
 *   bm_analytic_signal     <- analytic_signal sigproc.py:48-73
 *   bm_envelope            <- envelope sigproc.py:76-78
 *   bm_dynamic_adjustment  <- dynamic_adjustment sigproc.py:81-97
 *   bm_envelope_peak       <- analytic_signal + envelope + the `e.max()` of
 *                             dynamic_adjustment (sigproc.py:48-90), fused
 *   bm_envelope_display    <- analytic_signal + envelope + dynamic_adjustment
 *                             (sigproc.py:48-97), one fused launch
 *   bm_display             <- the mapping half of dynamic_adjustment
 *                             (sigproc.py:91-97) given the peak
 *   bm_fir_filter          <- fir_filter sigproc.py:36-45 (operator
 *                             `fir_filter`, pipeline.py:96-105)
 *   bm_sliding_moments     <- qus.sliding_moments qus.py:122-158
 *   bm_dense_forward       <- qus.dense_forward qus.py:170-183 (with the
 *                             moments: estimate_hk_map qus.py:186-192)
 *   bm_quantize_u8         <- the pixel mapping of write_pgm formats.py:189-200
 *   bm_simulate_rf         <- simulate_rf environment.py:91-129 (synthetic RF)
 *   bm_host_upload,        <- the x_pad copy of a host frame into the kernel's
 *   bm_stream_write_u32       input (beamform.py:273-274) as an H2D upload the
 *                             DAS launch overlaps (g->tx_ready)
 *
 * ABI 4 (this version): bm_das_geometry gained tx_ready / tx_ready_base,
 * weight_pad, tile_ls_nearest / window_hint_g4_nearest; bm_host_upload and
 * bm_stream_write_u32 are new; BM_DBG_DAS_LATE_PRODUCER joined the debug keys.
 */
#ifndef BMODE200_H
#define BMODE200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BMODE200_ABI_VERSION 4

/* element type of every floating-point buffer of one call */
enum { BM_F32 = 0, BM_F64 = 1 };
/* transmit scheme (types.py:62-92) */
enum { BM_STA = 0, BM_PW = 1 };
/* interpolation (beamform.py:43) */
enum { BM_NEAREST = 0, BM_LINEAR = 1 };
/* receive window (types.py:251-265) */
enum { BM_RECTANGULAR = 0, BM_HANN = 1 };

enum {
  BM_OK = 0,
  BM_ERR_INVALID_ARGUMENT = 1, /* a size/enum/pointer violates the contract */
  BM_ERR_UNSUPPORTED = 2,      /* valid but outside what this build supports */
  BM_ERR_CUDA = 3,             /* CUDA launch/runtime failure */
  BM_ERR_AXIS_TOO_SHORT = 4    /* analytic signal axis length < 2 (sigproc.py:60-61) */
};

/*
 * DAS geometry: the device-side form of echopipe's DasPlan (beamform.py:195-245).
 * Instead of [n_elements, n_px] delay/weight LUTs the plan keeps only the
 * separable inputs; the kernel rebuilds every delay with the reference's
 * exact operation sequence, so the result is bitwise equal to das_beamform.
 *
 * All pointers are DEVICE pointers.
 */
typedef struct bm_das_geometry {
  int32_t dtype;      /* BM_F32 | BM_F64: frame dtype, the arithmetic type   */
  int32_t scheme;     /* BM_STA | BM_PW                                      */
  int32_t interp;     /* BM_NEAREST | BM_LINEAR                              */
  int32_t window;     /* BM_RECTANGULAR | BM_HANN                            */
  int32_t uniform;    /* 1 iff rectangular and f_number == 0 (DasPlan.uniform) */
  int32_t n_tx;       /* acquisitions                                        */
  int32_t n_rx;       /* channels per acquisition                            */
  int32_t n_samples;  /* samples per trace                                   */
  int32_t n_elements; /* probe elements                                      */
  int32_t n_z;        /* image rows (depth)                                  */
  int32_t n_x;        /* image columns (lateral)                             */
  int32_t window_hint; /* set by bm_das_prepare: max samples a 16 x 16-pixel tile's
                          window can span (0 = not prepared -> generic kernel) */
  int32_t t0_nonzero;  /* set by bm_das_prepare: 1 if any fs*t0 != 0 (the fast
                          kernel then keeps the reference's "- t0" rounding step) */
  int32_t rx_identity; /* set by bm_das_prepare: 1 if rx_map[e][j] == j for all e, j */
  int32_t window_hint_wide; /* set by bm_das_prepare: window bound of 16 x 24 tiles */
  int32_t window_hint_g4; /* set by bm_das_prepare: window bound of a 16 x 16 tile
                             over 4 adjacent elements (one TMA box; 0 = unusable) */
  double speed_of_sound;     /* c  (cast to dtype, beamform.py:206)          */
  double sampling_frequency; /* fs (cast to dtype, beamform.py:207)          */
  const double* elem_x;      /* [n_elements] element centres, f64            */
  const double* x_pos;       /* [n_x] grid lateral positions, f64            */
  const double* z_pos;       /* [n_z] grid depths, f64                       */
  const int32_t* tx_elements;/* [n_tx] STA transmit element per acquisition  */
  const void* cos_a;         /* [n_tx] dtype, cos(angle) (PW, beamform.py:190) */
  const void* sin_a;         /* [n_tx] dtype, sin(angle)                     */
  const int32_t* rx_map;     /* [n_tx * n_rx] channel -> element             */
  const void* t0_smp;        /* [n_tx] dtype, fs * t0 (beamform.py:230)      */
  const void* hann;          /* [(n_elements + 1) * n_elements] dtype Hann table
                                (beamform.py:48-63); NULL unless BM_HANN      */
  const int32_t* span;       /* [2 * n_z * n_x] inclusive active span (i0, i1)
                                per pixel, from bm_das_aperture_span; NULL
                                when f_number == 0 (all elements active)      */
  int32_t rx_contig;         /* set by bm_das_prepare: 1 if every acquisition's
                                channels are consecutive elements,
                                rx_map[e][j] == rx_map[e][0] + j (identity maps
                                and echopipe's centered_rx_map, types.py:319-333) */
  int32_t tile_ls;           /* set by bm_das_prepare: TMA-kernel tile shape for
                                contiguous maps, log2 of the lane-block width:
                                3 = 16 x 16 pixels (lane blocks 4 x 8), 2 = 32 x 8,
                                1 = 64 x 4, 4 = 8 x 32; window_hint_g4 is for it */
  const float* rx_table;     /* optional DEVICE table from bm_das_build_table: the
                                receive delays of every tile, read instead of being
                                rebuilt by each CTA (same bits); NULL = rebuild */
  const uint32_t* tx_ready;  /* optional DEVICE counter for a launch that starts while
                                its frame is still being copied in: the launch reads
                                transmit e's RF only after the counter has reached
                                tx_ready_base + e + 1 (compared modulo 2^32), the
                                copy side advancing it behind each landed transmit
                                group with bm_stream_write_u32.  NULL = RF resident */
  uint32_t tx_ready_base;
  const float* weight_pad;   /* optional DEVICE table (f32 Hann + F-number plans): the
                                `hann` rows zero-padded by n_elements on both sides,
                                [n_elements + 1][3 n_elements]; the TMA kernel then
                                reads a pixel's weight of element m at row (span
                                width), column m - i0 + n_elements, without span
                                tests.  NULL = the span tests and `hann` */
  int32_t tile_ls_nearest;   /* set by bm_das_prepare (contiguous maps): the tile shape
                                for nearest-interpolation launches without a delay
                                table when its staged window is smaller than
                                tile_ls's (more pipeline stages pay for nearest's
                                lighter gathers); 0 = tile_ls */
  int32_t window_hint_g4_nearest; /* its 4-channel window bound */
} bm_das_geometry;

/* Per-pixel dynamic-aperture span |x_elem - x| <= z / (2 F), in f64
 * (beamform.py:66-81).  span_out: device int32[2 * n_z * n_x]. */
int bm_das_aperture_span(const bm_das_geometry* g, double f_number, int32_t* span_out,
                         void* stream);

/* Host-side preparation of the fast (shared-memory-staged) DAS path: from
 * HOST copies of the element/grid positions, of fs*t0 (as double) and of the
 * [n_tx * n_rx] receive map, bound
 * the sample window any tile of the fast kernel can touch and check that all
 * delays stay in the exactly-representable range of its index arithmetic.
 * Writes g->window_hint (0 when the fast path does not apply).  Pure host
 * code: no device access, no stream. */
int bm_das_prepare(bm_das_geometry* g, const double* elem_x_host, const double* x_host,
                   const double* z_host, const double* t0_smp_host,
                   const int32_t* rx_map_host);

/* Which DAS kernel bm_das_beamform would run for this geometry and frame
 * stride: 0 generic, 1 shared-memory fast path, 2/3/4 tensor-memory fast path
 * (scalar / pixel pair / hybrid), -1 invalid geometry.  Host only. */
int bm_das_select(const bm_das_geometry* g, int64_t rf_frame_stride);

/* Launch shape of the TMA kernel (bm_das_select == 5) for n_frames frames:
 * shape[6] = {frames per CTA, FP consumer warp groups sharing one TMEM delay
 * table, FT frames per thread, receive channels per pipeline stage, stages,
 * samples per staged window}.  A pass covers FP * FT frames.  Returns 0, or
 * -1 when another kernel would run.  Host only. */
int bm_das_launch_shape(const bm_das_geometry* g, int64_t rf_frame_stride, int32_t n_frames,
                        int32_t* shape);

/* Per-plan receive-delay table of the TMA kernel (the role of DasPlan's
 * d_rx LUT, beamform.py:211-216, in the kernel's tile order): bytes, and the
 * build (stream-ordered, one launch).  A launch with g->rx_table set reads
 * each CTA's 128 pixel pairs x n_elements delays from it instead of
 * evaluating fs*(sqrt(dx^2+z^2)/c) per CTA -- the dominant per-CTA cost of a
 * one-frame launch (f32: n_el x n_px f32 pairs; f64: n_el x n_px f64, the
 * f64 kernel's one pixel per thread; `table` is then a double* cast).  Valid
 * for the geometry (positions, c, fs, tile shape) it was built from.  0 / BM_ERR_UNSUPPORTED when the TMA kernel does not
 * apply. */
int64_t bm_das_table_bytes(const bm_das_geometry* g);
int bm_das_build_table(const bm_das_geometry* g, float* table, void* stream);

/* Delay-and-Sum of n_frames frames.
 *   rf : device dtype[n_frames][n_tx][n_rx][n_samples], frame f at rf + f*rf_frame_stride
 *   out: device dtype[n_frames][n_z][n_x],  frame f at out + f*out_frame_stride
 * Strides are in elements.  Output is fully overwritten (no pre-zeroing needed). */
int bm_das_beamform(const bm_das_geometry* g, const void* rf, int64_t rf_frame_stride,
                    void* out, int64_t out_frame_stride, int32_t n_frames, void* stream);

/* K2 workspace: bytes of caller-owned DEVICE scratch the sigproc op `op`
 * needs for this shape (0 when its lanes fit on chip).  op: 0 analytic signal,
 * 1 envelope + peak, 2 envelope + display.  Lanes of length n run along the
 * middle axis of [outer][n][inner]; for images, outer = frames, n = n_z,
 * inner = n_x.  Host only (reads the device's occupancy limits). */
int64_t bm_sigproc_ws_bytes(int32_t op, int32_t dtype, int64_t outer, int64_t n, int64_t inner);

/* Trace padding for bm_das_beamform: n_traces traces of n_samples samples
 * (row pitch src_pitch elements) copied into rows of dst_samples, the tail
 * zeroed (the TMA kernel needs rows that are a multiple of 16 bytes; zeros
 * past the trace are exactly what the reference's sentinels contribute).
 * Device pointers, stream-ordered DMA, no kernel. */
int bm_pad_traces(int32_t dtype, const void* src, int64_t src_pitch, int64_t n_traces,
                  int64_t n_samples, void* dst, int64_t dst_samples, void* stream);

/* bm_das_beamform over the transmits [e_begin, e_end) only; with accumulate
 * the per-pixel sums continue from the values already in `out` (same f32
 * sums, same e -> j order, so consecutive ranges give bm_das_beamform's bits).
 * Lets a caller start beamforming the first transmits of a frame while the
 * host->device copy of the rest is still in flight. */
int bm_das_beamform_range(const bm_das_geometry* g, const void* rf, int64_t rf_frame_stride,
                          void* out, int64_t out_frame_stride, int32_t n_frames, int32_t e_begin,
                          int32_t e_end, int32_t accumulate, void* stream);

/* Analytic signal along the middle axis of a contiguous [outer, n, inner]
 * real array x; z is complex interleaved (re, im) of the same dtype.  Any
 * n >= 2 (mixed radix, Bluestein for prime factors > 61): ws / ws_bytes as
 * bm_sigproc_ws_bytes(0, ...) says (may be NULL / 0 when that is 0). */
int bm_analytic_signal(int32_t dtype, const void* x, void* z, int64_t outer, int64_t n,
                       int64_t inner, void* ws, int64_t ws_bytes, void* stream);

/* e[i] = |z[i]| for `count` complex elements. */
int bm_envelope(int32_t dtype, const void* z, void* e, int64_t count, void* stream);

/* Fused analytic -> |.| -> per-frame max, along axis 0 of n_frames images
 * [n_z, n_x] (frame f at rf_img + f*n_z*n_x).  env receives the envelope;
 * peak receives, per frame, the max envelope as raw IEEE bits
 * (uint32 for BM_F32, uint64 for BM_F64; NaN wins).  peak is reset by this
 * call.  ws: bm_sigproc_ws_bytes(1, ...). */
int bm_envelope_peak(int32_t dtype, const void* rf_img, void* env, void* peak,
                     int32_t n_frames, int64_t n_z, int64_t n_x, void* ws, int64_t ws_bytes,
                     void* stream);

/* K2 + K3 in one launch: analytic -> |.| -> per-frame max -> display
 * (sigproc.py:48-97) over n_frames images, the envelope kept on chip (a
 * persistent cooperative kernel; frames whose shape it cannot hold run
 * bm_envelope_peak into disp and the display mapping in place).  disp, peak
 * and status as bm_envelope_peak / bm_display.  ws: bm_sigproc_ws_bytes(2,
 * ...), never 0 (per-frame completion counters). */
int bm_envelope_display(int32_t dtype, const void* rf_img, void* disp, void* peak,
                        int32_t* status, int32_t n_frames, int64_t n_z, int64_t n_x,
                        double range_db, void* ws, int64_t ws_bytes, void* stream);

/* e[i] = |x[i]| for `count` real elements (envelope of a real input, np.abs). */
int bm_abs(int32_t dtype, const void* x, void* e, int64_t count, void* stream);

/* Per-frame max of `frame_elems` non-negative values (same peak encoding). */
int bm_frame_peak(int32_t dtype, const void* e, void* peak, int32_t n_frames,
                  int64_t frame_elems, void* stream);

/* disp = clip(20 log10(e / peak) + R, 0, R) / R, 0 where e == 0
 * (sigproc.py:93-96), per frame; status[f] = 1 where peak <= 0 (AllZeroInput,
 * sigproc.py:91-92), else 0.  disp has the dtype of e. */
int bm_display(int32_t dtype, const void* e, const void* peak, void* disp, int32_t* status,
               int32_t n_frames, int64_t frame_elems, double range_db, void* stream);

/* Display of one frame split laterally over n_tiles ranks:
 * tile t starts at tiles + t*tile_stride and holds the envelope of its column
 * slab as [n_z][w_t] followed, in its LAST element, by the slab's peak bits
 * (bm_envelope_peak's encoding); slabs follow an even split of n_x (the first
 * n_x % n_tiles one column wider).  disp [n_z][n_x] is mapped with the max of
 * the tiles' peaks; *status = 1 if that is not > 0 (AllZeroInput). */
int bm_display_tiles(int32_t dtype, const void* tiles, int32_t n_tiles, int64_t tile_stride,
                     int64_t n_z, int64_t n_x, void* disp, int32_t* status, double range_db,
                     void* stream);

/* Finiteness scan of a device frame (RfFrame validation, types.py:41-42):
 * *flag (device int32) = 1 if any value is NaN or +-inf, else 0. */
int bm_check_finite(int32_t dtype, const void* x, int64_t count, int32_t* flag, void* stream);

/* Cross-GPU frame handshakes for the peer-memory (NVLink) column split:
 * bm_signal_flag stores `value` into *flag (possibly a peer GPU's memory) with
 * system-scope release after every earlier operation of `stream`;
 * bm_wait_flags holds `stream` until flags[0 .. n) are all >= value
 * (system-scope acquire).  One tiny kernel each. */
int bm_signal_flag(int32_t* flag, int32_t value, void* stream);
int bm_wait_flags(const int32_t* flags, int32_t n, int32_t value, void* stream);

/* Stream-ordered 32-bit store *addr = value (device memory) performed by the
 * stream's front end once every earlier operation of `stream` -- copies
 * included -- has completed and is visible (cuStreamWriteValue32 with its
 * default memory barrier).  It needs no SM, so it can release a kernel that
 * is already running on another stream and waits on *addr: the RF copy of a
 * host frame advances g->tx_ready with it behind each transmit group while
 * the DAS launch beamforms the groups that have landed. */
int bm_stream_write_u32(uint32_t* addr, uint32_t value, void* stream);

/* Upload of one HOST frame (the RF ingest in front of
 * das_beamform): copies `src` (pageable host memory) into the caller's pinned
 * `staging` buffer and on to the device buffer `dst`, in n_pieces pieces
 * (piece k = bytes [ends[k-1], ends[k]), ends[-1] = 0).  Each piece is
 * copied by the library's host threads (up to 8) with non-temporal stores,
 * so the DMA that follows reads DRAM rather than CPU-dirty cache lines;
 * then its DMA staging -> dst is enqueued on `stream` and, when `counter` is
 * non-NULL, the store *counter = values[k] (bm_stream_write_u32) -- the
 * progress a DAS launch with g->tx_ready waits on.  The DMA of piece k
 * overlaps the host copy of piece k + 1.  Returns once every piece is
 * enqueued; `staging` must stay untouched until `stream` passes the last
 * DMA.  Calls from several host threads are serialised. */
int bm_host_upload(void* dst, const void* src, void* staging, const int64_t* ends,
                   int32_t n_pieces, uint32_t* counter, const uint32_t* values, void* stream);

/* dynamic_adjustment as one call: bm_frame_peak then bm_display. */
int bm_dynamic_adjustment(int32_t dtype, const void* e, void* peak_ws, void* disp,
                          int32_t* status, int32_t n_frames, int64_t frame_elems,
                          double range_db, void* stream);

/* FIR pre-filter  <- sigproc.fir_filter sigproc.py:36-45 (lfilter(h, [1], x)),
 * operator `fir_filter` pipeline.py:96-105.  x, y: [outer][n][inner] device
 * arrays filtered along n; taps: device f64 [n_taps]; arithmetic in f64,
 * y written in out_dtype.  BM_ERR_AXIS_TOO_SHORT if n < 1. */
int bm_fir_filter(int32_t in_dtype, const void* x, int32_t out_dtype, void* y, int64_t outer,
                  int64_t n, int64_t inner, const double* taps, int32_t n_taps, void* stream);

/* Sliding-window moments  <- qus.sliding_moments qus.py:122-158.  img: device
 * [n_rows][n_cols] (f32 or f64, widened to f64); m1/m2/m3: device f64
 * [(n_rows-wh)/sh + 1][(n_cols-ww)/sw + 1], means of x, x^2, x^3. */
int bm_sliding_moments(int32_t dtype, const void* img, int64_t n_rows, int64_t n_cols,
                       int32_t wh, int32_t ww, int32_t sh, int32_t sw, double* m1, double* m2,
                       double* m3, void* stream);

/* Dense homodyned-K model  <- qus.dense_forward qus.py:170-183.  x: device f64
 * [n][in0]; params: device f64, per layer W (out x in, row-major) then b;
 * dims: device int32 [n_layers][3] = {in, out, activation (0 relu, 1 identity,
 * 2 softplus)}; max_width >= every layer width; y: device f64 [n][out_last]. */
int bm_dense_forward(const double* x, int64_t n, const double* params, const int32_t* dims,
                     int32_t n_layers, int32_t max_width, double* y, void* stream);

/* Display -> 8-bit PGM pixels  <- write_pgm formats.py:189-200:
 * out[i] = floor(disp[i] * 255 + 0.5), rounded in the display dtype. */
int bm_quantize_u8(int32_t dtype, const void* disp, uint8_t* out, int64_t count, void* stream);

/* RF simulator  <- environment.simulate_rf environment.py:91-129.  Device
 * arrays: elem_x f64 [n_el]; tx_elements int32 [n_tx] (STA) or cos_a/sin_a
 * f64 [n_tx] (PW, evaluated on the host); rx_map int32 [n_tx][n_rx];
 * t0 f64 [n_tx] seconds; scatterers f64 [n][3] (x, z, amplitude).
 * out: [n_tx][n_rx][n_samples] in out_dtype (f64 sums, one final rounding). */
int bm_simulate_rf(int32_t scheme, int32_t n_tx, int32_t n_rx, int32_t n_samples,
                   const double* elem_x, const int32_t* tx_elements, const double* cos_a,
                   const double* sin_a, const int32_t* rx_map, const double* t0, double c,
                   double fs, double center_frequency, double n_cycles, const double* scatterers,
                   int32_t n_scatterers, int32_t out_dtype, void* out, void* stream);

/* Test and tuning hooks: process-wide, thread-safe integers, 0 = default.
 * They select which kernel / launch shape runs (every variant computes the
 * same bits or the same tolerance class); production callers never set them.
 * The library reads no environment variables. */
enum {
  BM_DBG_DAS_KERNEL = 0,       /* 1: never the TMA kernel (generic kernel)           */
  BM_DBG_DAS_FP = 1,           /* TMA: consumer warp groups per delay table (1 | 2)  */
  BM_DBG_DAS_FT = 2,           /* TMA: frames per thread (1 | 2 | 4)                 */
  BM_DBG_DAS_FPC = 3,          /* TMA: frames per CTA                                */
  BM_DBG_DAS_TJC = 4,          /* TMA: receive channels per stage (32 | 64 | 128)    */
  BM_DBG_DAS_RUNTIME_W = 5,    /* TMA: 1 = runtime window width kernels              */
  BM_DBG_DAS_TILE = 6,         /* bm_das_prepare: tile shape 1..4 (contiguous maps)  */
  BM_DBG_DAS_VERBOSE = 7,      /* TMA: print the launch shape to stderr              */
  BM_DBG_DAS_GENERIC_TZ = 8,   /* generic kernel, f64: tile rows 1 | 2 | 4           */
  BM_DBG_FFT_PATH = 9,         /* analytic signal: 1 lane kernel, 2 global stages,
                                  3 Bluestein (0: register kernel where it applies)  */
  BM_DBG_NO_FUSED_DISPLAY = 10,/* bm_envelope_display: envelope + display launches  */
  BM_DBG_FIR_ONE_OUTPUT = 11,  /* FIR: one output per thread kernel                  */
  BM_DBG_DAS_PREFETCH = 12,    /* TMA: -1 = no L2 prefetch of the next tiles' tables */
  BM_DBG_DAS_LATE_PRODUCER = 13, /* TMA: 1 = the producer waits for the delay table
                                    (pre-v4 order; default: it fills the RF stages
                                    while the consumers build their delays)         */
  BM_DBG_COUNT = 14
};
int bm_debug_set(int32_t key, int32_t value); /* returns the previous value     */
int bm_debug_get(int32_t key);

const char* bm_error_string(int code);
int bm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* BMODE200_H */
