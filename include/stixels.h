/*
 * stixels.h -- C ABI of the B200-native multi-stixel estimation hot path
 * (Hernandez-Juarez et al., "GPU-accelerated real-time stixel computation",
 * arXiv 1610.04124).  Citations "P:n" are lines of the paper's source
 * (PAPER.md); "L#n" are the readings of DESIGN.md section 3.
 *
 * The library computes, for each frame of a batch of disparity images:
 *   a1/a2  column reduction + transpose
 *   a3     ground-model inputs
 *   a4/a5  per-column prefix sums / object LUT
 *   a6     the Eq. 5-6 min-plus DP
 *   a7     backtracking + stixel extraction
 * entirely in hand-written sm_100a CUDA kernels.  There is no CPU fallback:
 * every entry point that computes fails with STIXELS_ERR_CUDA if the device
 * cannot run the kernels.
 *
 * Conventions
 *  - Rows of a column are counted from the BOTTOM image row (v = 0) upward
 *    ("base (beginning) and top"); image row r = H-1-v (L#12).
 *  - Classes: 0 = ground, 1 = object, 2 = sky (tie order G < O < S, L#17).
 *  - All device pointers are CUDA device memory on the handle's device; all
 *    calls that take device pointers enqueue work on the handle's stream and
 *    return without synchronising (no host<->device copies).
 *  - Handles are bound to one device and one stream, are not thread-safe, and
 *    one handle per GPU / process is the intended use (multi-GPU: one process
 *    per GPU, frames sharded, no collective on the hot path).
 */
#ifndef STIXELS_H_
#define STIXELS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes -------------------------------------------------------- */
#define STIXELS_OK 0
#define STIXELS_ERR_ARG (-1)         /* null pointer or bad dimension / size    */
#define STIXELS_ERR_PARAM (-2)       /* model parameter violates its invariant  */
#define STIXELS_ERR_UNSUPPORTED (-3) /* h, D, shared memory or range limits     */
#define STIXELS_ERR_CUDA (-4)        /* CUDA error (sticky per handle)          */
#define STIXELS_ERR_CAPACITY (-5)    /* a column produced more stixels than the
                                        per-column capacity (impossible with the
                                        default capacity h)                     */

/* ---- input formats ------------------------------------------------------- */
#define STIXELS_U8 0  /* uint8 fixed point, disp_frac_bits fractional bits  */
#define STIXELS_U16 1 /* uint16 fixed point, disp_frac_bits fractional bits */
#define STIXELS_F32 2 /* float32 disparity in pixels; invalid if not finite, negative
                         or >= D (invalid_value and disp_frac_bits unused); a valid
                         value is converted once to 1/256 px, half up (L#28) */

/* ---- column reduction (a2) ---------------------------------------------- */
#define STIXELS_REDUCE_MEAN 0   /* mean of the valid pixels of the s-wide segment */
#define STIXELS_REDUCE_MEDIAN 1 /* their median; mean of the two middle values when the
                                   count is even; same half-up rounding to 1/256 (NEXT
                                   f4, L#24); stixel_width <= 64           */

/* ---- classes ------------------------------------------------------------- */
#define STIXELS_GROUND 0
#define STIXELS_OBJECT 1
#define STIXELS_SKY 2

/*
 * Model and input description.  Everything the paper's problem statement puts
 * in: camera/ground geometry, stixel width s, d_range,
 * and the model's probabilities.
 */
typedef struct stixels_params {
  /* --- geometry ("ground slope and horizon line are assumed known") --- */
  float focal_px;        /* focal length in pixels (used only to derive alpha)   */
  float baseline_m;      /* stereo baseline, metres                               */
  float camera_height_m; /* camera height above the road, metres                  */
  float horizon_row;     /* image row of the horizon (0 = top); fractional, may
                            lie outside the image, must be finite                */
  float principal_row;   /* image row of the principal point                      */
  float ground_slope;    /* alpha of P:79 (disparity per row).  If <= 0 it is
                            derived: alpha = baseline*cos(theta)/camera_height,
                            theta = atan((principal_row-horizon_row)/focal_px)
                            (L#21)                                                */
  /* --- sensor model, Eq. 3-4 ----------------------------------- */
  float p_out;           /* outlier rate, 0 < p_out < 1                           */
  float sigma[3];        /* per-class Gaussian sigma (G, O, S), > 0 (L#2)        */
  float a_norm;          /* A_norm > 0 (L#3)                                      */
  /* --- prior, as probabilities; cost = -ln p, p = 0 forbids (P:65-66, P:120,
         L#1).  Structurally forbidden entries MUST be 0: p_first[SKY]
         (sky cannot be the bottom stixel), p_trans[G][G], p_trans[S][S],
         p_trans[S][G] (ground above sky), p_trans[S][O] (object above sky). -- */
  float p_first[3];      /* first (bottom) stixel of class c                      */
  float p_trans[3][3];   /* [lower class][upper class]                            */
  float p_ord;           /* ordering: upper object nearer than lower + margin     */
  float p_grav;          /* gravity: object nearer than ground at its base        */
  float p_blg;           /* diving: object farther than ground at its base        */
  float p_exist;         /* BIC: per-stixel existence probability                 */
  int32_t ord_margin;    /* disparity margin of the ordering constraint, >= 0     */
  int32_t grav_margin;   /* disparity margin of gravity/diving, >= 0              */
  /* --- sizes ----------------------------------------------------------------- */
  int32_t stixel_width;  /* s >= 1                                          */
  int32_t max_disparity; /* D = d_range, 2 <= D <= 256                     */
  /* --- input encoding (a1) ----------------------------------------------- */
  int32_t disp_format;   /* STIXELS_U8, STIXELS_U16 or STIXELS_F32                */
  int32_t disp_frac_bits;/* Q: fractional bits of the input, 0..8                 */
  uint32_t invalid_value;/* sentinel of an invalid pixel; values decoding to >= D
                            are invalid too (L#23)                                */
  int32_t reduce_mode;   /* STIXELS_REDUCE_MEAN or STIXELS_REDUCE_MEDIAN  */
  /* --- numerics -------------------------------------------------------------- */
  int32_t cost_frac_bits;/* q: costs are integers in units of 2^-q nats ("exact
                            mode", L#22); 0 = continuous fp32 Eq. 4            */
  int32_t max_stixels;   /* per-column output capacity; 0 = h (never overflows)   */
  /* --- NEXT f2: the noise model sigma^c(f, v) of P:108 as tables (host memory,
         read by stixels_create only; NULL = the per-class constant sigma[]) --- */
  const float* sigma_object_f; /* D entries: sigma_O of the object disparity f;
                                  Pair[f][d] becomes a genuine D x D table.
                                  Band (|d - f| with Pair < cap) <= 7: sparse band
                                  rounds; wider: a dense W-row ring over the table */
  const float* sigma_ground_v; /* height entries: sigma_G of model row v; either
                                  table selects the 2-D (PAIR2D) kernels, a missing
                                  sigma_object_f meaning the constant sigma[1]     */
} stixels_params;

/* One output stixel (L#19): rows [bottom, top] (bottom <= top, model
 * rows), class, and disparity (object: its integer mean f; ground: the ground
 * model at `bottom`; sky: 0).  12 bytes. */
typedef struct stixel_t {
  uint16_t bottom;
  uint16_t top;
  uint8_t cls;
  uint8_t pad[3];
  float disparity;
} stixel_t;

typedef struct stixels_handle stixels_handle;

/* Fill *p with the model defaults of DESIGN.md (reading L#1).  Returns OK. */
int stixels_default_params(stixels_params* p);

/*
 * Validate parameters, build the input-independent tables on the host (Eq. 4
 * quantized per class, the D x D object pair-cost LUT of P:175 in its 1-D
 * |f - d| form, per-row ground model and gravity thresholds, prior constants),
 * upload them to `device`, and allocate the workspace for up to `max_batch`
 * frames of width x height.
 *   width >= s, 1 <= height <= 1024, 1 <= max_batch <= 65535.
 *   cuda_stream: a cudaStream_t (NULL = the legacy default stream).
 * On success *out owns all tables and workspace.  Errors: ARG, PARAM,
 * UNSUPPORTED (height, D, shared memory, exact-mode range), CUDA.
 */
int stixels_create(const stixels_params* params, int width, int height, int max_batch,
                   int device, void* cuda_stream, stixels_handle** out);

/* Output sizes: n_cols = floor(width / s), cap = per-column capacity. */
int stixels_query(const stixels_handle* h, int* n_cols, int* cap);

/*
 * The DP kernel variant stixels_create chose for this model (diagnostics and
 * tests).  Any pointer may be NULL.
 *   variant     : STIXELS_DP_DENSE   fp32, dense W-row ring (pair-cost band > 7)
 *                 STIXELS_DP_SPARSE  fp32, sparse band rounds (band <= 7)
 *                 STIXELS_DP_PAIR2D  fp32, sigma_O(f) / sigma_G(v) tables (NEXT f2),
 *                                    sparse band rounds (band <= 7)
 *                 STIXELS_DP_PAIR2D_DENSE  the same, dense ring (band > 7)
 *                 STIXELS_DP_INT32   int32 quanta, atomic band rounds (band <= 3,
 *                                    exact mode: cost_frac_bits > 0)
 *   dp_slots    : object-mean slots per W-row (128 for D <= 128, else 256)
 *   cols_per_cta: column groups per CTA (one CTA per SM) at a full batch
 * Errors: ARG (h NULL).
 */
#define STIXELS_DP_DENSE 0
#define STIXELS_DP_SPARSE 1
#define STIXELS_DP_PAIR2D 2
#define STIXELS_DP_INT32 3
#define STIXELS_DP_PAIR2D_DENSE 4
int stixels_query_kernel(const stixels_handle* h, int* variant, int* dp_slots, int* cols_per_cta);

/*
 * Run the whole hot path on `batch` frames, asynchronously on the handle's stream.
 *   d_disp    : device, [batch][height][row_pitch_bytes], U8/U16 per params.
 *   d_out     : device, [batch][n_cols][cap] stixel_t; entries >= count are
 *               left untouched.  Stixels are ordered bottom -> top and tile
 *               the column [0, height-1].
 *   d_count   : device, [batch][n_cols] int32 stixels per column.
 *   d_col_cost: device, [batch][n_cols] float, the column's minimum total cost
 *               in nats (nullable).
 * 1 <= batch <= max_batch.  A column with more than `cap` stixels writes the
 * first `cap` (bottom-most), stores its true count, and the NEXT call to
 * stixels_sync() reports STIXELS_ERR_CAPACITY.
 */
int stixels_compute(stixels_handle* h, const void* d_disp, int64_t row_pitch_bytes, int batch,
                    stixel_t* d_out, int32_t* d_count, float* d_col_cost);

/*
 * End-to-end variant with HOST buffers (pinned memory recommended): copies the
 * inputs host->device and the outputs device->host in chunks of the workspace
 * batch, overlapping copies with compute on two internal streams (each with its
 * own DP scratch; both start after work already queued on the handle's stream),
 * and synchronises before returning.  Same layouts as stixels_compute; the host
 * row pitch must be a multiple of the pixel size (else ARG).
 */
int stixels_compute_host(stixels_handle* h, const void* h_disp, int64_t row_pitch_bytes,
                         int batch, stixel_t* h_out, int32_t* h_count, float* h_col_cost);

/* Individual stages (for testing and stage timing; same stream semantics):
 *  reduce : d_disp -> d_cols [batch][n_cols][height] uint16 reduced columns in
 *           units of 1/256 disparity (so D <= 256 fits), model row order,
 *           0xFFFF = invalid (a1-a2). */
int stixels_reduce(stixels_handle* h, const void* d_disp, int64_t row_pitch_bytes, int batch,
                   uint16_t* d_cols);
/*  Values are not clamped (L#27: only the object model clamps a
 *  pixel below D - 1/2, so that its rounding indexes the D x D pair LUT of
 *  P:175); the one limit is 0xFFFE (reachable only at D = 256 with 8
 *  fractional input bits), since 0xFFFF marks an invalid value.
 *  solve  : d_cols (as produced by stixels_reduce) -> stixels (a3-a7); a value
 *           >= D * 256 is invalid (L#23). */
int stixels_solve(stixels_handle* h, const uint16_t* d_cols, int batch, stixel_t* d_out,
                  int32_t* d_count, float* d_col_cost);

/* Synchronise the handle's stream; returns CAPACITY if an overflow was
 * recorded since the last sync, CUDA on a CUDA error, else OK. */
int stixels_sync(stixels_handle* h);

/* Number of kernel launches the last compute/solve/reduce call enqueued. */
int stixels_last_launch_count(const stixels_handle* h);

/* Shape of the last DP launch (stixels_compute / stixels_solve /
 * stixels_compute_host), for tests and benchmarks:
 *   warps_per_column: 4 when the batch fills the GPU (4 column groups per SM);
 *                     8 when it has at most 2 columns per SM (e.g. one 1024x440
 *                     frame): the per-column critical path then sets the frame
 *                     latency (BASELINE configs[1]; P:283-287 report per-frame
 *                     rates), so each column gets twice the warps;
 *   cols_per_cta    : column groups per CTA of that launch.
 * Either pointer may be NULL.  Both are 0 before the first launch.
 * Errors: ARG (h NULL). */
int stixels_query_launch(const stixels_handle* h, int* warps_per_column, int* cols_per_cta);

/* Exact chunk bound of the int32 (STIXELS_DP_INT32) DP kernel: the cumulative
 * number of DP cells (bottom x target pairs of 32 x 32 rectangle chunks) that
 * the kernel skipped since the handle was created, because a lower bound on
 * every candidate of the chunk (each pixel costs at least Pair(0); pixels of the
 * rows between the chunk and the target block that no one mean's band can hold
 * cost the outlier cap, Eq. 4 / P:113) exceeded the best candidate already found
 * for every target of the block.  Skipped candidates are strictly worse than the
 * minimum, so costs and stixel lists are unchanged; the count lets a benchmark
 * separate evaluated from algorithmic cells.  Synchronises the handle's streams.
 * Errors: ARG (h or cells NULL), CUDA. */
int stixels_skipped_cells(stixels_handle* h, unsigned long long* cells);

/* The chunk bound for the following calls: 0 = automatic (the default: on for
 * the int32 kernel when the height is >= 320 rows), 1 = off, 2 = on (any height
 * whose per-block tables fit; tests compare both settings bit for bit).
 * Errors: ARG (h NULL or another value), UNSUPPORTED (2 without the int32
 * kernel, or when nb * DP / 8 > height + 2: the P2 table lives in the spare
 * halves of a per-row array). */
int stixels_set_chunk_bound(stixels_handle* h, int mode);

/* Launch plan of the DP kernel for the following calls: 0 = automatic (the
 * default: 8 warps per column when a batch has at most 2 columns per SM, else
 * 4), 4 or 8 = forced (tests cover both plans on every shape; 8 on a full batch
 * is correct but slower).  Errors: ARG (h NULL or another value), UNSUPPORTED
 * (8 when the column's shared memory does not allow it). */
int stixels_set_launch_plan(stixels_handle* h, int warps_per_column);

/* Synchronise and free everything the handle owns.  NULL is a no-op. */
int stixels_destroy(stixels_handle* h);

const char* stixels_error_string(int status);
/* Last error message of a handle (or of the last failed create if h == NULL). */
const char* stixels_last_error(const stixels_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* STIXELS_H_ */
