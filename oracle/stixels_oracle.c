/*
 * stixels_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity oracle).
 *
 * A plain, slow, obviously-correct CPU implementation (double precision) of the
 * multi-stixel estimation hot path of Hernandez-Juarez et al., "GPU-accelerated
 * real-time stixel computation" (arXiv 1610.04124).  Citations "P:n" are lines of
 * /root/reference/PAPER.md; "S:n" lines of SPEC.md; "L#n" the readings ledger in
 * DESIGN.md section 3 (= SURVEY.md section 8(c) ledger).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  It shares no code, header, table or
 * constant generator with the CUDA product path (paper_1610_04124_b200/csrc);
 * every formula below is written out independently from the paper.
 *
 * Pins (tests/test_oracle_*.py): Eq. 4 closed forms, reduction
 * examples, prefix == direct summation, brute-force enumeration of
 * every labelled segmentation for h <= 8, textbook optimal partitioning for the
 * object-only special case, h = 1 and on-ground-model closed forms, invariants,
 * synthetic-scene recovery, the prior reading against hand-computed quanta of
 * every branch (tests/golden/prior_reading.json: BIC, gravity / diving at their
 * exact boundaries, the ordering direction, forbidden pairs), and the Eq. 6
 * greedy-predecessor recurrence against an independent plain-Python statement
 * (tests/eq6_plain.py).  The numeric VALUES of the prior probabilities are a
 * reading (L#1: the paper defers them to [PfeifferThesis]); their
 * structure is pinned by the golden file.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_G 0
#define ORC_O 1
#define ORC_S 2
#define ORC_START 3

/* Model description, in the paper's terms (double precision). */
typedef struct {
  int h;              /* column height (rows of the reduced image) */
  int D;              /* d_range: number of disparities */
  int R_bits;         /* reduced disparities are integers in units of 1/2^R_bits (L#8) */
  int q;              /* cost quantum 2^-q nats; 0 = continuous Eq. 4 (L#22) */
  double p_out;       /* outlier rate, Eq. 3 */
  double a_norm;      /* A_norm, Eq. 3 (L#3) */
  double sigma[3];    /* per-class sigma (L#2), index G,O,S */
  double p_first[3];  /* prior of the first (bottom) stixel, Eq. 5 */
  double p_trans[3][3]; /* [lower class][upper class] (L#16) */
  double p_ord, p_grav, p_blg, p_exist; /* ordering, gravity, below-ground, BIC */
  int ord_margin, grav_margin;          /* disparity margins (L#1) */
  double alpha;       /* ground slope (disparity per row) */
  double horizon_row; /* image row of the horizon (0 = top) */
  /* NEXT f2: the noise model sigma^c(f, v) of Eq. 4 as tables, NULL =
   * the per-class constant above (L#2): sigma_O of the object's disparity f
   * (D entries) and sigma_G of the model row v (h entries). */
  const double* sigma_o_f;
  const double* sigma_g_v;
} orc_model;

typedef struct {
  int vb, vt, cls;
  double disp;
} orc_stixel;

/* --------------------------------------------------------------------------
 * Camera -> ground slope ("ground slope and horizon line are assumed to be
 * known"; L#21 reading).  If ground_slope > 0 it is used as given.
 * ------------------------------------------------------------------------ */
double orc_alpha(double focal_px, double baseline_m, double camera_height_m,
                 double horizon_row, double principal_row, double ground_slope) {
  if (ground_slope > 0.0) return ground_slope;
  double theta = atan((principal_row - horizon_row) / focal_px);
  return baseline_m * cos(theta) / camera_height_m;
}

/* Quantization of a cost in nats to an integer number of 2^-q quanta (L#22).
 * q == 0 leaves the value continuous.  +inf stays +inf. */
static double qz(const orc_model* m, double x) {
  if (isinf(x)) return x;
  if (m->q <= 0) return x;
  return (double)llrint(ldexp(x, m->q));
}

/* -ln p with p = 0 meaning "forbidden" (+inf cost), "cost tables
 * (log-likelihoods instead of actual probabilities)". */
static double nlog(double p) {
  if (p <= 0.0) return INFINITY;
  return -log(p);
}

/* --------------------------------------------------------------------------
 * Eq. 4: the data cost of one pixel,
 *   C = min( log(d_range) - log(p_out),
 *            log(A_norm) + log(sigma*sqrt(2*pi)) - log(1-p_out) + (d-f)^2/(2 sigma^2) )
 * (L#4: Eq. 4 is followed, including its ln(sigma sqrt(2 pi)) term; L#5: the
 * unclosed "min(" of P:113 closes after the quadratic term; L#7: natural log.)
 * `delta` is d - f in disparity units.  Unquantized.
 * ------------------------------------------------------------------------ */
double orc_eq4(const orc_model* m, double delta, double sigma) {
  double uniform_branch = log((double)m->D) - log(m->p_out);
  double gauss_branch = log(m->a_norm) + log(sigma * sqrt(2.0 * M_PI)) - log(1.0 - m->p_out)
                        + (delta * delta) / (2.0 * sigma * sigma);
  return gauss_branch < uniform_branch ? gauss_branch : uniform_branch;
}

/* --------------------------------------------------------------------------
 * Ground model: f_ground(v) = alpha*(v_horizon - v), clamped at 0 (L#14),
 * with v counted from the bottom row of the column (L#12): the horizon's model
 * row is (h-1) - horizon_row.  Result in units of 1/2^R_bits, rounded half up.
 * ------------------------------------------------------------------------ */
long long orc_ground_R(const orc_model* m, int v) {
  double v_hor = (double)(m->h - 1) - m->horizon_row;
  double x = m->alpha * (v_hor - (double)v);
  if (x <= 0.0) return 0;
  return (long long)floor(x * (double)(1 << m->R_bits) + 0.5);
}

/* --------------------------------------------------------------------------
 * Column reduction + transpose ("replacing the disparities of s
 * consecutive pixels in the same row by their average"; L#8: mean of the VALID
 * pixels, all-invalid -> invalid, trailing W mod s dropped).
 * Input: raw fixed-point disparities with Q_bits fractional bits (a1); a pixel
 * is invalid if it equals `invalid` or decodes to >= D (L#23).
 * Output: out[c*H + v] = round_half_up(2^R_bits * sum / (2^Q_bits * n)) in
 * units of 1/2^R_bits, v = H-1-r (model row from the bottom), or -1 = invalid.
 * Not clamped (L#27: only the object model clamps, see object_disp); the one
 * representational limit is 0xFFFE (reduced columns are 16-bit with 0xFFFF =
 * invalid in the C ABI; reachable only at D = 256 with 8 fractional input bits).
 * ------------------------------------------------------------------------ */
/* One input pixel (a1).  u8/u16: the raw fixed-point value (Q_bits fractional
 * bits), invalid if it equals `invalid` or decodes to >= D.  f32 (bytes_per_px 4,
 * DESIGN.md L#28): a disparity in pixels, invalid if not finite, negative or
 * >= D; a valid value is converted once to the 1/2^8 grid, half up:
 * u = floor(256 d + 1/2) (the caller then uses Q_bits = 8).  Returns validity. */
static int pixel_value(const void* img, int bytes_per_px, long long idx, unsigned int invalid,
                       int D, int Q_bits, unsigned int* u) {
  if (bytes_per_px == 4) {
    double d = (double)((const float*)img)[idx];
    if (!isfinite(d) || d < 0.0 || d >= (double)D) return 0;
    *u = (unsigned int)floor(d * 256.0 + 0.5);
    return 1;
  }
  unsigned int x = bytes_per_px == 1 ? ((const uint8_t*)img)[idx] : ((const uint16_t*)img)[idx];
  if (x == invalid) return 0;
  if ((long long)x >= ((long long)D << Q_bits)) return 0; /* d >= D: invalid */
  *u = x;
  return 1;
}

static int clamp_reduced(long long x, int D, int R_bits) {
  (void)D; (void)R_bits;
  return (int)(x < 0xFFFE ? x : 0xFFFE);
}
void orc_reduce(const void* img, int bytes_per_px, int W, int H, long long pitch_px, int s,
                int Q_bits, unsigned int invalid, int D, int R_bits, int* out) {
  int n_cols = W / s;
  if (bytes_per_px == 4) Q_bits = 8;   /* f32: values converted to the 1/256 grid */
  for (int c = 0; c < n_cols; ++c) {
    for (int r = 0; r < H; ++r) {
      long long sum = 0, n = 0;
      for (int x = c * s; x < c * s + s; ++x) {
        unsigned int u;
        if (!pixel_value(img, bytes_per_px, (long long)r * pitch_px + x, invalid, D, Q_bits, &u))
          continue;
        sum += u;
        n += 1;
      }
      int v = H - 1 - r;
      if (n == 0) {
        out[(long long)c * H + v] = -1;
      } else {
        /* round half up of (2^R * sum) / (2^Q * n) = floor((2*2^R*sum + 2^Q*n) / (2*2^Q*n)) */
        long long num = 2 * (sum << R_bits) + (n << Q_bits);
        long long den = 2 * (n << Q_bits);
        out[(long long)c * H + v] = clamp_reduced(num / den, D, R_bits);
      }
    }
  }
}

/* --------------------------------------------------------------------------
 * Median column reduction (NEXT row f4 of SURVEY 8(f); BASELINE north_star
 * "median/mean" reduction of the s pixels; reading L#24): the median
 * of the VALID pixels among the s of a row segment -- the middle value of the
 * sorted valid values, the mean of the two middle values when their count is
 * even -- in units of 1/2^R_bits, rounded half up exactly like the mean
 * (orc_reduce with the middle value(s) as the summands), with the same
 * 0xFFFE limit.  All invalid -> -1.
 * Written the plain way: collect, sort (qsort), pick.
 * ------------------------------------------------------------------------ */
static int cmp_uint(const void* a, const void* b) {
  unsigned int x = *(const unsigned int*)a, y = *(const unsigned int*)b;
  return (x > y) - (x < y);
}

void orc_reduce_median(const void* img, int bytes_per_px, int W, int H, long long pitch_px,
                       int s, int Q_bits, unsigned int invalid, int D, int R_bits, int* out) {
  int n_cols = W / s;
  if (bytes_per_px == 4) Q_bits = 8;   /* f32: values converted to the 1/256 grid */
  unsigned int* vals = (unsigned int*)malloc(sizeof(unsigned int) * (size_t)(s > 0 ? s : 1));
  for (int c = 0; c < n_cols; ++c) {
    for (int r = 0; r < H; ++r) {
      int n = 0;
      for (int x = c * s; x < c * s + s; ++x) {
        unsigned int u;
        if (!pixel_value(img, bytes_per_px, (long long)r * pitch_px + x, invalid, D, Q_bits, &u))
          continue;
        vals[n++] = u;
      }
      int v = H - 1 - r;
      if (n == 0) {
        out[(long long)c * H + v] = -1;
        continue;
      }
      qsort(vals, (size_t)n, sizeof(unsigned int), cmp_uint);
      long long sum, cnt;
      if (n % 2) { sum = vals[n / 2]; cnt = 1; }
      else { sum = (long long)vals[n / 2 - 1] + vals[n / 2]; cnt = 2; }
      long long num = 2 * (sum << R_bits) + (cnt << Q_bits);
      long long den = 2 * (cnt << Q_bits);
      out[(long long)c * H + v] = clamp_reduced(num / den, D, R_bits);
    }
  }
  free(vals);
}

/* --------------------------------------------------------------------------
 * Per-pixel data costs (Eq. 4 per class).
 *  ground: f = f_ground(v) (fixed point); sky: f = 0;
 *  object: f integer mean, measured disparity rounded half up to an
 *          integer ("pairs of pixel disparity and mean disparity", L#9).
 * dR < 0 marks an invalid pixel -> the uniform (outlier) branch for every class
 * ("sometimes due to non-valid disparity measurements").
 * ------------------------------------------------------------------------ */
static double cap_cost(const orc_model* m) { return log((double)m->D) - log(m->p_out); }

double orc_cost_ground(const orc_model* m, int dR, int v) {
  if (dR < 0) return qz(m, cap_cost(m));
  double R = (double)(1 << m->R_bits);
  double delta = (double)((long long)dR - orc_ground_R(m, v)) / R;
  return qz(m, orc_eq4(m, delta, m->sigma_g_v ? m->sigma_g_v[v] : m->sigma[ORC_G]));
}
double orc_cost_sky(const orc_model* m, int dR) {
  if (dR < 0) return qz(m, cap_cost(m));
  double R = (double)(1 << m->R_bits);
  double delta = (double)dR / R;
  return qz(m, orc_eq4(m, delta, m->sigma[ORC_S]));
}
int orc_round_disp(const orc_model* m, int dR) {
  return (dR + (1 << (m->R_bits - 1))) >> m->R_bits;
}
/* The pixel disparity as the object model sees it (L#27): the pair LUT of P:175
 * is D x D ("all possible pairs of pixel disparity and mean disparity"), so the
 * object model takes d' clamped below D - 1/2, where its half-up rounding is
 * D - 1; its LUT index and its span mean use this value.  Ground and
 * sky (Eq. 4) use d' itself. */
static int object_disp(const orc_model* m, int dR) {
  int mx = ((m->D - 1) << m->R_bits) + (1 << (m->R_bits - 1)) - 1;
  return dR < mx ? dR : mx;
}
double orc_cost_object(const orc_model* m, int dR, int f) {
  if (dR < 0) return qz(m, cap_cost(m));
  double delta = (double)(orc_round_disp(m, object_disp(m, dR)) - f);
  return qz(m, orc_eq4(m, delta, m->sigma_o_f ? m->sigma_o_f[f] : m->sigma[ORC_O]));
}

/* --------------------------------------------------------------------------
 * Object model value f_n ("the mean of the measured disparities of the
 * considered stixel"), rounded to an integer, half up (L#10), in exact
 * integer arithmetic, of the object disparities object_disp (L#27; hence in
 * [0, D-1], the clamp below is a guard); 0 if the span has no valid pixel
 * (L#11).  From the span's disparity sum S (units 1/2^R) and valid count n.
 * ------------------------------------------------------------------------ */
static int mean_from_sums(const orc_model* m, long long S, long long n) {
  if (n == 0) return 0;
  long long R = 1LL << m->R_bits;
  long long f = (2 * S + R * n) / (2 * R * n);
  if (f > m->D - 1) f = m->D - 1;
  return (int)f;
}

int orc_span_mean(const orc_model* m, const int* col, int vb, int vt) {
  long long S = 0, n = 0;
  for (int v = vb; v <= vt; ++v) {
    if (col[v] < 0) continue;
    S += object_disp(m, col[v]);
    n += 1;
  }
  return mean_from_sums(m, S, n);
}

/* Data term of a stixel ("the aggregation of the costs of all of its
 * pixels"), by direct summation over its rows. */
double orc_stixel_data(const orc_model* m, const int* col, int cls, int vb, int vt, int f) {
  double s = 0.0;
  for (int v = vb; v <= vt; ++v) {
    if (cls == ORC_G) s += orc_cost_ground(m, col[v], v);
    else if (cls == ORC_S) s += orc_cost_sky(m, col[v]);
    else s += orc_cost_object(m, col[v], f);
  }
  return s;
}

/* --------------------------------------------------------------------------
 * Prior / smoothness term (P:65-66 five constraints, "cost tables"; the
 * proposed model is reading L#1, L#15, L#16):
 *   first stixel: -ln p_first[c] - ln p_exist            (Eq. 5, BIC per stixel)
 *   transition  : -ln p_trans[c'][c] - ln p_exist
 *               + ordering (O above O): -ln p_ord if f > f' + ord_margin else -ln(1-p_ord)
 *               + gravity/diving (O above G at base row vb):
 *                   -ln p_grav if f > f_ground(vb) + grav_margin   (floating object)
 *                   -ln p_blg  if f < f_ground(vb) - grav_margin   (object below ground)
 *                   -ln(1-p_grav-p_blg) otherwise
 * Each constant is quantized on its own (L#22), then summed exactly.
 * ------------------------------------------------------------------------ */
double orc_prior_first(const orc_model* m, int cls) {
  return qz(m, nlog(m->p_first[cls]) + nlog(m->p_exist));
}

double orc_prior_trans(const orc_model* m, int prev_cls, int prev_f, int cls, int vb, int f) {
  double t = qz(m, nlog(m->p_trans[prev_cls][cls]) + nlog(m->p_exist));
  if (isinf(t)) return t;
  if (cls == ORC_O && prev_cls == ORC_O) {
    if (f > prev_f + m->ord_margin) t += qz(m, nlog(m->p_ord));
    else t += qz(m, nlog(1.0 - m->p_ord));
  } else if (cls == ORC_O && prev_cls == ORC_G) {
    long long R = 1LL << m->R_bits;
    long long g = orc_ground_R(m, vb);
    long long fR = (long long)f * R;
    if (fR > g + (long long)m->grav_margin * R) t += qz(m, nlog(m->p_grav));
    else if (fR < g - (long long)m->grav_margin * R) t += qz(m, nlog(m->p_blg));
    else t += qz(m, nlog(1.0 - m->p_grav - m->p_blg));
  }
  return t;
}

/* Output disparity of a stixel (L#19): O -> its integer mean f; G -> the ground
 * model at its base row; S -> 0. */
static double stixel_disp(const orc_model* m, int cls, int vb, int f) {
  if (cls == ORC_O) return (double)f;
  if (cls == ORC_G) return (double)orc_ground_R(m, vb) / (double)(1 << m->R_bits);
  return 0.0;
}

/* --------------------------------------------------------------------------
 * Re-score a labelled segmentation by direct summation with its TRUE
 * predecessors: sum of data terms + first prior + pairwise priors.
 * This is the MAP objective -ln P(D|L) - ln P(L) of Eq. 1 under the model.
 * ------------------------------------------------------------------------ */
double orc_rescore(const orc_model* m, const int* col, const orc_stixel* st, int n) {
  double total = 0.0;
  int prev_f = 0;
  for (int i = 0; i < n; ++i) {
    int f = (st[i].cls == ORC_O) ? orc_span_mean(m, col, st[i].vb, st[i].vt) : 0;
    total += orc_stixel_data(m, col, st[i].cls, st[i].vb, st[i].vt, f);
    if (i == 0) total += orc_prior_first(m, st[i].cls);
    else total += orc_prior_trans(m, st[i - 1].cls, prev_f, st[i].cls, st[i].vb, f);
    prev_f = f;
  }
  return total;
}

/* --------------------------------------------------------------------------
 * Eq. 5-6 dynamic program for one column, followed by backtracking
 * through the index table.
 *
 * C[c][k]  = minimum cost of segmenting rows 0..k with the last stixel of class c
 *            (OB^k, GR^k, SK^k of P:129);
 * arg[c][k]= (j, c') of the winning candidate: last stixel spans j..k and the
 *            predecessor segmentation ends at j-1 with class c' (START if j = 0);
 * F[c][k]  = the object model value f of that last stixel ("the stixel at the end
 *            of the segmentation associated with each minimum cost"),
 *            which the prior of later steps consumes (Eq. 6; L#18).
 * Candidates are enumerated in a fixed order -- j = 0 first, then j = 1..k
 * ascending, and c' in G < O < S -- and the first strict minimum wins (L#17).
 *
 * mode 0 ("direct"): data terms and span means by direct per-pixel summation,
 *                    O(h^3) per column.
 * mode 1 ("prefix"): data terms as differences of prefix sums (L#13)
 *                    and span means from a disparity prefix sum, O(h^2).
 *                    The per-pixel costs and prior constants are evaluated once
 *                    per column with exactly the same expressions as mode 0.
 * Returns the number of stixels written to out (bottom -> top) and the column's
 * minimum cost in *cost.  C/arg/F outputs may be NULL.
 * ------------------------------------------------------------------------ */
int orc_solve_column(const orc_model* m, const int* col, int mode, orc_stixel* out, double* cost,
                     double* Cout, int* argj_out, int* argc_out, int* F_out) {
  int h = m->h;
  double* C = (double*)malloc(sizeof(double) * 3 * h);
  int* aj = (int*)malloc(sizeof(int) * 3 * h);
  int* ac = (int*)malloc(sizeof(int) * 3 * h);
  int* F = (int*)malloc(sizeof(int) * 3 * h);
  double *PG = NULL, *PS = NULL, *PO = NULL;
  long long *PD = NULL, *PN = NULL;
  double first[3], trans[3][3], ord_hi = 0, ord_lo = 0, grav_hi = 0, grav_lo = 0, grav_mid = 0;
  long long* gR = NULL;
  if (mode == 1) {
    PG = (double*)calloc((size_t)h + 1, sizeof(double));
    PS = (double*)calloc((size_t)h + 1, sizeof(double));
    PO = (double*)calloc((size_t)m->D * (h + 1), sizeof(double));
    PD = (long long*)calloc((size_t)h + 1, sizeof(long long));
    PN = (long long*)calloc((size_t)h + 1, sizeof(long long));
    gR = (long long*)calloc((size_t)h + 1, sizeof(long long));
    for (int v = 0; v < h; ++v) {
      PG[v + 1] = PG[v] + orc_cost_ground(m, col[v], v);
      PS[v + 1] = PS[v] + orc_cost_sky(m, col[v]);
      for (int f = 0; f < m->D; ++f)
        PO[(size_t)f * (h + 1) + v + 1] = PO[(size_t)f * (h + 1) + v] + orc_cost_object(m, col[v], f);
      PD[v + 1] = PD[v] + (col[v] >= 0 ? object_disp(m, col[v]) : 0);
      PN[v + 1] = PN[v] + (col[v] >= 0 ? 1 : 0);
      gR[v] = orc_ground_R(m, v);
    }
    for (int c = 0; c < 3; ++c) {
      first[c] = orc_prior_first(m, c);
      for (int cp = 0; cp < 3; ++cp) trans[cp][c] = qz(m, nlog(m->p_trans[cp][c]) + nlog(m->p_exist));
    }
    ord_hi = qz(m, nlog(m->p_ord));
    ord_lo = qz(m, nlog(1.0 - m->p_ord));
    grav_hi = qz(m, nlog(m->p_grav));
    grav_lo = qz(m, nlog(m->p_blg));
    grav_mid = qz(m, nlog(1.0 - m->p_grav - m->p_blg));
  }
  long long R = 1LL << m->R_bits;
  for (int k = 0; k < h; ++k) {
    for (int c = 0; c < 3; ++c) {
      double best = 0.0;
      int bj = 0, bc = ORC_START, bf = 0;
      for (int j = 0; j <= k; ++j) {
        int f = 0;
        double data;
        if (mode == 0) {
          if (c == ORC_O) f = orc_span_mean(m, col, j, k);
          data = orc_stixel_data(m, col, c, j, k, f);
        } else {
          if (c == ORC_O) f = mean_from_sums(m, PD[k + 1] - PD[j], PN[k + 1] - PN[j]);
          if (c == ORC_G) data = PG[k + 1] - PG[j];
          else if (c == ORC_S) data = PS[k + 1] - PS[j];
          else data = PO[(size_t)f * (h + 1) + k + 1] - PO[(size_t)f * (h + 1) + j];
        }
        if (j == 0) {
          /* Eq. 5 / first line of Eq. 6: the stixel starts at the column base */
          best = data + (mode == 0 ? orc_prior_first(m, c) : first[c]);
          bj = 0; bc = ORC_START; bf = f;
          continue;
        }
        for (int cp = 0; cp < 3; ++cp) {
          double prior;
          if (mode == 0) {
            prior = orc_prior_trans(m, cp, F[cp * h + (j - 1)], c, j, f);
          } else {
            /* same terms as orc_prior_trans, constants hoisted */
            prior = trans[cp][c];
            if (!isinf(prior)) {
              if (c == ORC_O && cp == ORC_O) {
                prior += (f > F[ORC_O * h + (j - 1)] + m->ord_margin) ? ord_hi : ord_lo;
              } else if (c == ORC_O && cp == ORC_G) {
                long long fR = (long long)f * R;
                if (fR > gR[j] + (long long)m->grav_margin * R) prior += grav_hi;
                else if (fR < gR[j] - (long long)m->grav_margin * R) prior += grav_lo;
                else prior += grav_mid;
              }
            }
          }
          double cand = data + prior + C[cp * h + (j - 1)];
          if (cand < best) {
            best = cand; bj = j; bc = cp; bf = f;
          }
        }
      }
      C[c * h + k] = best;
      aj[c * h + k] = bj;
      ac[c * h + k] = bc;
      F[c * h + k] = bf;
    }
  }
  /* Backtracking: start at min(OB^{h-1}, GR^{h-1}, SK^{h-1}), ties G<O<S. */
  int c = 0;
  for (int cc = 1; cc < 3; ++cc)
    if (C[cc * h + h - 1] < C[c * h + h - 1]) c = cc;
  *cost = C[c * h + h - 1];
  orc_stixel* tmp = (orc_stixel*)malloc(sizeof(orc_stixel) * h);
  int n = 0, k = h - 1;
  while (1) {
    int j = aj[c * h + k];
    tmp[n].vb = j; tmp[n].vt = k; tmp[n].cls = c;
    tmp[n].disp = stixel_disp(m, c, j, F[c * h + k]);
    n++;
    if (j == 0 || n >= h) break;
    int cp = ac[c * h + k];
    k = j - 1;
    c = cp;
  }
  for (int i = 0; i < n; ++i) out[i] = tmp[n - 1 - i];
  if (Cout) memcpy(Cout, C, sizeof(double) * 3 * h);
  if (argj_out) memcpy(argj_out, aj, sizeof(int) * 3 * h);
  if (argc_out) memcpy(argc_out, ac, sizeof(int) * 3 * h);
  if (F_out) memcpy(F_out, F, sizeof(int) * 3 * h);
  free(tmp); free(C); free(aj); free(ac); free(F);
  free(PG); free(PS); free(PO); free(PD); free(PN); free(gR);
  return n;
}

/* --------------------------------------------------------------------------
 * Brute force (Eq. 1 argmax, by exhaustive enumeration): every split of
 * the column into consecutive stixels and every labelling, 3*4^(h-1) candidates
 * (S:393).  Scored with orc_rescore (true predecessors).  First minimum in
 * enumeration order wins.  h <= 12.
 * ------------------------------------------------------------------------ */
static void bf_rec(const orc_model* m, const int* col, orc_stixel* cur, int n, int start,
                   double* best, orc_stixel* best_seg, int* best_n, long long* count) {
  if (start == m->h) {
    double s = orc_rescore(m, col, cur, n);
    (*count)++;
    if (s < *best) {
      *best = s;
      memcpy(best_seg, cur, sizeof(orc_stixel) * n);
      *best_n = n;
    }
    return;
  }
  for (int vt = start; vt < m->h; ++vt) {
    for (int c = 0; c < 3; ++c) {
      cur[n].vb = start; cur[n].vt = vt; cur[n].cls = c;
      int f = (c == ORC_O) ? orc_span_mean(m, col, start, vt) : 0;
      cur[n].disp = stixel_disp(m, c, start, f);
      bf_rec(m, col, cur, n + 1, vt + 1, best, best_seg, best_n, count);
    }
  }
}

long long orc_bruteforce_column(const orc_model* m, const int* col, orc_stixel* out, int* n_out,
                                double* cost) {
  if (m->h > 12 || m->h < 1) return -1;
  orc_stixel cur[12];
  double best = INFINITY;
  int best_n = 0;
  long long count = 0;
  bf_rec(m, col, cur, 0, 0, &best, out, &best_n, &count);
  *n_out = best_n;
  *cost = best;
  return count;
}

/* --------------------------------------------------------------------------
 * Whole frame: columns are independent, so OpenMP over columns
 * (S:360); results do not depend on the thread count.
 * cols: [n_cols][h] reduced columns (model order); out: [n_cols][h] stixels.
 * ------------------------------------------------------------------------ */
void orc_solve_frame(const orc_model* m, const int* cols, int n_cols, int mode, int n_threads,
                     orc_stixel* out, int* count, double* cost) {
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int c = 0; c < n_cols; ++c) {
    count[c] = orc_solve_column(m, cols + (long long)c * m->h, mode, out + (long long)c * m->h,
                                cost + c, NULL, NULL, NULL, NULL);
  }
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
