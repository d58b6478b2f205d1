// api.cu -- host side of the C ABI declared in include/stixels.h.
//
// Builds the input-independent tables of the paper's LUT scheme on the host
// ("most of the terms in the equation do not depend on the input
// data and can be pre-computed"; the off-line D x D pair-cost LUT, here
// in its |f - d| form since sigma is per class, L#2), validates parameters,
// owns device memory, and launches the two sm_100a kernels of kernels.cuh.
// There is no CPU compute path: the host only prepares tables and launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/stixels.h"
#include "kernels.cuh"

using namespace stx;

struct stixels_handle {
  stixels_params p{};
  int W = 0, H = 0, max_batch = 0, device = 0;
  cudaStream_t stream = nullptr;
  int n_cols = 0, cap = 0, dp_slots = 128, cols_per_cta = 0, smem = 0, grid = 0, sms = 0;
  int col_bytes8 = 0, cols_per_cta8 = 0;   // CW = 8 column groups (small batches), 0 = off
  int last_cw = 0, last_cpc = 0;            // warps per column, groups per CTA of the last DP launch
  int plan_cw = 0;                          // stixels_set_launch_plan: 0 auto, 4 or 8
  bool bound_ok = false, bound_auto = false;  // chunk bound possible / on by default
  int bound_mode = 0;                       // stixels_set_chunk_bound: 0 auto, 1 off, 2 on
  bool sparse = true;
  bool pair2d = false;          // NEXT f2: sigma_O(f) table given
  bool iw = false;              // int32 W-rows with atomic band rounds (band <= 3, exact mode)
  int red_tc = 0, red_smem = 0, red_w2 = 0;
  int smem_optin = 0;           // opt-in shared memory per block (reduce_strip_kernel stages)
  DPArgs args{};
  float* d_E = nullptr;
  float* d_E2 = nullptr;        // NEXT f2: [D+2][DP] 2-D pair table
  float* d_WT = nullptr;        // NEXT f2: [DP+17][16] band weights
  uint32_t* d_M2 = nullptr;
  float* d_gG = nullptr;
  float* d_gS = nullptr;
  int* d_dgR = nullptr;
  uint32_t* d_thr = nullptr;
  int* d_overflow = nullptr;
  unsigned long long* d_skipped = nullptr;   // IW chunk bound: cumulative skipped cells
  float* d_scratch = nullptr;   // per-column-slot DP scratch of h->stream (and hs[0])
  uint16_t* d_cols = nullptr;   // reduced columns of the two-launch plan [max_batch][n_cols][H]
  size_t scratch_bytes = 0;
  // host-buffer path (lazily allocated): two stage streams, each with its own DP
  // scratch (hs[0] shares d_scratch with h->stream, which it waits for; hs[1] has
  // hscratch1), so DP launches of consecutive stages may overlap on the SMs
  cudaStream_t hs[2] = {nullptr, nullptr};
  float* hscratch1 = nullptr;
  cudaEvent_t ev_entry = nullptr;
  uint8_t* hin[2] = {nullptr, nullptr};
  stixel_t* hout[2] = {nullptr, nullptr};
  int32_t* hcnt[2] = {nullptr, nullptr};
  float* hcost[2] = {nullptr, nullptr};
  uint16_t* hcols[2] = {nullptr, nullptr};
  int h_chunk = 0;
  int64_t h_pitch = 0;
  std::string err;
  int sticky = 0;
  int launches = 0;
};


// The DP kernel instantiation for the handle's model (f2 tables, sparse / dense
// band, int32 atomic bands) and column-group width cw; `go(kernel)` launches it.
template <int CW, typename Go>
static void dispatch_dp_cw(const stixels_handle* h, Go&& go) {
  if (h->dp_slots == 128) {
    if (h->pair2d && h->sparse) go(dp_kernel<128, true, true, false, CW>);
    else if (h->pair2d) go(dp_kernel<128, false, true, false, CW>);
    else if (h->iw) go(dp_kernel<128, true, false, true, CW>);
    else if (h->sparse) go(dp_kernel<128, true, false, false, CW>);
    else go(dp_kernel<128, false, false, false, CW>);
  } else {
    if (h->pair2d && h->sparse) go(dp_kernel<256, true, true, false, CW>);
    else if (h->pair2d) go(dp_kernel<256, false, true, false, CW>);
    else if (h->iw) go(dp_kernel<256, true, false, true, CW>);
    else if (h->sparse) go(dp_kernel<256, true, false, false, CW>);
    else go(dp_kernel<256, false, false, false, CW>);
  }
}
template <typename Go>
static void dispatch_dp(const stixels_handle* h, int cw, Go&& go) {
  if (cw == 8) dispatch_dp_cw<8>(h, go);
  else dispatch_dp_cw<kCW>(h, go);
}
static const void* dp_kernel_ptr(const stixels_handle* h, int cw) {
  const void* f = nullptr;
  dispatch_dp(h, cw, [&](auto k) { f = (const void*)k; });
  return f;
}

static thread_local std::string g_create_err;

static int bytes_per_px(int fmt) { return fmt == STIXELS_F32 ? 4 : fmt == STIXELS_U16 ? 2 : 1; }

static int fail(stixels_handle* h, int code, const std::string& msg) {
  if (h) {
    h->err = msg;
    if (code == STIXELS_ERR_CUDA) h->sticky = code;
  } else {
    g_create_err = msg;
  }
  return code;
}

#define CU(call, h)                                                                         \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(h, STIXELS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------------------
// Model arithmetic on the host (double), written from the paper.
// ---------------------------------------------------------------------------
namespace {

constexpr double kPi = 3.14159265358979323846;

struct Host {
  const stixels_params& p;
  int h;
  double R = 256.0;
  explicit Host(const stixels_params& pp, int hh) : p(pp), h(hh) {}

  // cost quantization to 2^-q nats (L#22); continuous when q == 0
  double Q(double x) const {
    if (std::isinf(x)) return x;
    if (p.cost_frac_bits <= 0) return x;
    return (double)std::llrint(std::ldexp(x, p.cost_frac_bits));
  }
  static double nl(double prob) { return prob <= 0.0 ? INFINITY : -std::log(prob); }
  // Eq. 4, sigma per class, natural log (L#4, L#5, L#7)
  double eq4(double delta, double sigma) const {
    double unif = std::log((double)p.max_disparity) - std::log((double)p.p_out);
    double g = std::log((double)p.a_norm) + std::log(sigma * std::sqrt(2.0 * kPi)) -
               std::log(1.0 - (double)p.p_out) + (delta * delta) / (2.0 * sigma * sigma);
    return g < unif ? g : unif;
  }
  double cap() const { return std::log((double)p.max_disparity) - std::log((double)p.p_out); }
  double alpha() const {
    if (p.ground_slope > 0.0f) return (double)p.ground_slope;
    double th = std::atan(((double)p.principal_row - (double)p.horizon_row) / (double)p.focal_px);
    return (double)p.baseline_m * std::cos(th) / (double)p.camera_height_m;
  }
  // ground model f_ground(v) = alpha (v_hor - v), v from the bottom, clamp >= 0,
  // in 1/256 units rounded half up (L#12, L#14)
  long long ground_R(int v) const {
    double vh = (double)(h - 1) - (double)p.horizon_row;
    double x = alpha() * (vh - (double)v);
    if (x <= 0.0) return 0;
    return (long long)std::floor(x * R + 0.5);
  }
};

long long floor_div(long long a, long long b) {
  long long q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
long long ceil_div(long long a, long long b) { return -floor_div(-a, b); }

bool prob_ok(float x) { return std::isfinite(x) && x >= 0.f && x <= 1.f; }

int validate(const stixels_params* p, int W, int H, int max_batch, std::string& msg) {
  if (!p) { msg = "params is NULL"; return STIXELS_ERR_ARG; }
  if (H < 1 || W < 1 || max_batch < 1) { msg = "width, height and max_batch must be >= 1"; return STIXELS_ERR_ARG; }
  // the reduction grid carries the frame index in gridDim.z (<= 65535)
  if (max_batch > 65535) { msg = "max_batch > 65535 not supported"; return STIXELS_ERR_UNSUPPORTED; }
  if (p->stixel_width < 1) { msg = "stixel_width must be >= 1 (S:56)"; return STIXELS_ERR_PARAM; }
  if (W < p->stixel_width) { msg = "width < stixel_width gives no column (S:125)"; return STIXELS_ERR_ARG; }
  if (p->stixel_width > 512) { msg = "stixel_width > 512 not supported"; return STIXELS_ERR_UNSUPPORTED; }
  if (H > kMaxH) { msg = "height > 1024 not supported"; return STIXELS_ERR_UNSUPPORTED; }
  if (!(p->p_out > 0.f && p->p_out < 1.f)) { msg = "need 0 < p_out < 1 (S:44)"; return STIXELS_ERR_PARAM; }
  for (int c = 0; c < 3; ++c)
    if (!(p->sigma[c] > 0.f) || !std::isfinite(p->sigma[c])) { msg = "sigma must be > 0"; return STIXELS_ERR_PARAM; }
  if (!(p->a_norm > 0.f) || !std::isfinite(p->a_norm)) { msg = "a_norm must be > 0"; return STIXELS_ERR_PARAM; }
  if (p->max_disparity < 2) { msg = "max_disparity must be >= 2 (S:44)"; return STIXELS_ERR_PARAM; }
  if (p->max_disparity > 256) { msg = "max_disparity > 256 not supported"; return STIXELS_ERR_UNSUPPORTED; }
  if (!std::isfinite(p->horizon_row)) { msg = "horizon_row must be finite (S:38)"; return STIXELS_ERR_PARAM; }
  if (!(p->ground_slope > 0.f)) {
    if (!(p->focal_px > 0.f) || !(p->camera_height_m > 0.f) || !(p->baseline_m > 0.f) ||
        !std::isfinite(p->principal_row)) {
      msg = "ground_slope <= 0 needs focal_px, baseline_m, camera_height_m > 0"; return STIXELS_ERR_PARAM;
    }
  }
  for (int c = 0; c < 3; ++c) {
    if (!prob_ok(p->p_first[c])) { msg = "p_first must be in [0,1]"; return STIXELS_ERR_PARAM; }
    for (int d = 0; d < 3; ++d)
      if (!prob_ok(p->p_trans[c][d])) { msg = "p_trans must be in [0,1]"; return STIXELS_ERR_PARAM; }
  }
  if (!prob_ok(p->p_ord) || !prob_ok(p->p_grav) || !prob_ok(p->p_blg) || !prob_ok(p->p_exist) ||
      p->p_grav + p->p_blg > 1.f) {
    msg = "p_ord, p_grav, p_blg, p_exist must be probabilities, p_grav + p_blg <= 1"; return STIXELS_ERR_PARAM;
  }
  if (p->p_first[STIXELS_SKY] != 0.f || p->p_trans[0][0] != 0.f || p->p_trans[2][2] != 0.f ||
      p->p_trans[2][0] != 0.f || p->p_trans[2][1] != 0.f) {
    msg = "structurally forbidden prior entries must be 0: p_first[sky], p_trans[G][G], "
          "p_trans[S][S], p_trans[S][G], p_trans[S][O] (L#16)";
    return STIXELS_ERR_PARAM;
  }
  if (p->ord_margin < 0 || p->grav_margin < 0 || p->ord_margin > 255 || p->grav_margin > 255) {
    msg = "margins must be in [0, 255]"; return STIXELS_ERR_PARAM;
  }
  if (p->disp_format != STIXELS_U8 && p->disp_format != STIXELS_U16 && p->disp_format != STIXELS_F32) {
    msg = "disp_format must be U8, U16 or F32"; return STIXELS_ERR_PARAM;
  }
  if (p->disp_frac_bits < 0 || p->disp_frac_bits > 8) { msg = "disp_frac_bits must be in [0, 8]"; return STIXELS_ERR_PARAM; }
  if (p->reduce_mode != STIXELS_REDUCE_MEAN && p->reduce_mode != STIXELS_REDUCE_MEDIAN) {
    msg = "reduce_mode must be STIXELS_REDUCE_MEAN (P:195) or STIXELS_REDUCE_MEDIAN"; return STIXELS_ERR_UNSUPPORTED;
  }
  if (p->reduce_mode == STIXELS_REDUCE_MEDIAN && p->stixel_width > kMedianMaxS) {
    msg = "the median reduction supports stixel_width <= 64"; return STIXELS_ERR_UNSUPPORTED;
  }
  if (p->cost_frac_bits < 0 || p->cost_frac_bits > 20) { msg = "cost_frac_bits must be in [0, 20]"; return STIXELS_ERR_PARAM; }
  if (p->max_stixels < 0) { msg = "max_stixels must be >= 0"; return STIXELS_ERR_PARAM; }
  return STIXELS_OK;
}

}  // namespace

extern "C" {

int stixels_default_params(stixels_params* p) {
  if (!p) return STIXELS_ERR_ARG;
  std::memset(p, 0, sizeof(*p));
  p->focal_px = 1000.f; p->baseline_m = 0.3f; p->camera_height_m = 1.2f;
  p->horizon_row = 132.f; p->principal_row = 0.f; p->ground_slope = 0.4f;
  p->p_out = 0.15f;
  p->sigma[0] = 2.0f; p->sigma[1] = 1.0f; p->sigma[2] = 0.5f;
  p->a_norm = 1.0f;
  p->p_first[0] = 1.0f; p->p_first[1] = (float)std::exp(-2.0); p->p_first[2] = 0.f;
  for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) p->p_trans[a][b] = 1.f;
  p->p_trans[0][0] = p->p_trans[2][2] = p->p_trans[2][0] = p->p_trans[2][1] = 0.f;
  p->p_ord = 0.2f; p->p_grav = 0.1f; p->p_blg = 0.04f; p->p_exist = (float)std::exp(-4.0);
  p->ord_margin = 1; p->grav_margin = 1;
  p->stixel_width = 5; p->max_disparity = 128;
  p->disp_format = STIXELS_U16; p->disp_frac_bits = 4; p->invalid_value = 0xFFFF;
  p->reduce_mode = 0; p->cost_frac_bits = 11; p->max_stixels = 0;
  return STIXELS_OK;
}

const char* stixels_error_string(int s) {
  switch (s) {
    case STIXELS_OK: return "ok";
    case STIXELS_ERR_ARG: return "invalid argument";
    case STIXELS_ERR_PARAM: return "invalid parameter";
    case STIXELS_ERR_UNSUPPORTED: return "unsupported configuration";
    case STIXELS_ERR_CUDA: return "CUDA error";
    case STIXELS_ERR_CAPACITY: return "per-column stixel capacity exceeded";
    default: return "unknown status";
  }
}

const char* stixels_last_error(const stixels_handle* h) {
  return h ? h->err.c_str() : g_create_err.c_str();
}

static void free_all(stixels_handle* h) {
  cudaFree(h->d_E); cudaFree(h->d_E2); cudaFree(h->d_WT); cudaFree(h->d_M2); cudaFree(h->d_gG); cudaFree(h->d_gS);
  cudaFree(h->d_dgR); cudaFree(h->d_thr); cudaFree(h->d_overflow); cudaFree(h->d_skipped); cudaFree(h->d_scratch); cudaFree(h->d_cols);
  cudaFree(h->hscratch1);
  if (h->ev_entry) cudaEventDestroy(h->ev_entry);
  for (int i = 0; i < 2; ++i) {
    cudaFree(h->hin[i]); cudaFree(h->hout[i]); cudaFree(h->hcnt[i]); cudaFree(h->hcost[i]);
    cudaFree(h->hcols[i]);
    if (h->hs[i]) cudaStreamDestroy(h->hs[i]);
  }
}

int stixels_create(const stixels_params* params, int width, int height, int max_batch,
                   int device, void* cuda_stream, stixels_handle** out) {
  g_create_err.clear();
  if (!out) return fail(nullptr, STIXELS_ERR_ARG, "out is NULL");
  *out = nullptr;
  std::string msg;
  int st = validate(params, width, height, max_batch, msg);
  if (st != STIXELS_OK) return fail(nullptr, st, msg);

  stixels_handle* h = new stixels_handle();
  h->p = *params;
  h->W = width; h->H = height; h->max_batch = max_batch; h->device = device;
  h->stream = (cudaStream_t)cuda_stream;
  h->n_cols = width / params->stixel_width;
  h->cap = params->max_stixels > 0 ? std::min(params->max_stixels, height) : height;
  const int D = params->max_disparity;
  h->dp_slots = D <= 128 ? 128 : 256;

  auto bail = [&](int code, const std::string& m) {
    g_create_err = m.empty() ? h->err : m;
    free_all(h);
    delete h;
    return code;
  };

  // ---------------- host tables --------------------------------------------
  Host hm(*params, height);
  const double capQ = hm.Q(hm.cap());
  const int R = 256;
  std::vector<float> gG, gS;
  // NEXT f2 noise-model tables (host copies; the caller's arrays are read here only)
  std::vector<double> sig_o, sig_g;
  if (params->sigma_object_f) {
    for (int f = 0; f < D; ++f) {
      const float x = params->sigma_object_f[f];
      if (!(x > 0.f) || !std::isfinite(x)) return bail(STIXELS_ERR_PARAM, "sigma_object_f entries must be finite and > 0");
      sig_o.push_back((double)x);
    }
  }
  if (params->sigma_ground_v) {
    for (int v = 0; v < height; ++v) {
      const float x = params->sigma_ground_v[v];
      if (!(x > 0.f) || !std::isfinite(x)) return bail(STIXELS_ERR_PARAM, "sigma_ground_v entries must be finite and > 0");
      sig_g.push_back((double)x);
    }
  }
  h->p.sigma_object_f = nullptr;   // the handle keeps no caller pointers
  h->p.sigma_ground_v = nullptr;
  // ground / sky cost by distance to the model disparity in 1/256 units; with a
  // per-row sigma_G(v) one table per row, all of the longest row's length
  int LGr = 0;
  {
    const int nrows = sig_g.empty() ? 1 : height;
    std::vector<std::vector<float>> rows(nrows);
    for (int r = 0; r < nrows; ++r) {
      const double sg = sig_g.empty() ? (double)params->sigma[0] : sig_g[r];
      for (int i = 0;; ++i) {
        double v = hm.Q(hm.eq4((double)i / R, sg));
        rows[r].push_back((float)v);
        if (v >= capQ || i > D * R) break;
      }
      rows[r].back() = (float)capQ;
      LGr = std::max(LGr, (int)rows[r].size());
    }
    for (int r = 0; r < nrows; ++r) {
      rows[r].resize(LGr, (float)capQ);   // beyond a row's own table: the cap
      gG.insert(gG.end(), rows[r].begin(), rows[r].end());
    }
  }
  for (int i = 0;; ++i) {
    double v = hm.Q(hm.eq4((double)i / R, (double)params->sigma[2]));
    gS.push_back((float)v);
    if (v >= capQ || i > D * R) break;
  }
  gS.back() = (float)capQ;   // clamp index -> cap (monotone Eq. 4)
  // object pair-cost LUT Pair[f][d] = Eq4(d - f, sigma_O), stored shifted by
  // the outlier cap as E'[f - d + D] = Pair - cap (<= 0, exact integers in exact
  // mode): the DP kernel works with W-rows LUT_object[f][v] - cap * v.
  const int DPv = h->dp_slots;
  const int einv = ((D + DPv + 4) + 3) & ~3;
  const int esz = einv + DPv + 8;
  std::vector<float> E1((size_t)esz + 8);
  for (int i = 0; i < esz + 8; ++i)
    E1[i] = (i < einv) ? (float)(hm.Q(hm.eq4((double)(i - D), (double)params->sigma[1])) - capQ) : 0.f;
  std::vector<float> E4((size_t)4 * esz);
  for (int c = 0; c < 4; ++c)
    for (int i = 0; i < esz; ++i) E4[(size_t)c * esz + i] = E1[i + c];
  // band of the pair cost: |f - d| beyond which Pair == cap.  If <= 7 the kernel
  // updates W-rows sparsely (wt[d + 7] = cap - Pair for |d| <= 7).
  int band = 0;
  for (int d = -D; d <= D; ++d)
    if (E1[d + D] != 0.f) band = std::max(band, std::abs(d));
  // NEXT f2: Pair[f][d] = Eq4(d - f, sigma_O(f)), a genuine D x D table
  // any noise table selects the PAIR2D kernel; a missing sigma_O(f) table is the constant
  const bool pair2d = !sig_o.empty() || !sig_g.empty();
  if (pair2d && sig_o.empty()) sig_o.assign(D, (double)params->sigma[1]);
  std::vector<float> E2, WT;
  if (pair2d) {
    band = 0;
    E2.assign((size_t)(D + 2) * DPv, 0.f);          // rows d = 0..D (pixel), D+1 invalid
    for (int d = 0; d <= D; ++d)
      for (int f = 0; f < D; ++f) {
        const double x = hm.Q(hm.eq4((double)(d - f), sig_o[f])) - capQ;
        E2[(size_t)d * DPv + f] = (float)x;
        if (x != 0.0) band = std::max(band, std::abs(d - f));
      }
    // band > 7 (a wide sigma_O(f)): the dense W-row ring reads whole rows of E2
    WT.assign((size_t)(DPv + 17) * 16, 0.f);        // [wt_rows<DP>()][16]
    for (int d = 0; d <= D; ++d)                    // row drp = d + 1, lane offset o = f - d + 7
      for (int o = 0; o < 15; ++o) {
        const int f = d + o - 7;
        if (f >= 0 && f < D) WT[(size_t)(d + 1) * 16 + o] = -E2[(size_t)d * DPv + f];
      }
  }
  const bool sparse = band <= 7;
  const bool iw = sparse && !pair2d && band <= 3 && params->cost_frac_bits > 0;
  // magic reciprocals: floor(y/(2n)) = umulhi(y, ceil(2^31/n))
  std::vector<uint32_t> M2(height + 1);
  M2[0] = 0;
  for (int n = 1; n <= height; ++n) M2[n] = (uint32_t)(((1ull << 31) + n - 1) / n);
  // per-row ground model and gravity thresholds (a3)
  std::vector<int> dgR(height);
  for (int v = 0; v < height; ++v) dgR[v] = (int)hm.ground_R(v);

  DPArgs& A = h->args;
  std::memset(&A, 0, sizeof(A));
  // gravity / diving thresholds on the integer object mean f at base row v:
  // f*R > dgR + gm*R  <=>  f >= floor((dgR + gm*R)/R) + 1 ;  f*R < dgR - gm*R  <=>
  // f < ceil((dgR - gm*R)/R).  Packed as clamped u16 pair (unsigned compares).
  const long long gmR = (long long)params->grav_margin * R;
  std::vector<uint32_t> thrg(height);
  for (int v = 0; v < height; ++v) {
    long long a1 = floor_div(dgR[v] + gmR, R) + 1;
    long long bb = ceil_div(dgR[v] - gmR, R);
    a1 = std::max(0LL, std::min(1023LL, a1));     // f <= 255 < 1023: clamping is exact
    bb = std::max(0LL, std::min(1023LL, bb));
    A.thrA1[v] = (int)a1;
    A.thrB[v] = (int)bb;
    thrg[v] = (uint32_t)a1 | ((uint32_t)bb << 16);
  }
  for (int d = -7; d <= 7; ++d) A.wt[d + 7] = (sparse && !pair2d) ? -E1[d + D] : 0.f;
  A.wt[15] = 0.f;
  // priors (L#1): each constant quantized on its own
  const double bic = Host::nl(params->p_exist);
  double first[3], trans[3][3];
  for (int c = 0; c < 3; ++c) {
    first[c] = hm.Q(Host::nl(params->p_first[c]) + bic);
    for (int d = 0; d < 3; ++d) trans[c][d] = hm.Q(Host::nl(params->p_trans[c][d]) + bic);
  }
  const double ord_hi = hm.Q(Host::nl(params->p_ord));
  const double ord_lo = hm.Q(Host::nl(1.0 - (double)params->p_ord));
  const double grav_hi = hm.Q(Host::nl(params->p_grav));
  const double grav_lo = hm.Q(Host::nl(params->p_blg));
  const double grav_mid = hm.Q(Host::nl(1.0 - (double)params->p_grav - (double)params->p_blg));
  A.piFirstO = (float)first[1];
  A.piFirstG = (float)first[0];
  A.kOO_lo = (float)(trans[1][1] + ord_lo);
  A.kOO_hi = (float)(trans[1][1] + ord_hi);
  A.kGO_mid = (float)(trans[0][1] + grav_mid);
  A.kGO_hi = (float)(trans[0][1] + grav_hi);
  A.kGO_lo = (float)(trans[0][1] + grav_lo);
  A.kOG = (float)trans[1][0];
  A.kGS = (float)trans[0][2];
  A.kOS = (float)trans[1][2];
  if (params->cost_frac_bits > 0) {
    // exact mode: every finite cost must stay an exact fp32 integer (< 2^24)
    double pmax = 0;
    double cands[] = {first[0], first[1], trans[0][1] + std::max({grav_hi, grav_lo, grav_mid}),
                      trans[1][1] + std::max(ord_hi, ord_lo), trans[1][0], trans[0][2], trans[1][2]};
    for (double c : cands)
      if (std::isfinite(c)) pmax = std::max(pmax, c);
    // Every finite intermediate is bounded by h*cap + 4*pmax: C values are minima,
    // hence at most the cost of a one- or two-stixel segmentation; W-row
    // differences P_k - W_j are sums of at most h terms in [-cap, 0]; shifted
    // predecessor terms C[j-1] + t - cap*j lie in [-cap*h, 4*pmax].
    double bound = (double)height * capQ + 4.0 * pmax;
    if (bound >= 16777216.0)
      return bail(STIXELS_ERR_UNSUPPORTED,
                  "exact mode range: h*cap + priors >= 2^24 quanta; lower cost_frac_bits (L#22)");
  }
  h->sparse = sparse;
  h->pair2d = pair2d;
  h->iw = iw;
  A.h = height; A.D = D; A.n_cols = h->n_cols; A.cap = h->cap;
  A.LG = LGr; A.gG_stride = sig_g.empty() ? 0 : LGr; A.LS = (int)gS.size(); A.esz = esz; A.dmr_inv = einv;
  A.ord_margin = params->ord_margin;
  A.capQ = (float)capQ;
  A.cost_scale = params->cost_frac_bits > 0 ? (float)std::ldexp(1.0, -params->cost_frac_bits) : 1.f;

  // ---------------- device ---------------------------------------------------
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return bail(STIXELS_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return bail(STIXELS_ERR_CUDA, std::string("cudaGetDeviceProperties: ") + cudaGetErrorString(e));
  if (prop.major != 10) return bail(STIXELS_ERR_CUDA, "this library is built for sm_100a (B200) only");
  h->sms = prop.multiProcessorCount;
  int optin = (int)prop.sharedMemPerBlockOptin;
  h->smem_optin = optin;
  auto kfun = [&](int cw) { return dp_kernel_ptr(h, cw); };
  auto cbytes = [&](int cw) {
    if (cw == 8)
      return DPv == 128 ? (sparse ? col_smem_bytes<128, true, 8>(height) : col_smem_bytes<128, false, 8>(height))
                        : (sparse ? col_smem_bytes<256, true, 8>(height) : col_smem_bytes<256, false, 8>(height));
    return DPv == 128 ? (sparse ? col_smem_bytes<128, true>(height) : col_smem_bytes<128, false>(height))
                      : (sparse ? col_smem_bytes<256, true>(height) : col_smem_bytes<256, false>(height));
  };
  int cb = cbytes(4);
  int sb = stx::kM2Pad + al16((height + 1) * 4) + (sparse ? stx::e_copies<true>() : stx::e_copies<false>()) * esz * 4 +
           al16(kTri * 2) +   // pad, M2, E copies, triangle decode
           (pair2d && sparse ? (DPv + 17) * 16 * 4 : 0) +  // NEXT f2 band weights
           al16(height * 8);                     // gravity thresholds per row
  int cpc = std::min(4, (optin - sb) / cb);   // columns per CTA (4 warps each)
  if (cpc < 1) return bail(STIXELS_ERR_UNSUPPORTED, "per-column shared memory exceeds the SM");
  h->cols_per_cta = cpc;
  h->smem = sb + cpc * cb;
  A.col_bytes = cb; A.shared_bytes = sb; A.cols_per_cta = cpc;
  e = cudaFuncSetAttribute(kfun(4), cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem);
  if (e != cudaSuccess) return bail(STIXELS_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfun(4), cpc * kCW * 32, h->smem);
  if (e != cudaSuccess || per_sm < 1) return bail(STIXELS_ERR_UNSUPPORTED, "dp_kernel does not fit on an SM");
  h->grid = h->sms * per_sm;
  // CW = 8 groups for batches of at most 2 columns per SM (latency): up to 2 per CTA,
  // within the scratch slots of the CW = 4 plan
  {
    const int cb8 = cbytes(8);
    const int cpc8 = std::min({2, cpc, (optin - sb) / cb8});
    if (cpc8 >= 1 && per_sm == 1 &&
        cudaFuncSetAttribute(kfun(8), cudaFuncAttributeMaxDynamicSharedMemorySize, sb + cpc8 * cb8) == cudaSuccess) {
      h->col_bytes8 = cb8;
      h->cols_per_cta8 = cpc8;
    }
  }
  // reduction tile
  const int in_bpp = bytes_per_px(params->disp_format);
  h->red_tc = std::max(1, std::min(h->n_cols, (in_bpp == 4 ? 256 : 512) / params->stixel_width));
  h->red_w2 = red_tile_words(h->red_tc, params->stixel_width, in_bpp);
  h->red_smem = kRedRows * h->red_w2 * 4;

  auto alloc = [&](void** ptr, size_t n) { return cudaMalloc(ptr, n); };
  if (pair2d && ((e = alloc((void**)&h->d_E2, E2.size() * 4)) != cudaSuccess ||
                  (e = alloc((void**)&h->d_WT, WT.size() * 4)) != cudaSuccess))
    return bail(STIXELS_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  if (pair2d) {
    cudaMemcpy(h->d_E2, E2.data(), E2.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(h->d_WT, WT.data(), WT.size() * 4, cudaMemcpyHostToDevice);
  }
  if ((e = alloc((void**)&h->d_E, E4.size() * 4)) != cudaSuccess ||
      (e = alloc((void**)&h->d_M2, M2.size() * 4)) != cudaSuccess ||
      (e = alloc((void**)&h->d_gG, gG.size() * 4)) != cudaSuccess ||
      (e = alloc((void**)&h->d_gS, gS.size() * 4)) != cudaSuccess ||
      (e = alloc((void**)&h->d_dgR, dgR.size() * 4)) != cudaSuccess ||
      (e = alloc((void**)&h->d_thr, thrg.size() * 4)) != cudaSuccess ||
      (e = alloc((void**)&h->d_overflow, 4)) != cudaSuccess ||
      (e = alloc((void**)&h->d_skipped, 8)) != cudaSuccess ||
      (e = alloc((void**)&h->d_scratch, h->scratch_bytes = (size_t)h->grid * cpc * 4 *
                        (DPv == 128 ? col_scratch_floats<128>(height) : col_scratch_floats<256>(height)))) != cudaSuccess ||
      (e = alloc((void**)&h->d_cols, (size_t)max_batch * h->n_cols * height * 2)) != cudaSuccess)
    return bail(STIXELS_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  cudaMemcpy(h->d_E, E4.data(), E4.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(h->d_M2, M2.data(), M2.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(h->d_gG, gG.data(), gG.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(h->d_gS, gS.data(), gS.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(h->d_dgR, dgR.data(), dgR.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(h->d_thr, thrg.data(), thrg.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(h->d_overflow, 0, 4);
  cudaMemset(h->d_skipped, 0, 8);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return bail(STIXELS_ERR_CUDA, std::string("table upload: ") + cudaGetErrorString(e));
  A.E = h->d_E; A.E2g = h->d_E2; A.WTg = h->d_WT; A.M2 = h->d_M2; A.gG = h->d_gG; A.gS = h->d_gS; A.dgR = h->d_dgR; A.thrg = h->d_thr;
  A.overflow = h->d_overflow;
  A.skipped = h->d_skipped;
  // exact chunk bound of the int32 kernel: on for columns of >= kBoundMinH rows
  // (B200 f1 sweep: +5% at h = 440, +15% at 880, +25% at 1024; -6% at 220, where
  // its per-column tables cost more than the few far chunks it skips) whose P2
  // table fits the eo words' free low halves (nb * DP / 8 <= h + 2)
  {
    constexpr int kBoundMinH = 320;
    const int nbk = (height + 31) / 32;
    h->bound_ok = iw && nbk * (DPv / 8) <= height + 2;
    h->bound_auto = h->bound_ok && height >= kBoundMinH;
    A.bound = h->bound_auto ? 1 : 0;
  }
  A.scratch = h->d_scratch;
  *out = h;
  return STIXELS_OK;
}

#ifdef STX_TRACE
// diagnostic build only: device buffer of 4*64*32 u64 for the phase timeline
extern "C" int stixels_trace_buffer(stixels_handle* h, void* d_buf) {
  if (!h) return STIXELS_ERR_ARG;
  h->args.trace = (unsigned long long*)d_buf;
  return STIXELS_OK;
}
#endif

int stixels_query(const stixels_handle* h, int* n_cols, int* cap) {
  if (!h) return STIXELS_ERR_ARG;
  if (n_cols) *n_cols = h->n_cols;
  if (cap) *cap = h->cap;
  return STIXELS_OK;
}

int stixels_query_kernel(const stixels_handle* h, int* variant, int* dp_slots, int* cols_per_cta) {
  if (!h) return STIXELS_ERR_ARG;
  if (variant)
    *variant = h->pair2d ? (h->sparse ? STIXELS_DP_PAIR2D : STIXELS_DP_PAIR2D_DENSE)
               : h->iw ? STIXELS_DP_INT32 : h->sparse ? STIXELS_DP_SPARSE : STIXELS_DP_DENSE;
  if (dp_slots) *dp_slots = h->dp_slots;
  if (cols_per_cta) *cols_per_cta = h->cols_per_cta;
  return STIXELS_OK;
}

static int launch_reduce(stixels_handle* h, const void* d_disp, int64_t pitch, int batch,
                         uint16_t* d_cols, cudaStream_t s) {
  ReduceArgs r;
  r.disp = (const uint8_t*)d_disp; r.pitch = pitch; r.W = h->W; r.H = h->H; r.n_cols = h->n_cols;
  r.bpp = bytes_per_px(h->p.disp_format);
  r.s = h->p.stixel_width; r.tc = h->red_tc; r.D = h->p.max_disparity;
  r.q_bits = r.bpp == 4 ? 8 : h->p.disp_frac_bits;   // f32: converted to the 1/256 grid (L#28)
  r.invalid = h->p.invalid_value;
  r.w2 = h->red_w2;
  r.vec = ((uintptr_t)d_disp % 16 == 0) && (pitch % 16 == 0);
  r.out = d_cols;
  dim3 grid((h->n_cols + h->red_tc - 1) / h->red_tc, (h->H + kRedRows - 1) / kRedRows, batch);
  const bool med = h->p.reduce_mode == STIXELS_REDUCE_MEDIAN;
  // row-wise register kernel for the common widths (16-byte aligned frames)
  if (r.vec && (r.s == 3 || r.s == 5 || r.s == 7 || r.s == 10)) {
    // strip kernel (TMA row streams) for full batches whose rows fit 2+ strip buffers
    const int rowb = (h->W * r.bpp + 15) & ~15;       // bytes copied per image row
    const int rs = rowb + (((rowb >> 4) & 1) ? 0 : 16); // smem row stride: odd multiple of 16 B
    const int nstrips = batch * ((h->H + 31) >> 5);
    const int stages = std::min(4, (h->smem_optin - kStripHdr - 128) / (32 * rs));
    const bool strip = rowb <= pitch && stages >= 2 && nstrips >= 4 * h->sms;
    auto go_rr = [&](auto kern, auto kstrip, int G) {
      const int ngroups = (h->n_cols + G - 1) / G;
      r.batch = batch;
      if (strip) {
        r.tma_rs = rs; r.tma_rowb = rowb; r.tma_stages = stages;
        const int smem = kStripHdr + stages * 32 * rs + 128;   // (+ slack: a ragged group's last loads)
        cudaFuncSetAttribute(kstrip, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int per = (ngroups + 14) / 15;                // compute warps: the same number of groups each
        const int nw = (ngroups + per - 1) / per;
        kstrip<<<std::min(nstrips, h->sms), 32 * (nw + 1), smem, s>>>(r);   // + the copy-issuing warp
        return;
      }
      const int rows_blocks = (h->H + 32 * kRRWarps - 1) / (32 * kRRWarps);
      // full batches: 8 groups per warp (loads of the next group in flight); a
      // batch of a few frames: one group per warp, so the grid covers the SMs and
      // the latency is one span's round trip (BASELINE configs[1])
      r.rr_groups = ((long)batch * rows_blocks * ((ngroups + kRRGroups - 1) / kRRGroups) >= 4L * h->sms)
                        ? kRRGroups : 1;
      dim3 g((ngroups + r.rr_groups - 1) / r.rr_groups, rows_blocks, batch);
      kern<<<g, 32 * kRRWarps, 0, s>>>(r);
    };
    // integer input with the sentinel at or above D 2^Q (e.g. 0xFFFF): one compare per pixel
    const bool invhi = r.bpp != 4 && r.invalid >= ((uint32_t)r.D << r.q_bits);
#define STX_RR2(MED, BPPV, SWV, IH) \
    go_rr(reduce_rows_kernel<MED, BPPV, SWV, IH>, reduce_strip_kernel<MED, BPPV, SWV, IH>, RowRed<BPPV, SWV>::G)
#define STX_RR(BPPV, SWV)                                                                        \
    if (r.bpp == BPPV && r.s == SWV) {                                                            \
      if (med) {                                                                                  \
        if (invhi && BPPV != 4) STX_RR2(true, BPPV, SWV, BPPV != 4);                              \
        else STX_RR2(true, BPPV, SWV, false);                                                     \
      } else {                                                                                    \
        if (invhi && BPPV != 4) STX_RR2(false, BPPV, SWV, BPPV != 4);                             \
        else STX_RR2(false, BPPV, SWV, false);                                                    \
      }                                                                                           \
    }
    STX_RR(2, 5) else STX_RR(2, 3) else STX_RR(2, 7) else STX_RR(2, 10)
    else STX_RR(1, 5) else STX_RR(1, 3) else STX_RR(1, 7) else STX_RR(1, 10)
    else STX_RR(4, 5) else STX_RR(4, 3) else STX_RR(4, 7) else STX_RR(4, 10)
#undef STX_RR2
#undef STX_RR
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(h, STIXELS_ERR_CUDA, std::string("reduce_rows_kernel: ") + cudaGetErrorString(e));
    return STIXELS_OK;
  }
  const bool s5 = r.s == 5;                          // the headline width, compile-time
  auto go = [&](auto kern) { kern<<<grid, kRedThreads, h->red_smem, s>>>(r); };
  if (r.bpp == 4) {
    if (med) go(reduce_kernel<true, 4, 0>); else go(reduce_kernel<false, 4, 0>);
  } else if (r.bpp == 2) {
    if (med) { if (s5) go(reduce_kernel<true, 2, 5>); else go(reduce_kernel<true, 2, 0>); }
    else { if (s5) go(reduce_kernel<false, 2, 5>); else go(reduce_kernel<false, 2, 0>); }
  } else {
    if (med) go(reduce_kernel<true, 1, 0>); else go(reduce_kernel<false, 1, 0>);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(h, STIXELS_ERR_CUDA, std::string("reduce_kernel: ") + cudaGetErrorString(e));
  return STIXELS_OK;
}

// Warps per column of the DP launch for `batch` frames: 8 (latency plan) when the
// batch has at most cols_per_cta8 columns per SM, else 4; or the forced plan.
static int plan_cw(const stixels_handle* h, int batch) {
  if (h->plan_cw) return h->plan_cw;
  const long need = ((long)batch * h->n_cols + h->sms - 1) / h->sms;
  return (h->cols_per_cta8 > 0 && need <= h->cols_per_cta8) ? 8 : kCW;
}

static int launch_dp(stixels_handle* h, const uint16_t* d_cols, int batch, stixel_t* d_out,
                     int32_t* d_count, float* d_cost, cudaStream_t s, float* scratch) {
  DPArgs A = h->args;
  A.scratch = scratch;
  A.cols = d_cols; A.out = d_out; A.count = d_count; A.col_cost = d_cost;
  A.items = batch * h->n_cols;
  // Column groups per CTA: the full count when the batch fills the GPU; fewer when
  // it does not (e.g. one frame: 204 columns for 148 SMs), so the columns spread
  // over more SMs instead of sharing a few; and then 8 warps per column (CW = 8),
  // which shortens the per-column critical path (latency, BASELINE configs[1]).
  const int need = (A.items + h->sms - 1) / h->sms;     // columns per SM
  const int cw = plan_cw(h, batch);
  const int C = std::max(1, std::min(cw == 8 ? h->cols_per_cta8 : h->cols_per_cta, need));
  A.cols_per_cta = C;
  A.bound = h->bound_mode == 0 ? (h->bound_auto ? 1 : 0) : (h->bound_mode == 2 ? 1 : 0);
  if (cw == 8) A.col_bytes = h->col_bytes8;
  const int smem = A.shared_bytes + C * A.col_bytes;
  int grid = std::min(h->grid, (A.items + C - 1) / C);
  const int threads = C * cw * 32;
  // launched with programmatic stream serialisation: its CTA-table setup may
  // overlap the preceding reduction; it waits (griddepcontrol.wait) before
  // reading the reduced columns
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&](auto kern) { cudaLaunchKernelEx(&cfg, kern, A); };
  dispatch_dp(h, cw, go);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(h, STIXELS_ERR_CUDA, std::string("dp_kernel: ") + cudaGetErrorString(e));
  h->last_cw = cw;
  h->last_cpc = C;
  return STIXELS_OK;
}

static int check_disp_args(stixels_handle* h, const void* d, int64_t pitch, int batch) {
  if (!h) return STIXELS_ERR_ARG;
  if (h->sticky) return h->sticky;
  int bpp = bytes_per_px(h->p.disp_format);
  if (!d || batch < 1 || batch > h->max_batch || pitch < (int64_t)h->W * bpp || (pitch % bpp))
    return fail(h, STIXELS_ERR_ARG, "bad input pointer, batch or row pitch");
  return STIXELS_OK;
}

int stixels_reduce(stixels_handle* h, const void* d_disp, int64_t pitch, int batch, uint16_t* d_cols) {
  int st = check_disp_args(h, d_disp, pitch, batch);
  if (st) return st;
  if (!d_cols) return fail(h, STIXELS_ERR_ARG, "d_cols is NULL");
  cudaSetDevice(h->device);
  h->launches = 1;
  return launch_reduce(h, d_disp, pitch, batch, d_cols, h->stream);
}

int stixels_solve(stixels_handle* h, const uint16_t* d_cols, int batch, stixel_t* d_out,
                  int32_t* d_count, float* d_cost) {
  if (!h) return STIXELS_ERR_ARG;
  if (h->sticky) return h->sticky;
  if (!d_cols || !d_out || !d_count || batch < 1 || batch > h->max_batch)
    return fail(h, STIXELS_ERR_ARG, "bad pointer or batch");
  cudaSetDevice(h->device);
  h->launches = 1;
  return launch_dp(h, d_cols, batch, d_out, d_count, d_cost, h->stream, h->d_scratch);
}

int stixels_compute(stixels_handle* h, const void* d_disp, int64_t pitch, int batch,
                    stixel_t* d_out, int32_t* d_count, float* d_cost) {
  int st = check_disp_args(h, d_disp, pitch, batch);
  if (st) return st;
  if (!d_out || !d_count) return fail(h, STIXELS_ERR_ARG, "output pointer is NULL");
  cudaSetDevice(h->device);
  h->launches = 2;
  st = launch_reduce(h, d_disp, pitch, batch, h->d_cols, h->stream);
  if (st) return st;
  return launch_dp(h, h->d_cols, batch, d_out, d_count, d_cost, h->stream, h->d_scratch);
}

int stixels_compute_host(stixels_handle* h, const void* h_disp, int64_t pitch, int batch,
                         stixel_t* h_out, int32_t* h_count, float* h_cost) {
  if (!h) return STIXELS_ERR_ARG;
  if (h->sticky) return h->sticky;
  int bpp = bytes_per_px(h->p.disp_format);
  if (!h_disp || !h_out || !h_count || batch < 1 || pitch < (int64_t)h->W * bpp || (pitch % bpp))
    return fail(h, STIXELS_ERR_ARG, "bad host pointer, batch or pitch");
  cudaSetDevice(h->device);
  if (!h->hscratch1) CU(cudaMalloc(&h->hscratch1, h->scratch_bytes), h);
  if (!h->ev_entry) CU(cudaEventCreateWithFlags(&h->ev_entry, cudaEventDisableTiming), h);
  // frames per H2D / compute / D2H stage: about 32, chosen so that the stage's
  // columns fill the column slots evenly (1024x440: 29 frames = 5916 columns =
  // 10 per slot on 588 of 592 slots; 32 frames would leave 16 slots a 12th column)
  int chunk = std::min(h->max_batch, 32);
  {
    const long slots = (long)h->grid * h->cols_per_cta;
    double best = -1.0;
    for (int f = std::min(h->max_batch, 40); f >= std::min(h->max_batch, 24); --f) {
      const long items = (long)f * h->n_cols;
      const double eff = (double)items / (double)(slots * ((items + slots - 1) / slots));
      if (eff > best + 1e-3) { best = eff; chunk = f; }
    }
  }
  const size_t in_b = (size_t)h->H * pitch;
  if (h->h_chunk != chunk || h->h_pitch != pitch) {
    for (int i = 0; i < 2; ++i) {
      cudaFree(h->hin[i]); cudaFree(h->hout[i]); cudaFree(h->hcnt[i]); cudaFree(h->hcost[i]);
      cudaFree(h->hcols[i]);
      h->hcols[i] = nullptr;
      h->hin[i] = nullptr; h->hout[i] = nullptr; h->hcnt[i] = nullptr; h->hcost[i] = nullptr;
      if (!h->hs[i]) CU(cudaStreamCreateWithFlags(&h->hs[i], cudaStreamNonBlocking), h);
      CU(cudaMalloc(&h->hin[i], in_b * chunk), h);
      CU(cudaMalloc(&h->hout[i], sizeof(stixel_t) * (size_t)chunk * h->n_cols * h->cap), h);
      CU(cudaMalloc(&h->hcnt[i], sizeof(int32_t) * (size_t)chunk * h->n_cols), h);
      CU(cudaMalloc(&h->hcost[i], sizeof(float) * (size_t)chunk * h->n_cols), h);
      CU(cudaMalloc(&h->hcols[i], 2 * (size_t)chunk * h->n_cols * h->H), h);
    }
    h->h_chunk = chunk;
    h->h_pitch = pitch;
  }
  // work already queued on the handle's stream (stixels_compute) uses d_scratch:
  // both stage streams start after it
  CU(cudaEventRecord(h->ev_entry, h->stream), h);
  CU(cudaStreamWaitEvent(h->hs[0], h->ev_entry, 0), h);
  CU(cudaStreamWaitEvent(h->hs[1], h->ev_entry, 0), h);
  int launches = 0;
  // the first stage is small (a quarter) so that compute starts after a short
  // copy; the rest are full stages
  const int first = std::max(1, chunk / 4);
  for (int b0 = 0, it = 0, nb = 0; b0 < batch; b0 += nb, ++it) {
    nb = std::min(it == 0 ? first : chunk, batch - b0);
    const int i = it & 1;
    cudaStream_t s = h->hs[i];
    const size_t items = (size_t)nb * h->n_cols;
    CU(cudaMemcpyAsync(h->hin[i], (const uint8_t*)h_disp + (size_t)b0 * in_b, in_b * nb,
                       cudaMemcpyHostToDevice, s), h);
    int st = launch_reduce(h, h->hin[i], pitch, nb, h->hcols[i], s);
    if (st) return st;
    st = launch_dp(h, h->hcols[i], nb, h->hout[i], h->hcnt[i], h->hcost[i], s,
                   i ? h->hscratch1 : h->d_scratch);
    if (st) return st;
    launches += 2;
    CU(cudaMemcpyAsync(h_out + (size_t)b0 * h->n_cols * h->cap, h->hout[i],
                       sizeof(stixel_t) * items * h->cap, cudaMemcpyDeviceToHost, s), h);
    CU(cudaMemcpyAsync(h_count + (size_t)b0 * h->n_cols, h->hcnt[i], sizeof(int32_t) * items,
                       cudaMemcpyDeviceToHost, s), h);
    if (h_cost)
      CU(cudaMemcpyAsync(h_cost + (size_t)b0 * h->n_cols, h->hcost[i], sizeof(float) * items,
                         cudaMemcpyDeviceToHost, s), h);
  }
  h->launches = launches;
  CU(cudaStreamSynchronize(h->hs[0]), h);
  CU(cudaStreamSynchronize(h->hs[1]), h);
  return stixels_sync(h);
}

int stixels_sync(stixels_handle* h) {
  if (!h) return STIXELS_ERR_ARG;
  cudaSetDevice(h->device);
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return fail(h, STIXELS_ERR_CUDA, std::string("sync: ") + cudaGetErrorString(e));
  int ov = 0;
  e = cudaMemcpy(&ov, h->d_overflow, 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fail(h, STIXELS_ERR_CUDA, std::string("sync: ") + cudaGetErrorString(e));
  if (ov) {
    cudaMemset(h->d_overflow, 0, 4);
    return fail(h, STIXELS_ERR_CAPACITY, "a column produced more stixels than max_stixels");
  }
  return h->sticky ? h->sticky : STIXELS_OK;
}

int stixels_last_launch_count(const stixels_handle* h) { return h ? h->launches : 0; }

int stixels_set_launch_plan(stixels_handle* h, int warps_per_column) {
  if (!h || (warps_per_column != 0 && warps_per_column != 4 && warps_per_column != 8))
    return STIXELS_ERR_ARG;
  if (warps_per_column == 8 && h->cols_per_cta8 < 1)
    return fail(h, STIXELS_ERR_UNSUPPORTED, "8 warps per column: shared memory too small for this shape");
  h->plan_cw = warps_per_column;
  return STIXELS_OK;
}

int stixels_skipped_cells(stixels_handle* h, unsigned long long* cells) {
  if (!h || !cells) return STIXELS_ERR_ARG;
  cudaSetDevice(h->device);
  CU(cudaStreamSynchronize(h->stream), h);
  if (h->hs[0]) CU(cudaStreamSynchronize(h->hs[0]), h);
  if (h->hs[1]) CU(cudaStreamSynchronize(h->hs[1]), h);
  CU(cudaMemcpy(cells, h->d_skipped, 8, cudaMemcpyDeviceToHost), h);
  return STIXELS_OK;
}

int stixels_set_chunk_bound(stixels_handle* h, int mode) {
  if (!h || mode < 0 || mode > 2) return STIXELS_ERR_ARG;
  if (mode == 2 && !h->bound_ok)
    return fail(h, STIXELS_ERR_UNSUPPORTED, "chunk bound: needs the int32 kernel and nb * DP / 8 <= height + 2");
  h->bound_mode = mode;
  return STIXELS_OK;
}

int stixels_query_launch(const stixels_handle* h, int* warps_per_column, int* cols_per_cta) {
  if (!h) return STIXELS_ERR_ARG;
  if (warps_per_column) *warps_per_column = h->last_cw;
  if (cols_per_cta) *cols_per_cta = h->last_cpc;
  return STIXELS_OK;
}

int stixels_destroy(stixels_handle* h) {
  if (!h) return STIXELS_OK;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  free_all(h);
  delete h;
  return STIXELS_OK;
}

}  // extern "C"
