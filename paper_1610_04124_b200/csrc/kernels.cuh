// kernels.cuh -- sm_100a device code of the stixel hot path.
//
// K1 reduce_kernel : column reduction + transpose, HBM-bound.
// K3 dp_kernel     : per-column prefix sums and object-LUT rows (P:163-177,
//                    P:207-219), the Eq. 5-6 min-plus DP (P:129-157,
//                    P:221-235) and fused backtracking.
//
// Design: a group of 4 warps per column, lanes own targets
// k in blocks of 32 ("lanes own targets"), bottoms j iterate warp-uniformly.  The
// object LUT LUT_object[f][v] (D x (h+1) per column, 220 KiB at 1024x440,
// P:209 "too large to fit into Shared Memory") is never materialised: the 32
// rows of the current target block live in shared memory ("priv"), and the row
// of the current bottom is carried incrementally in per-warp buffers updated
// only within the pair-cost band (row_{j+1} = row_j + Pair[.][d_j]).  Costs are
// fp32; in exact mode (L#22) they are integer quanta < 2^24, so every add and
// min is exact and decisions match the double-precision oracle bit for bit.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#include "../../include/stixels.h"

namespace stx {

constexpr int kRBits = 8;       // reduced disparities in units of 1/256 (L#8)
constexpr int kMaxH = 1024;
constexpr int kStart = 3;       // start marker class (first stixel)

// ---------------------------------------------------------------------------
// K1: column reduction + transpose (HBM-bound).
// One CTA = a tile of kRedRows image rows x (tc reduced columns) of one frame.
// The rows' byte range is read with 16-byte vector loads (rounded out to 16-byte
// boundaries) into a shared tile whose row stride is an odd number of words, so
// the transposed reads below -- 32 threads on 32 rows of one column -- are
// bank-conflict free.  Each thread then emits one reduced value (c, v),
// consecutive threads -> consecutive v (coalesced transposed writes).
// ---------------------------------------------------------------------------
constexpr int kRedRows = 32;
constexpr int kRedThreads = 256;

struct ReduceArgs {
  const uint8_t* disp;
  int64_t pitch;        // bytes
  int W, H, n_cols, s, tc, q_bits, D, bpp;
  int w2;               // tile row stride in 32-bit words (odd)
  int vec;              // 16-byte loads allowed (base and pitch 16-byte aligned)
  int rr_groups;        // reduce_rows_kernel: column groups walked per warp
  int batch;            // frames in this launch
  int tma_rs, tma_rowb; // reduce_strip_kernel: smem row stride (16 x odd bytes), bytes copied per row
  int tma_stages;       // reduce_strip_kernel: strip buffers in flight
  uint32_t invalid;
  uint16_t* out;        // [batch][n_cols][H], 0xFFFF = invalid
};
constexpr int kMedianMaxS = 64;

__host__ __device__ inline int red_tile_words(int tc, int s, int bpp) {
  return (((tc * s * bpp + 32 + 15) / 16 * 16) / 4) | 1;   // odd word stride
}

// SW > 0: the stixel width as a compile-time constant (the headline s = 5), 0: a.s
template <bool MEDIAN, int BPP, int SW>
__global__ void __launch_bounds__(kRedThreads) reduce_kernel(ReduceArgs a) {
  asm volatile("griddepcontrol.launch_dependents;");   // the DP kernel may start its setup
  const int sw = SW > 0 ? SW : a.s;
  extern __shared__ uint32_t tile32[];           // [kRedRows][w2] raw input bytes
  // floor(x / d) for d = 2n <= 2 kMedianMaxS... via a multiply-high by floor(2^32/d)
  // and one correction step (exact for 32-bit x); the table is per CTA
  __shared__ uint32_t rcp[2 * kMedianMaxS + 2];
  for (int i = threadIdx.x; i < 2 * kMedianMaxS + 2; i += kRedThreads)
    rcp[i] = i < 2 ? 0u : (uint32_t)((1ull << 32) / (unsigned)i);
  const int frame = blockIdx.z;
  const int r0 = blockIdx.y * kRedRows;
  const int c0 = blockIdx.x * a.tc;
  const int ncl = min(a.tc, a.n_cols - c0);
  const int px = ncl * sw;
  const int nrows = min(kRedRows, a.H - r0);
  const uint8_t* base = a.disp + (int64_t)frame * a.H * a.pitch + (int64_t)r0 * a.pitch;
  const int b0 = c0 * sw * BPP;                    // first byte of the tile in a row
  int off;                                         // element offset of pixel c0*s in the tile
  if (a.vec) {
    const int bs = b0 & ~15;
    const int be = (b0 + px * a.bpp + 15) & ~15;
    const int nvec = (be - bs) >> 4;
    off = (b0 - bs) / a.bpp;
    const int t = threadIdx.x;
    const int rstep = kRedThreads / nvec;
    const int v = t % nvec;
    const int rb = t / nvec;
    if (t < rstep * nvec) {
      // this thread's rows rb, rb + rstep, ...: four 16-byte loads in flight at a time
      for (int r0i = rb; r0i < nrows; r0i += 4 * rstep) {
        uint4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int rr = r0i + u * rstep;
          if (rr < nrows) x[u] = __ldg(reinterpret_cast<const uint4*>(base + (int64_t)rr * a.pitch + bs) + v);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int rr = r0i + u * rstep;
          if (rr < nrows) {
            uint32_t* d = tile32 + rr * a.w2 + 4 * v;
            d[0] = x[u].x; d[1] = x[u].y; d[2] = x[u].z; d[3] = x[u].w;
          }
        }
      }
    }
  } else {
    off = 0;
    for (int i = threadIdx.x; i < nrows * px; i += kRedThreads) {
      const int r = i / px, x = i - r * px;
      const uint8_t* row = base + (int64_t)r * a.pitch + b0;
      if constexpr (BPP == 4)
        tile32[r * a.w2 + x] = __ldg(reinterpret_cast<const uint32_t*>(row) + x);
      else if constexpr (BPP == 2)
        reinterpret_cast<uint16_t*>(tile32)[r * 2 * a.w2 + x] = __ldg(reinterpret_cast<const uint16_t*>(row) + x);
      else
        reinterpret_cast<uint8_t*>(tile32)[r * 4 * a.w2 + x] = __ldg(row + x);
    }
  }
  __syncthreads();
  const uint32_t lim = (uint32_t)a.D << a.q_bits;
  const int shift = kRBits + 1 - a.q_bits;
  for (int i = threadIdx.x; i < ncl * kRedRows; i += kRedThreads) {
    const int cl = i / kRedRows, rr = kRedRows - 1 - (i - cl * kRedRows);  // v ascending
    if (rr >= nrows) continue;
    const int e0 = off + cl * sw;
    const int rowe = rr * (4 / BPP) * a.w2 + e0;   // element index of the segment start
    // a pixel: its value in input units (f32: converted once to the 1/256 grid,
    // half up, L#28) and validity
    const float Df = (float)a.D;
    auto px_ok = [&](int x, uint32_t& u) -> bool {
      if constexpr (BPP == 4) {
        const float d = __uint_as_float(tile32[rowe + x]);
        const bool ok = d >= 0.f && d < Df;           // false for NaN and +-inf too
        u = ok ? (uint32_t)__float2int_rd(d * 256.f + 0.5f) : 0u;   // exact: d * 256 < 2^16
        return ok;
      } else {
        u = BPP == 2 ? reinterpret_cast<const uint16_t*>(tile32)[rowe + x]
                     : reinterpret_cast<const uint8_t*>(tile32)[rowe + x];
        return (u != a.invalid) && (u < lim);
      }
    };
    uint32_t sum = 0, n = 0;
#pragma unroll 5
    for (int x = 0; x < sw; ++x) {
      uint32_t u;
      const bool ok = px_ok(x, u);
      sum += ok ? u : 0u;
      n += ok ? 1u : 0u;
    }
    if (MEDIAN && n) {
      // median of the n valid values (L#24): the values of ranks (n-1)/2 and n/2
      // by rank counting (s <= 64, no sort), averaged with the mean's rounding
      const uint32_t k1 = (n - 1) >> 1, k2 = n >> 1;
      uint32_t va = 0, vb = 0;
      for (int x = 0; x < sw; ++x) {
        uint32_t u;
        if (!px_ok(x, u)) continue;
        uint32_t less = 0, leq = 0;
        for (int y = 0; y < sw; ++y) {
          uint32_t t;
          const bool ok = px_ok(y, t);
          less += (ok && t < u) ? 1u : 0u;
          leq += (ok && t <= u) ? 1u : 0u;
        }
        if (less <= k1 && k1 < leq) va = u;
        if (less <= k2 && k2 < leq) vb = u;
      }
      sum = va + vb;
      n = 2;
    }
    uint16_t val = 0xFFFF;
    if (n) {
      // round half up of 2^R*sum/(2^Q*n) = floor((sum*2^(R+1-Q) + n) / (2n)); 32-bit
      // when it cannot overflow (sum < 2^(31-shift))
      uint32_t q;
      if (sum < (1u << (31 - shift)) && n <= (uint32_t)kMedianMaxS) {
        const uint32_t num = (sum << shift) + n, d = 2u * n;
        q = __umulhi(num, rcp[d]);
        if (num - q * d >= d) ++q;                   // floor(2^32/d) under-estimates by <= 1
      } else {
        q = (uint32_t)((((uint64_t)sum << shift) + n) / (2ull * n));
      }
      // 16-bit columns, 0xFFFF = invalid: the top value 65535 (D = 256 with 8
      // fractional input bits only) is stored as 0xFFFE (L#27)
      val = (uint16_t)min(q, 0xFFFEu);
    }
    const int r = r0 + rr;
    const int v = a.H - 1 - r;
    a.out[((int64_t)frame * a.n_cols + c0 + cl) * a.H + v] = val;
  }
}

// ---------------------------------------------------------------------------
// K1 (row-wise variant, the default when its span fits): lanes own consecutive
// image rows; a column group is G = 16 / gcd(16, s bpp) consecutive reduced
// columns, whose bytes start 16-byte aligned and are NV = G s bpp / 16 vector
// loads straight into registers (no shared-memory tile); the pixels are unpacked
// at compile-time offsets.  Each warp walks kRRGroups groups of its 32 rows with
// the next group's loads in flight while it reduces the current one (a sector
// shared by two consecutive spans is an L1 hit of the same lane), and writes, per
// column, 32 consecutive model rows (64 bytes, coalesced).  Same arithmetic as reduce_kernel
// (decode and validity L#23/L#28, mean P:195 or median L#24, half-up rounding to
// 1/256, the 0xFFFE limit of L#27); the rounding division is a multiply-high by a per-CTA
// table floor(2^32 / d) and one correction step.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int rr_gcd(int x, int y) { return y == 0 ? x : rr_gcd(y, x % y); }
template <int BPP, int SW>
struct RowRed {
  static constexpr int G = 16 / rr_gcd(16, SW * BPP);    // reduced columns per thread
  static constexpr int NV = G * SW * BPP / 16;           // 16-byte loads per thread
};
constexpr int kRRWarps = 8;                              // warps (column groups) per CTA

constexpr int kRRGroups = 8;                             // column groups per warp (loop), full batches

// One span of G reduced columns (NV 16-byte words of one image row in registers)
// -> G reduced values of that row, written at out[g H]: decode and validity
// (L#23/L#28), the mean or median (L#24) of the valid pixels, half-up
// rounding to 1/256 (the 16-bit code 0xFFFF = invalid, top value 0xFFFE, L#27).
// The rounding division floor(num / d), d = 2n <= 2 SW, is a multiply-high by
// rcp[d] = ceil(2^32 / d), exact without a correction step: every valid pixel is
// below D 2^Q (integers) or D 256 (f32), so num < SW D 2^9 + SW < 2^21 and the
// error num (rcp[d] - 2^32/d) / 2^32 < 2^-11 stays below the gap 1/d to the next
// integer.  INVHI: the sentinel lies at or above D 2^Q, so a pixel is valid iff
// u < D 2^Q (one compare and one predicated add per pixel).  FULL: all G columns
// of the span exist (no per-column bound test).
template <int SW>
__device__ __forceinline__ void rr_rcp_init(uint32_t* rcp) {
  for (int i = threadIdx.x; i < 2 * SW + 2; i += blockDim.x)
    rcp[i] = i < 2 ? 0u : (uint32_t)(((1ull << 32) + (unsigned)i - 1) / (unsigned)i);
}
__device__ __forceinline__ void add_if_below(uint32_t& sn, uint32_t t, uint32_t lim) {
  // sn += t if t < lim (one compare, one predicated add)
  asm("{\n .reg .pred p;\n setp.lt.u32 p, %1, %2;\n @p add.u32 %0, %0, %1;\n}" : "+r"(sn) : "r"(t), "r"(lim));
}
template <bool MEDIAN, int BPP, int SW, bool INVHI, int NV, bool FULL>
__device__ __forceinline__ void rr_reduce_span(const uint32_t (&cur)[NV * 4], int c0, int n_cols,
                                               uint16_t* out, int H, const uint32_t* rcp, uint32_t lim,
                                               int shift, float Df, bool inv_hi, uint32_t invalid) {
  constexpr int G = NV * 16 / (SW * BPP);
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (!FULL && c0 + g >= n_cols) break;
    uint32_t u[SW];
    bool ok[SW];
    // sum and count of the valid pixels packed in one word: count in bits 24..,
    // sum (< SW 2^17 <= 2^21 for SW <= 16) below
    uint32_t sn = 0;
#pragma unroll
    for (int x = 0; x < SW; ++x) {
      const int e = g * SW + x;                        // pixel index in the span
      const uint32_t w = cur[(e * BPP) >> 2];
      if constexpr (BPP == 4) {
        const float d = __uint_as_float(w);
        ok[x] = d >= 0.f && d < Df;                    // false for NaN and +-inf too
        u[x] = ok[x] ? (uint32_t)__float2int_rd(d * 256.f + 0.5f) : 0u;   // L#28
        if (ok[x]) sn += u[x] + (1u << 24);
      } else {
        u[x] = BPP == 2 ? ((w >> (8 * ((e * 2) & 3))) & 0xffffu) : ((w >> (8 * (e & 3))) & 0xffu);
        // (the sentinel test is redundant when it is >= the range limit)
        if constexpr (INVHI) {
          ok[x] = u[x] < lim;
          if constexpr (!MEDIAN) {
            // t = u + 2^24 in one byte permute (pixel bytes, then 0x00, 0x01)
            const uint32_t t = BPP == 2 ? __byte_perm(w, 0x01000000u, ((e * 2) & 3) ? 0x7432u : 0x7410u)
                                        : __byte_perm(w, 0x01000000u, 0x7440u | (uint32_t)(e & 3));
            add_if_below(sn, t, lim + (1u << 24));
          } else if (ok[x]) {
            sn += u[x] + (1u << 24);
          }
        } else {
          ok[x] = (inv_hi || u[x] != invalid) && (u[x] < lim);
          if (ok[x]) sn += u[x] + (1u << 24);
        }
      }
    }
    uint32_t sum = sn & 0xffffffu, n = sn >> 24;
    if (MEDIAN && n) {
      const uint32_t k1 = (n - 1) >> 1, k2 = n >> 1;
      uint32_t va = 0, vb = 0;
#pragma unroll
      for (int x = 0; x < SW; ++x) {
        uint32_t less = 0, leq = 0;
#pragma unroll
        for (int y = 0; y < SW; ++y) {
          less += (ok[y] && u[y] < u[x]) ? 1u : 0u;
          leq += (ok[y] && u[y] <= u[x]) ? 1u : 0u;
        }
        if (ok[x] && less <= k1 && k1 < leq) va = u[x];
        if (ok[x] && less <= k2 && k2 < leq) vb = u[x];
      }
      sum = va + vb;
      n = 2;
    }
    // n = 0 is replaced by the invalid code
    const uint32_t q = __umulhi((sum << shift) + n, rcp[2 * n]);
    // (0xFFFF = invalid; the top value 65535 is stored as 0xFFFE, L#27)
    out[g * H] = n ? (uint16_t)min(q, 0xFFFEu) : (uint16_t)0xFFFF;
  }
}

// INVHI (integer input whose invalid sentinel lies at or above the range limit
// D 2^Q, e.g. 0xFFFF): a pixel is valid iff u < D 2^Q, one compare; the valid
// sum and count then take one predicated add per pixel (round 2: ~62 -> ~30
// lane-instructions per output value).
template <bool MEDIAN, int BPP, int SW, bool INVHI>
__global__ void __launch_bounds__(32 * kRRWarps, 4) reduce_rows_kernel(ReduceArgs a) {
  asm volatile("griddepcontrol.launch_dependents;");   // the DP kernel may start its setup
  using RR = RowRed<BPP, SW>;
  constexpr int G = RR::G, NV = RR::NV;
  __shared__ uint32_t rcp[2 * SW + 2];
  rr_rcp_init<SW>(rcp);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int r = (blockIdx.y * kRRWarps + (threadIdx.x >> 5)) * 32 + lane;   // image row
  const int frame = blockIdx.z;
  if (r >= a.H) return;
  const int cg0 = blockIdx.x * a.rr_groups;
  const int cg1 = min(cg0 + a.rr_groups, (a.n_cols + G - 1) / G);
  const uint8_t* row = a.disp + ((int64_t)frame * a.H + r) * a.pitch;
  const uint32_t lim = (uint32_t)a.D << a.q_bits;
  const int shift = kRBits + 1 - a.q_bits;
  const float Df = (float)a.D;
  const int v = a.H - 1 - r;
  const bool inv_hi = INVHI || a.invalid >= lim;
  // the span of column group cg into registers: NV vector loads, or element loads
  // within [0, W bpp) when it would overrun the row's pitch
  auto load_span = [&](int cg, uint32_t (&wv)[NV * 4]) {
    const int64_t sb = (int64_t)cg * G * SW * BPP;
    if (sb + NV * 16 <= a.pitch) {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(row + sb) + i);
        wv[4 * i] = x.x; wv[4 * i + 1] = x.y; wv[4 * i + 2] = x.z; wv[4 * i + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < NV * 4; ++i) wv[i] = 0u;
      const int lim_b = a.W * BPP - (int)sb;
#pragma unroll
      for (int e = 0; e < NV * 16 / BPP; ++e) {
        if (e * BPP < lim_b) {
          uint32_t x;
          if constexpr (BPP == 4) x = __ldg(reinterpret_cast<const uint32_t*>(row + sb) + e);
          else if constexpr (BPP == 2) x = __ldg(reinterpret_cast<const uint16_t*>(row + sb) + e);
          else x = __ldg(row + sb + e);
          wv[(e * BPP) >> 2] |= x << (8 * ((e * BPP) & 3));
        }
      }
    }
  };
  auto reduce_span = [&](const uint32_t (&cur)[NV * 4], int cg) {
    uint16_t* o = a.out + ((int64_t)frame * a.n_cols + cg * G) * a.H + v;
    if ((cg + 1) * G <= a.n_cols)
      rr_reduce_span<MEDIAN, BPP, SW, INVHI, NV, true>(cur, cg * G, a.n_cols, o, a.H, rcp, lim, shift, Df, inv_hi, a.invalid);
    else
      rr_reduce_span<MEDIAN, BPP, SW, INVHI, NV, false>(cur, cg * G, a.n_cols, o, a.H, rcp, lim, shift, Df, inv_hi, a.invalid);
  };
  // two span buffers in turn (no register copies): the next group's loads stay in
  // flight while the current one is reduced
  uint32_t bA[NV * 4], bB[NV * 4];
  int cg = cg0;
  if (cg < cg1) load_span(cg, bA);
  while (cg < cg1) {
    if (cg + 1 < cg1) load_span(cg + 1, bB);
    reduce_span(bA, cg);
    if (++cg >= cg1) break;
    if (cg + 1 < cg1) load_span(cg + 1, bA);
    reduce_span(bB, cg);
    ++cg;
  }
}


// ---------------------------------------------------------------------------
// K1 (strip variant, full batches): a persistent CTA per SM streams 32-row strips
// of a frame (whole image rows, W bpp bytes each) into shared memory with
// one-dimensional bulk copies (cp.async.bulk, the TMA engine; completion on an
// mbarrier per buffer), kTmaStages strips in flight, so DRAM sees whole-row
// requests.  Warps then reduce the strip exactly as reduce_rows_kernel does (lane
// = image row, NV 16-byte shared loads per column group, rr_reduce_span): the
// smem row stride is an odd multiple of 16 bytes, so the 8 rows a quarter-warp
// reads sit in distinct bank groups.  A producer warp refills a buffer once every
// compute warp has arrived on its `empty` mbarrier (no CTA-wide barrier).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
constexpr int kStripHdr = 256;          // bytes before the strip buffers: mbarriers (full, empty), rcp table

__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
template <bool MEDIAN, int BPP, int SW, bool INVHI>
__global__ void __launch_bounds__(512, 1) reduce_strip_kernel(ReduceArgs a) {
  asm volatile("griddepcontrol.launch_dependents;");   // the DP kernel may start its setup
  using RR = RowRed<BPP, SW>;
  constexpr int G = RR::G, NV = RR::NV;
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t full0 = (uint32_t)__cvta_generic_to_shared(sm);   // [NST] mbarriers: strip landed
  const uint32_t empty0 = full0 + 32;                               // [NST] mbarriers: strip consumed
  uint32_t* rcp = reinterpret_cast<uint32_t*>(sm + 64);
  const uint32_t buf0 = full0 + kStripHdr;
  const int NST = a.tma_stages;
  const int rs = a.tma_rs;
  const int nrb = (a.H + 31) >> 5;
  const int nstrips = a.batch * nrb;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x >> 5) - 1;   // compute warps; warp nw issues the bulk copies
  rr_rcp_init<SW>(rcp);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, nw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (wid == nw) {
    // producer: strip `it` of this CTA into buffer it % NST once its previous
    // occupant has been consumed by all compute warps
    if (lane == 0) {
      int it = 0;
      for (int strip = blockIdx.x; strip < nstrips; strip += gridDim.x, ++it) {
        const int st = it % NST;
        if (it >= NST) mbar_wait(empty0 + 8 * st, (uint32_t)((it / NST - 1) & 1));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads before async writes
        const int frame = strip / nrb, r0 = (strip - frame * nrb) << 5;
        const int nrows = min(32, a.H - r0);
        const uint32_t bar = full0 + 8 * st;
        mbar_expect_tx(bar, (uint32_t)(nrows * a.tma_rowb));
        const uint8_t* src = a.disp + ((int64_t)frame * a.H + r0) * a.pitch;
        for (int r = 0; r < nrows; ++r)
          bulk_g2s(buf0 + (uint32_t)((st * 32 + r) * rs), src + (int64_t)r * a.pitch, (uint32_t)a.tma_rowb, bar);
      }
    }
    return;
  }
  const int ngroups = (a.n_cols + G - 1) / G;
  const uint32_t lim = (uint32_t)a.D << a.q_bits;
  const int shift = kRBits + 1 - a.q_bits;
  const float Df = (float)a.D;
  const bool inv_hi = INVHI || a.invalid >= lim;
  int it = 0;
  for (int strip = blockIdx.x; strip < nstrips; strip += gridDim.x, ++it) {
    const int st = it % NST;
    mbar_wait(full0 + 8 * st, (uint32_t)((it / NST) & 1));
    const int frame = strip / nrb, r = ((strip - frame * nrb) << 5) + lane;
    if (r < a.H) {
      const uint32_t rowa = buf0 + (uint32_t)((st * 32 + lane) * rs);
      uint16_t* outr = a.out + (int64_t)frame * a.n_cols * a.H + (a.H - 1 - r);
      for (int cg = wid; cg < ngroups; cg += nw) {
        uint32_t cur[NV * 4];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const uint4 x = lds128(rowa + (uint32_t)(cg * NV * 16 + 16 * i));
          cur[4 * i] = x.x; cur[4 * i + 1] = x.y; cur[4 * i + 2] = x.z; cur[4 * i + 3] = x.w;
        }
        uint16_t* o = outr + (int64_t)cg * G * a.H;
        if ((cg + 1) * G <= a.n_cols)
          rr_reduce_span<MEDIAN, BPP, SW, INVHI, NV, true>(cur, cg * G, a.n_cols, o, a.H, rcp, lim, shift, Df,
                                                           inv_hi, a.invalid);
        else
          rr_reduce_span<MEDIAN, BPP, SW, INVHI, NV, false>(cur, cg * G, a.n_cols, o, a.H, rcp, lim, shift, Df,
                                                            inv_hi, a.invalid);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * st);   // this warp is done with buffer st
  }
}

// ---------------------------------------------------------------------------
// K3: DP kernel (prefix sums + object-LUT rows + Eq. 5-6 DP + backtracking).
//
// Work unit: one column, handled by a "column group" of kCW = 4 warps with its
// own named barriers (up to 4 groups per CTA, one CTA per SM).  Lanes own targets
// k = K0 + lane of a 32-row block b (K0 = 32 b).  The object LUT LUT_object[f][v]
// (D x (h+1)) is never materialised: per block, the 32 target rows
// priv[i][f] = W[f][K0+i+1] (W = LUT - cap * v, see below) live in shared memory,
// and the bottom row W[.][j] is carried incrementally in per-warp buffers seeded
// from an anchor row (W_{j+1} = W_j + band of Pair[.][d_j]).
//
// Roles.  Warp 0 (the "serial" warp) runs, per block, the part of Eq. 6 that is
// inherently sequential: targets K0 < j <= k in the same block need C[.][j-1]
// of the step before (the paper's barrier per step), done here in
// registers with warp shuffles; it also finalises each target -- ground and sky
// running minima (their data term does not depend on the predecessor, so
// GR^k = PG[k+1] + min_j (C_O[j-1] + t - PG[j])), the index table and the
// 32-byte record of row k+1 that later rectangles read (the candidate prior as a
// step function of the object mean f).  Meanwhile warps 1-2 build block b+1's
// priv rows and warps 1-3 (the "rectangle" warps) evaluate every cell of block
// b+1's targets whose bottom is already final (j <= K0), in 32-row chunks handed
// out dynamically; warp 0 joins them after its triangle.  Only the newest chunk
// (bottoms of block b) waits for warp 0: warps 0-1 take 16 rows each while warps
// 2-3 precompute block b+1's triangle cells.  (Latency plan, CW = 8: 7 rectangle
// warps, the newest chunk as 4 x 8 rows, the precompute in phase 1 into a second
// cell buffer.)
// Exact mode (L#22): all costs are integer quanta < 2^24 (int32 x 32 in the
// IW rectangle and chain, integer-valued fp32 elsewhere), so adds and mins are
// exact and every decision matches the oracle.
// ---------------------------------------------------------------------------
constexpr int kCW = 4;                 // warps per column
// IW scale: priv rows, W-rows and the records' predecessor terms are int32 quanta
// x 32, and each record carries (j - 1) & 31 of its row in the low 5 bits.  A
// candidate p - w + min(aO, aG) is then (cost x 32) | offset of its bottom in the
// 32-row block, so one IMNMX keeps the run's minimum and its first bottom; the
// argmin is decoded once per run.  |cost| < 2^25 (the host's 2^24 check), so the
// scaled values stay below 2^30.
constexpr int kIWS = 32;
// A record term at or beyond 2^24 quanta (an INF prior: a forbidden transition)
// is stored as 2^30: p - w <= 0 keeps every candidate built on it below 2^30 (no
// overflow) and above any finite cost; unscaled costs >= 2^24 read back as INF.
constexpr int kIWBig = 1 << 30;
// The serial chain's INF: finite costs are below 2^24 quanta (host check), so
// x 32 below 2^29; sums of three terms each <= 2^29 cannot overflow.
constexpr int kChainBig = 1 << 29;

// Diagnostic phase timeline (build with -DSTX_TRACE; scripts/trace_phases.py):
// CTA 0's column groups record %globaltimer stamps (ns; one clock for all SM
// sub-partitions) of their first column's phases.
#ifdef STX_TRACE
__device__ __forceinline__ unsigned long long stx_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define STX_STAMP(blk, slot)                                                             \
  do {                                                                                   \
    if (blockIdx.x == 0 && trace_item && lane == 0 && (blk) < 64)                        \
      a.trace[(cslot * 64 + (blk)) * 32 + (slot)] = stx_globaltimer();                  \
  } while (0)
#else
#define STX_STAMP(blk, slot) do { } while (0)
#endif

struct DPArgs {
  const uint16_t* cols;    // [items][h] reduced columns (model order), 0xFFFF invalid
  stixel_t* out;           // [items][cap]
  int32_t* count;          // [items]
  float* col_cost;         // [items] or null
  float* scratch;          // [grid*cols_per_cta][2][h+1]  ground / sky prefix sums
  const float* E;          // [4][esz] object pair-cost windows (host built; sparse mode loads copy 0)
  const uint32_t* M2;      // [h+1] magic reciprocals ceil(2^31/n)
  const float* gG;         // ground cost by |dR - dgR|, length LG (last = cap); with a
                           // row-dependent sigma_G(v) (NEXT f2) one table per row v at
                           // gG + v * gG_stride (gG_stride = 0: one shared table)
  const float* gS;         // sky cost by dR, length LS (last = cap)
  const int* dgR;          // [h] ground model, 1/256 units
  const uint32_t* thrg;    // [h] thrA1 | thrB << 16 (global copy for divergent reads)
  int* overflow;
  int h, D, n_cols, items, cap, LG, LS, esz, dmr_inv, ord_margin, cols_per_cta;
  int col_bytes, shared_bytes;   // smem layout
  float capQ, cost_scale;
  float piFirstO, piFirstG;      // first-stixel priors (incl. BIC)
  float kOO_lo, kOO_hi;          // O above O: trans + ordering (lo: no violation)
  float kGO_mid, kGO_hi, kGO_lo; // O above G: trans + gravity level
  float kOG, kGS, kOS;           // G above O, S above G, S above O
  float wt[16];                  // sparse W-row update: cap - Pair(d) for d = -7..7
  int thrA1[kMaxH];              // per row j: f >= thrA1[j] <=> floating object at base j
  int thrB[kMaxH];               //            f <  thrB[j]  <=> object below ground at base j
  // NEXT f2 tables (PAIR2D instantiation only)
  const float* E2g;        // NEXT f2, sigma_O(f): [D+2][DP] rows E'[d][f] = Pair[f][d] - cap
                           // for pixel disparity d = 0..D, row D+1 = 0 (invalid pixel)
  const float* WTg;        // NEXT f2: [DP+17][16] band weights cap - Pair[d+o-7][d] at row d+1
  int gG_stride;
  unsigned long long* skipped;   // IW: cumulative rectangle cells skipped by the chunk bound (or null)
  int bound;                     // IW: chunk bound on (host: columns of >= kBoundMinH rows)
#ifdef STX_TRACE
  unsigned long long* trace;     // diagnostic build only: [4 groups][64 blocks][32] globaltimer stamps
#endif
};

struct ColSmem {
  float* priv;      // [32][DP+1]     priv[i][f] = LUT_object[f][32b+i+1] of the block being built
  float* seed;      // [2][NSEED][DP] W-rows 32b+8i (i >= 1) of block b (slot b & 1): the
                    // newest chunk's seeds (NSEED = 1 for CW = 4, 3 for CW = 8)
  float* ring;      // [4][ring_stride] per-warp W-rows W_j = LUT_object[.][j] - cap*j (RR = 2 sparse, 4 dense)
  float4* cell;     // [496]          triangle cells (bottom K0+1+j', target K0+k' > j'), one
                    //                16-byte record each (one LDS.128 in the serial chain):
                    //                {object data term, the same plus its O-above-G prior
                    //                (gravity level), object mean f (int bits), unused}
  uint4* rec;       // [h+3][2]       row j: {V0,V1,V2,V3} {T[j], N4[j], b1 | b2<<16, b3 | cb<<10 | drp<<16}
                    //                (the prior of a bottom-j candidate as a step function of
                    //                the object mean f: V_i on [b_i, b_i+1), see write_record)
                    //                ({T, N4} also read per lane as a uint2: tn_at)
  uint32_t* eo;     // [h+2]          lo16: ring window byte offset; hi16: E0 byte offset
  uint16_t* argO;   // [h]            j | c'<<12
  uint16_t* argG;   // [h]            j (pred class O, or start if j == 0)
  uint16_t* argS;   // [h]            j | c'<<12
  uint8_t* fpv;     // [h]            f of the last stixel of the best O-ending segmentation
  float2* part;     // [4][32]        partial minima {cost, argj} of the 4 warps
  float4* pgps;     // [32]           serial warp: {PG[k], PG[k+1], PS[k], PS[k+1]}
  int* ctr;         // [1]            dynamic chunk counter
  int* ub;          // [32]           IW: per-target best candidate so far of the block's bulk chunks
                    //                (shifted, unscaled quanta), the chunk bound's upper side
  int* gmin;        // [nb+1]         IW: G[m] = min over chunk m's bottoms j of (least prior term of
                    //                record j + wtmax j), the chunk bound's lower side
                    // (and, IW only, the lo16 halves of eo -- the dense ring's window offsets,
                    // unused by the sparse kernels -- hold P2[b][c], b >= 1: the valid pixels
                    // of rows < 32 b whose object disparity falls in bins c or c+1 of 8)
};

constexpr int kTri = 496;              // cells of a 32-row triangle: sum_{j'<31} (31 - j')
__host__ __device__ constexpr int tri_off(int jp) { return 31 * jp - (jp * (jp - 1)) / 2; }

__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }

// Floats of W-row ring per warp.  Sparse mode: two W-row buffers, each with guard
// entries f in [-8, 0) and [DP, DP + 24) so band rounds need no range test (f of
// a valid pixel lies in [-8, DP + 8), the invalid code no_band() lands in
// [DP + 8, DP + 24)); buffer 0's f = 0 at float 8, buffer 1's at DP + 56 (16 banks
// apart, so the two half-warps of a band round -- nearly equal f -- do not
// conflict).
template <int DP, bool SPARSE>
__host__ __device__ constexpr int ring_stride() { return SPARSE ? 2 * DP + 80 : 4 * DP; }
template <int DP, bool SPARSE>
__host__ __device__ constexpr uint32_t ring_b0() { return SPARSE ? 8 * 4u : 0u; }
template <int DP, bool SPARSE>
__host__ __device__ constexpr uint32_t ring_b1() { return (DP + 48) * 4u; }   // from buffer 0
template <int DP>
__host__ __device__ constexpr int no_band() { return DP + 16; }   // drp code: invalid pixel
// priv row stride (floats): == 17 mod 32.  A rectangle gather reads 16 target rows
// t at their means f_t, bank (17 t + f_t) mod 32: targets whose means differ by one
// or two (the common case on one surface) collide only for (t, t') = (0, 15) or
// |t - t'| = 2 with |f - f'| = 2.  Simulated on C3 columns (scripts/micro/
// stride_sim.py): 1.075 wavefronts per gather (3 mod 32: 1.54, 1 mod 32: 1.90,
// matching ncu); B200 A/B: +0.45%.
template <int DP>
__host__ __device__ constexpr int priv_stride() { return DP + 17; }
// E' copies in shared memory: the dense ring reads 4 shifted copies, the sparse
// path (build only) one.
template <bool SPARSE>
__host__ __device__ constexpr int e_copies() { return SPARSE ? 1 : 4; }

// Warps sharing the newest chunk (the 32 bottoms of the block just finalised):
// 2 x 16 rows with 4 warps per column, 4 x 8 rows with 8 (latency plan).
__host__ __device__ constexpr int newest_warps(int cw) { return cw == 8 ? 4 : 2; }
// Triangle-cell buffers: the latency plan (CW = 8) precomputes block b+1's cells
// while the serial warp still reads block b's, so it double-buffers them.
__host__ __device__ constexpr int cell_bufs(int cw) { return cw == 8 ? 2 : 1; }
template <int DP, bool SPARSE, int CW = kCW>
__host__ __device__ inline int col_smem_bytes(int h) {
  int b = 0;
  b += al16(32 * priv_stride<DP>() * 4);
  b += al16((2 * newest_warps(CW) - 2) * DP * 4);
  b += al16(CW * ring_stride<DP, SPARSE>() * 4);
  b += kTri * 16 * cell_bufs(CW);
  b += al16((h + 3) * 32);
  b += al16((h + 2) * 4);
  b += al16(h * 2) * 3;
  b += al16(h);
  b += al16(CW * 32 * 8);
  b += al16(32 * 16);
  b += 16;          // ctr
  b += 32 * 4;      // ub
  b += al16((((h + 31) >> 5) + 1) * 4);   // gmin
  return b;
}
// IW chunk bound: disparity bins of 8 (pixel-count prefixes per bin pair at block
// boundaries)
template <int DP>
__host__ __device__ constexpr int bound_bins() { return DP / 8; }
// global scratch per column slot: PG[h+1], PS[h+1], anchor rows [nb+1][DP]
template <int DP>
__host__ __device__ inline int64_t col_scratch_floats(int h) {
  return 2 * (int64_t)(h + 1) + (int64_t)(((h + 31) >> 5) + 1) * DP;
}

template <int DP, bool SPARSE, int CW>
__device__ inline ColSmem carve(uint8_t* p, int h) {
  ColSmem w;
  w.priv = reinterpret_cast<float*>(p); p += al16(32 * priv_stride<DP>() * 4);
  w.seed = reinterpret_cast<float*>(p); p += al16((2 * newest_warps(CW) - 2) * DP * 4);
  w.ring = reinterpret_cast<float*>(p); p += al16(CW * ring_stride<DP, SPARSE>() * 4);
  w.cell = reinterpret_cast<float4*>(p); p += kTri * 16 * cell_bufs(CW);
  w.rec = reinterpret_cast<uint4*>(p); p += al16((h + 3) * 32);
  w.eo = reinterpret_cast<uint32_t*>(p); p += al16((h + 2) * 4);
  w.argO = reinterpret_cast<uint16_t*>(p); p += al16(h * 2);
  w.argG = reinterpret_cast<uint16_t*>(p); p += al16(h * 2);
  w.argS = reinterpret_cast<uint16_t*>(p); p += al16(h * 2);
  w.fpv = p; p += al16(h);
  w.part = reinterpret_cast<float2*>(p); p += al16(CW * 32 * 8);
  w.pgps = reinterpret_cast<float4*>(p); p += al16(32 * 16);
  w.ctr = reinterpret_cast<int*>(p); p += 16;
  w.ub = reinterpret_cast<int*>(p); p += 32 * 4;
  w.gmin = reinterpret_cast<int*>(p);
  return w;
}

__device__ __forceinline__ float warp_incl_scan(float x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    float y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Register copy the compiler cannot rematerialise as a constant-bank load
// (keeps selects between kernel-parameter constants branch-free): a shuffle
// result is opaque to ptxas.
__device__ __forceinline__ float opaque(float x) { return __shfl_sync(0xffffffffu, x, 0); }

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

constexpr int kM2Pad = 16;          // bytes of shared memory before the M2 table

// Object model value f of span [j, k] from prefix differences:
// f = floor(t / (256 n)), t = sum(d + 128) over valid pixels: the exact half-up
// rounded mean (L#10), via a multiply-high by ceil(2^31/n) (exact for t < 2^28).
// No clamp is needed: every object disparity is below D - 1/2 (L#27), so is their
// rounded mean.  n4 = 4n is the byte offset into M2 (kM2Pad bytes into dynamic smem).
__device__ __forceinline__ int span_f(uint32_t t, uint32_t n4, const uint8_t* smem0, int Dm1) {
  uint32_t y = t >> (kRBits - 1);
  uint32_t M = *reinterpret_cast<const uint32_t*>(smem0 + kM2Pad + n4);
  (void)Dm1;
  return (int)__umulhi(y, M);
}

__device__ __forceinline__ float ldsf(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

// Per-row uniform values of record j for the cell evaluation.
struct RowU {
  float V0, V1, V2, V3;            // min over predecessor classes of (C[j-1] + prior), shifted
                                   // by -cap*j, for f < b1, [b1, b2), [b2, b3), >= b3
  uint32_t T, N4;
  int b1, b2, b3, cb;              // breakpoints; cb bit i: the winner of interval i is O (else G)
  int drp;                         // drp = round(d_j) + 1, no_band<DP>() if pixel j is invalid
};
__device__ __forceinline__ RowU unpack_row(uint4 x, uint4 y) {
  RowU u;
  u.V0 = __uint_as_float(x.x); u.V1 = __uint_as_float(x.y);
  u.V2 = __uint_as_float(x.z); u.V3 = __uint_as_float(x.w);
  u.T = y.x; u.N4 = y.y;
  u.b1 = (int)(y.z & 0xffffu); u.b2 = (int)(y.z >> 16);
  u.b3 = (int)(y.w & 0x3ffu); u.cb = (int)((y.w >> 10) & 0xfu); u.drp = (int)(y.w >> 16);
  return u;
}
__device__ __forceinline__ RowU load_row(const uint4* rec, int j) {
  const uint32_t ra = (uint32_t)__cvta_generic_to_shared(rec + 2 * j);
  return unpack_row(lds128(ra), lds128(ra + 16));
}
// Plain (compiler-visible) version: records are read-only while a rectangle runs.
__device__ __forceinline__ RowU load_row_c(const uint4* rec, int j) {
  return unpack_row(rec[2 * j], rec[2 * j + 1]);
}
template <typename T>
__device__ __forceinline__ T* shp(uint32_t a) {     // shared u32 address -> pointer
  return reinterpret_cast<T*>(__cvta_shared_to_generic(a));
}

// Packed fp32x2 add (sm_100 FADD2): two independent adds in one instruction.
__device__ __forceinline__ void fadd2_inplace(float& a0, float& a1, float b0, float b1) {
  unsigned long long x, y, z;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b0), "f"(b1));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(z) : "l"(x), "l"(y));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(z));
}

// ---------------------------------------------------------------------------
// W-rows.  The kernel never stores LUT_object[f][v] itself but the shifted row
// W[f][v] = LUT_object[f][v] - cap * v = -sum_{u<v} (cap - Pair[f][d_u]), whose
// increments are zero except within +-band of the pixel's disparity (Eq. 4 hits
// the outlier cap): an object span's data term is
//   LUT[f][k+1] - LUT[f][j] = W[f][k+1] - W[f][j] + cap * (k+1-j).
// The per-target constant cap*(k+1) is dropped from rectangle candidates (it
// does not change the argmin over bottoms of one target) and the per-bottom
// constant -cap*j is folded into the bottom's record.  All values stay exact
// integers in exact mode (|.| <= 2 h cap < 2^24, checked on the host).
// ---------------------------------------------------------------------------
// NEXT f2 (PAIR2D, any noise table given): the object noise depends on the
// object's disparity f, sigma_O(f), so Pair[f][d] is a genuine 2-D table
// (P:175): the W-row band weights come from a [drp][offset] table in shared
// memory and the block W-rows from the full [d][f] table in global memory
// (L2-resident); the ground cost table is per row (sigma_G(v)).  The default
// instantiation (PAIR2D = false) keeps the 1-D |f - d| form.
template <int DP>
__host__ __device__ constexpr int wt_rows() { return DP + 17; }   // drp 0 .. no_band()

// IW (sparse, band <= 3, exact mode only): the rectangle's W-row buffers hold int32
// quanta, and the four pixel updates of a bottom pair are one round of native
// shared-memory integer atomics on 8-lane groups (float atomics would be CAS
// loops).  Exact: every W entry is an integer number of quanta below 2^24 (L#22),
// so the order of the adds does not matter and the gathers convert exactly.
// CW: warps per column group -- kCW = 4 (4 groups per CTA) when the batch fills the
// GPU; 8 (at most 2 groups per CTA) for small batches, where the per-column
// critical path (the frame latency, BASELINE configs[1]) rather than throughput binds.
template <int DP, bool SPARSE, bool PAIR2D, bool IW = false, int CW = kCW>
__global__ void __launch_bounds__(32 * kCW * 4, 1) dp_kernel(const __grid_constant__ DPArgs a) {
  constexpr int NR = DP / 128;         // LDS.128 ring windows per lane
  constexpr int NS = DP / 32;          // 32-wide f slices
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  // Warp roles: the C serial warps take the highest warp ids (the issue arbiter
  // prefers high ids; SMSP = wid % 4), the 3C rectangle warps the rest, spread so
  // that a column's warps sit on different SM sub-partitions where possible.
  const int C = a.cols_per_cta;
  int cslot, w;
  if (wid >= (CW - 1) * C) {
    cslot = wid - (CW - 1) * C; w = 0;
  } else if (CW == 4 && C == 4) {
    cslot = ((wid & 3) + (wid >> 2) + 1) & 3; w = 1 + (wid >> 2);
  } else {
    cslot = wid % C; w = 1 + wid / C;
  }
  const int ctid = w * 32 + lane;      // thread index within the column group
  const int h = a.h;
  const int Dm1 = a.D - 1;
  const int nb = (h + 31) >> 5;
  const float capQ = a.capQ;
  // IW serial chain: exact-mode costs as int32 quanta x 32 (below kChainBig = 2^29,
  // L#22's 2^24 bound), INF (a forbidden transition) saturated to kChainBig
  auto toI = [](float x) { return x >= 16777216.f ? kChainBig : __float2int_rn(x) * kIWS; };
  const int capI = IW ? __float2int_rn(capQ) * kIWS : 0;
  const int goHiI = toI(a.kGO_hi), goLoI = toI(a.kGO_lo), goMidI = toI(a.kGO_mid);
  const int bar_col = 1 + cslot;       // 128 threads: whole column group
  const int bar_rect = 1 + C + cslot;  // (CW - 1) * 32 threads: rectangle warps
  const int bar_x = 1 + 2 * C + cslot; // 96 arrive + 32 sync: next block's priv rows ready

  // CTA-shared tables: M2 at offset 0, then 4 shifted copies of the object
  // pair-cost window E' (Pair[f][d] - cap = E'[f - d + D]), then the
  // triangle cell decode table.
  // M2 sits kM2Pad bytes in: the rectangle's look-ahead rows may read up to 8
  // bytes before it (their value is never used)
  uint32_t* M2s = reinterpret_cast<uint32_t*>(smem + kM2Pad);
  float* E = reinterpret_cast<float*>(smem + kM2Pad + al16((h + 1) * 4));
  uint16_t* tri_jk = reinterpret_cast<uint16_t*>(smem + kM2Pad + al16((h + 1) * 4) + e_copies<SPARSE>() * a.esz * 4);
#pragma unroll 1
  for (int i = threadIdx.x; i <= h; i += blockDim.x) M2s[i] = a.M2[i];
  // IW: the object pair-cost window in int32 quanta (exact-mode costs are integers)
#pragma unroll 1
  for (int i = threadIdx.x; i < e_copies<SPARSE>() * a.esz; i += blockDim.x) {
    if constexpr (IW) reinterpret_cast<int*>(E)[i] = __float2int_rn(a.E[i]) * kIWS;
    else E[i] = a.E[i];
  }
  float* WT = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(tri_jk) + al16(kTri * 2));
  if constexpr (PAIR2D && SPARSE)
    for (int i = threadIdx.x; i < wt_rows<DP>() * 16; i += blockDim.x) WT[i] = a.WTg[i];
  // gravity thresholds {thrA1[j], thrB[j]} per row (one LDS.64 per row in the rectangle)
  int2* thrS = reinterpret_cast<int2*>(reinterpret_cast<uint8_t*>(WT) + (PAIR2D && SPARSE ? wt_rows<DP>() * 16 * 4 : 0));
#pragma unroll 1
  for (int i = threadIdx.x; i < h; i += blockDim.x) thrS[i] = make_int2(a.thrA1[i], a.thrB[i]);
  const uint32_t thr_s = (uint32_t)__cvta_generic_to_shared(thrS);
#pragma unroll 1
  for (int jp = 0; jp < 31; ++jp)                 // triangle cell index -> (j', k')
    for (int kp = jp + 1 + (int)threadIdx.x; kp < 32; kp += blockDim.x)
      tri_jk[tri_off(jp) + kp - jp - 1] = (uint16_t)(jp | (kp << 8));
  __syncthreads();
  const uint8_t* Eb = reinterpret_cast<const uint8_t*>(E);
  // programmatic dependent launch: everything above (CTA tables) overlaps the
  // reduction kernel's tail; the reduced columns are read only after this wait
  asm volatile("griddepcontrol.wait;" ::: "memory");

  ColSmem cs = carve<DP, SPARSE, CW>(smem + a.shared_bytes + cslot * a.col_bytes, h);
  // {T[j], N4[j]} of row j: the first 8 bytes of the record's second half
  auto tn_at = [&](int j) { return *reinterpret_cast<const uint2*>(cs.rec + 2 * j + 1); };
  // triangle cells of block bt (double-buffered in the latency plan)
  auto cells_of = [&](int bt) { return cs.cell + (cell_bufs(CW) == 2 ? (bt & 1) * kTri : 0); };
  float* ringw = cs.ring + w * ring_stride<DP, SPARSE>();
  const float INF = __int_as_float(0x7f800000);
  const int slot_global = blockIdx.x * a.cols_per_cta + cslot;
  float* PGg = a.scratch + (int64_t)slot_global * col_scratch_floats<DP>(h);
  float* PSg = PGg + (h + 1);
  float* ANg = PSg + (h + 1);          // anchor W-rows W[.][32m], global (L2)
  // IW chunk bound (L2): P2[b][c] = valid pixels of rows < 32 b whose object
  // disparity falls in bins c or c+1 (of 8), G[m] = min over chunk m's bottoms j
  // of (min prior term of record j + wtmax j)
  constexpr int NBIN = bound_bins<DP>();
  // P2[b][c] (b >= 1) in the lo16 half of eo word (b - 1) NBIN + c; P2[0][.] = 0
  uint16_t* P2s = reinterpret_cast<uint16_t*>(cs.eo);
  auto p2_at = [&](int b, int c) { return b > 0 ? (int)P2s[2 * ((b - 1) * NBIN + c)] : 0; };
  const bool bound = IW && a.bound;    // host: tall enough columns
  const int wtmax = IW ? (int)a.wt[7] : 0;   // cap - Pair(0): the largest band weight (quanta)
  constexpr int kUBInf = 0x3fffffff;
  unsigned long long skipped = 0;      // cells of chunks skipped by this warp

  // sparse update lanes: lanes 0-14 serve W-row buffer 1 (odd bottoms), lanes
  // 16-30 buffer 0 (even bottoms); each owns one offset d = (lane & 15) - 7 of
  // the band and its weight cap - Pair(d)
  constexpr int kNoBand = no_band<DP>();
  const int boff = (lane & 15) - 7;
  const float bwt = a.wt[lane & 15];
  // lanes 15/31 sit out (a loop-invariant predicate): with them each half-warp
  // would span 16 banks and the two halves would collide whenever their f differ
  const bool blive = (lane & 15) < 15;
  const uint32_t wt_s = PAIR2D ? (uint32_t)__cvta_generic_to_shared(WT) + (lane & 15) * 4u : 0u;
  // dead lanes (lane 15/31, zero weight) get an offset that puts every f out of range
  // ---- helpers --------------------------------------------------------------
  // dense W-row step: rr += E'[.][d_src] for f = 4*lane.. (+128 r); store to slot
  // (PAIR2D: the row E'[d_src][.] of the 2-D table, from global memory / L2)
  auto ring_step = [&](float (&rr)[4 * NR], int row_src, int slot) {
    uint32_t e = PAIR2D ? cs.eo[row_src] >> 16 : cs.eo[row_src] & 0xffffu;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      float4 x = PAIR2D ? __ldg(reinterpret_cast<const float4*>(a.E2g + e * DP) + lane + 32 * r)
                        : *reinterpret_cast<const float4*>(Eb + e + 16 * lane + 512 * r);
      fadd2_inplace(rr[4 * r + 0], rr[4 * r + 1], x.x, x.y);
      fadd2_inplace(rr[4 * r + 2], rr[4 * r + 3], x.z, x.w);
      *reinterpret_cast<float4*>(ringw + slot * DP + 4 * lane + 128 * r) =
          make_float4(rr[4 * r + 0], rr[4 * r + 1], rr[4 * r + 2], rr[4 * r + 3]);
    }
  };
  auto load_seed = [&](float (&rr)[4 * NR], const float* row) {
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) rr[4 * r + c] = row[4 * lane + 128 * r + c];
  };
  // Bottoms j0 .. j0+nsteps-1 (j0 = 1 mod 4, nsteps = 0 mod 4) for this warp's 32
  // targets; rr holds the W-row W[.][j0-1].  Lanes hold target PAIRS: lane l owns
  // targets t0 = l & 15 and t1 = t0 + 16 of the block, and half-warp hw = l >> 4
  // takes bottom jA + hw of each bottom pair (jA, jA+1).  So a lane loads one row
  // record (and its gravity thresholds) per pair and uses it for two cells: the
  // per-row work, which costs a warp instruction per 32 cells when lanes own one
  // target each, is halved per cell.  The two halves' running minima of a target
  // (odd / even bottoms) are merged at the end of the step (merge_part).
  // Candidates are shifted by -cap*(k+1):  (P_k - W_j)[f] + min(aO', aG').
  // Software-pipelined: the next pair's record and object means are computed
  // before the current pair's table loads.  Shared memory is addressed with
  // explicit 32-bit offsets.
  struct Tg { uint32_t pp0, pp1, T0, T1, N0, N1; };   // priv rows, T[k+1], N4[k+1] of t0 / t1
  // Cost type of the rectangle: IW keeps priv rows, W-rows, records and the running
  // minima in int32 quanta (exact mode), so a cell is p - w + min(aO, aG) in one
  // IADD3 and no conversion; otherwise fp32.
  using CT = std::conditional_t<IW, int, float>;

  constexpr int kRectUnroll = IW ? 2 : 1;
  struct Acc { CT b0, b1; int a0, a1; };              // running minima {cost, argj} of t0 / t1
  const int hw = lane >> 4;
  const uint32_t rec_s = (uint32_t)__cvta_generic_to_shared(cs.rec);
  const uint32_t m2_s = (uint32_t)__cvta_generic_to_shared(M2s);   // (dynamic smem does not start at 0)
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ringw) + ring_b0<DP, SPARSE>();
  // band rounds: round 1 lanes 0-14 -> buffer 1, lanes 16-30 -> buffer 0; round 2
  // the other way round (each half applies a pixel of its own row records)
  const uint32_t bbuf1_s = ring_s + ((lane < 16) ? ring_b1<DP, SPARSE>() : 0u) + (uint32_t)((boff - 1) * 4);
  const uint32_t bbuf2_s = ring_s + ((lane < 16) ? 0u : ring_b1<DP, SPARSE>()) + (uint32_t)((boff - 1) * 4);
  // the W-row this half reads: buffer 1 holds W_jA (half 0), buffer 0 W_{jA+1} (half 1)
  const uint32_t wbuf_s = ring_s + ((lane < 16) ? ring_b1<DP, SPARSE>() : 0u);
  // IW atomic round: 8-lane group g = lane >> 3 applies one pixel at offset
  // (lane & 7) - 3: g0 pixel jA -> buffer 1, g1 pixel jA+2 -> buffer 0 (half 0's
  // rows), g2 pixel jA+1 -> buffer 1, g3 pixel jA+1 -> buffer 0 (half 1's row).
  // Lane 7 of a group (offset +4) adds 0 (band <= 3) inside the guard entries, so
  // the round needs no predicate.
  const int igrp = lane >> 3;
  const uint32_t ibase_s = ring_s + ((igrp & 1) ? 0u : ring_b1<DP, SPARSE>()) + (uint32_t)(((lane & 7) - 4) * 4);
  const int iwt = (int)a.wt[(lane & 7) + 4] * kIWS;   // cap - Pair at offset (lane & 7) - 3
  auto rect_run = [&](float (&rr)[4 * NR], int j0, int nsteps, const Tg& tg, Acc& acc) {
    // sparse band round: f = drp - 1 + boff always lands in the buffer or its
    // guards (no range test; zero-weight lanes write back their value)
    auto band = [&](uint32_t base, int drp) {
      float* q = shp<float>(base + 4u * (uint32_t)drp);
      if constexpr (PAIR2D) {
        const float wgt = *shp<const float>(wt_s + 64u * (uint32_t)drp);
        if (blive) *q -= wgt;
      } else {
        if (blive) *q -= bwt;
      }
    };
    auto rowj = [&](int j) {
      const uint4* q = shp<const uint4>(rec_s + 32u * (uint32_t)j);
      return unpack_row(q[0], q[1]);
    };
    // the candidate's prior: the row's step function of f (3 compares, 3 selects)
    auto cell = [&](const RowU& r, int j, int f, CT p, CT w, CT& best, int& argj) {
      const float pr = (f >= r.b2) ? ((f >= r.b3) ? r.V3 : r.V2) : ((f >= r.b1) ? r.V1 : r.V0);
      if constexpr (IW) {              // records hold scaled int32 quanta (bits in the float fields)
        best = min(best, p - w + __float_as_int(pr));   // (cost x 32) | bottom offset: run minimum
        (void)argj; (void)j;
      } else {
        float cand = (p - w) + pr;
        if (cand < best) { best = cand; argj = j; }
      }
    };
    auto fmean = [&](const RowU& r, uint32_t Tk, uint32_t N4k) {
      const uint32_t n4 = N4k - r.N4;
      const uint32_t M = *shp<const uint32_t>(m2_s + n4);
      return (int)__umulhi((Tk - r.T) >> (kRBits - 1), M);   // < D: object disparities below D - 1/2 (L#27)
    };
    auto band_i = [&](int drp) {
      atomicAdd(shp<int>(ibase_s + 4u * (uint32_t)drp), -iwt);
    };
    // IW: the run's packed minima of t0 / t1 (decoded into acc at the end)
    int m0 = 0x7fffffff, m1 = 0x7fffffff;
    RowU r = rowj(j0 + hw);
    if constexpr (SPARSE && IW) {
      // both buffers := W_{j0-1} (int32); then buffer 1 = W_{j0}, buffer 0 = W_{j0+1}
      const int drm = rowj(j0 - 1).drp;
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const int4 v = make_int4(__float_as_int(rr[4 * q]), __float_as_int(rr[4 * q + 1]),   // int32 bits
                                 __float_as_int(rr[4 * q + 2]), __float_as_int(rr[4 * q + 3]));
        *shp<int4>(ring_s + 16u * lane + 512u * q) = v;
        *shp<int4>(ring_s + ring_b1<DP, SPARSE>() + 16u * lane + 512u * q) = v;
      }
      __syncwarp();
      band_i(igrp == 1 ? r.drp : (igrp == 2 ? kNoBand : drm));   // g0, g3: pixel j0-1; g1: j0
    } else if constexpr (SPARSE) {
      // both buffers := W_{j0-1}; then buffer 1 = W_{j0}, buffer 0 = W_{j0+1}
      const int drm = rowj(j0 - 1).drp;
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const float4 v = make_float4(rr[4 * q], rr[4 * q + 1], rr[4 * q + 2], rr[4 * q + 3]);
        *shp<float4>(ring_s + 16u * lane + 512u * q) = v;
        *shp<float4>(ring_s + ring_b1<DP, SPARSE>() + 16u * lane + 512u * q) = v;
      }
      __syncwarp();
      band(bbuf1_s, drm);                       // both buffers += pixel j0-1
      __syncwarp();
      band(bbuf2_s, hw ? kNoBand : r.drp);      // buffer 0 += pixel j0 (half 0's row)
    } else {
      ring_step(rr, j0 - 1, 1);
      ring_step(rr, j0, 2);
    }
    int f0 = fmean(r, tg.T0, tg.N0), f1 = fmean(r, tg.T1, tg.N1);
    __syncwarp();
    // bottoms per iteration (A/B on the B200): fp32 path 4 (unroll 2: -3.5%, 8: -13%);
    // IW int32 path 8 (with the chunk bound, where the kernel's size decides its
    // instruction-cache misses: 16 bottoms -1.4% at 1024x440 and -3.4% at 1024x220,
    // 4 bottoms -1.8%; before the bound 16 had been best at DP = 128)
#pragma unroll kRectUnroll
    for (int jj = 0; jj < nsteps; jj += 4) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int jA = j0 + jj + 2 * half;          // odd
        const int jm = jA + hw;                     // this half's bottom
        // next pair (row jm+2).  After the run's last row jl <= k these are at most
        // rows k+2, k+3 (<= h+2): their mean lookup reads M2 at n4 >= -8 (inside the
        // pad before M2) and is never used.
        const RowU n = rowj(jm + 2);
        const int g0 = fmean(n, tg.T0, tg.N0), g1 = fmean(n, tg.T1, tg.N1);
        const uint32_t wb = SPARSE ? wbuf_s : ring_s + (hw ? ((2 + 2 * half) & 3) : ((1 + 2 * half) & 3)) * DP * 4u;
        const CT p0 = *shp<const CT>(tg.pp0 + 4u * f0), p1 = *shp<const CT>(tg.pp1 + 4u * f1);
        const CT w0 = *shp<const CT>(wb + 4u * f0), w1 = *shp<const CT>(wb + 4u * f1);
        if constexpr (IW) {
          cell(r, jm, f0, p0, w0, m0, acc.a0);
          cell(r, jm, f1, p1, w1, m1, acc.a1);
        } else {
          cell(r, jm, f0, p0, w0, acc.b0, acc.a0);
          cell(r, jm, f1, p1, w1, acc.b1, acc.a1);
        }
        if constexpr (SPARSE && IW) {
          __syncwarp();
          band_i(igrp == 1 ? n.drp : r.drp);       // W_jA -> W_{jA+2}, W_{jA+1} -> W_{jA+3}
        } else if constexpr (SPARSE) {
          // buffer 1: W_jA -> W_{jA+2} (pixels jA: half 0, jA+1: half 1);
          // buffer 0: W_{jA+1} -> W_{jA+3} (pixels jA+1: half 1, jA+2: half 0's next row)
          __syncwarp();
          band(bbuf1_s, r.drp);
          __syncwarp();
          band(bbuf2_s, hw ? r.drp : n.drp);
        } else {
          ring_step(rr, jA + 1, (3 + 2 * half) & 3);
          ring_step(rr, jA + 2, (4 + 2 * half) & 3);
        }
        r = n; f0 = g0; f1 = g1;
        __syncwarp();
      }
    }
    if constexpr (IW) {
      // a run lies inside one 32-row block: bottom = block base + low bits; bulk
      // chunks come nearest first (decreasing j), so an equal cost takes the lower
      // bottom (L#17)
      const int jb = ((j0 - 1) & ~31) + 1;
      auto fold = [&](int m, CT& best, int& argj) {
        const int c = m >> 5;            // arithmetic: floor((cost x 32 + off) / 32) = cost
        const int jm = jb + (m & 31);
        if (m != 0x7fffffff && (c < best || (c == best && jm < argj))) { best = c; argj = jm; }
      };
      fold(m0, acc.b0, acc.a0);
      fold(m1, acc.b1, acc.a1);
    }
  };
  // The step's result of target lane (t = lane): the two halves' minima merged,
  // ties to the lower bottom (the first in bottom order, L#17).
  auto merge_part = [&](const Acc& acc) {
    const CT sb = __shfl_xor_sync(0xffffffffu, hw ? acc.b0 : acc.b1, 16);
    const int sa = __shfl_xor_sync(0xffffffffu, hw ? acc.a0 : acc.a1, 16);
    CT mb = hw ? acc.b1 : acc.b0;
    int ma = hw ? acc.a1 : acc.a0;
    if (sb < mb || (sb == mb && sa < ma)) { mb = sb; ma = sa; }
    float mf;
    if constexpr (IW) mf = (mb >= (1 << 24)) ? INF : (float)mb;   // exact: finite |mb| < 2^24
    else mf = mb;
    return make_float2(mf, __int_as_float(ma));
  };

  // Full 32-row chunks m < mend for this warp's targets, handed out dynamically
  // (with the chunk bound on: nearest first, m = mend - 1 down to 0, so that the
  // far chunks meet a tight best candidate, and the run fold takes the lower
  // bottom on equal costs; otherwise increasing m, which the fp32 paths' strict-less
  // running minima need for L#17's first-bottom ties); the anchor row of the next
  // chunk is prefetched from L2 while one runs.
  // IW chunk bound (branch and bound, exact): every candidate of chunk m for a
  // target k of block B = mend + 1 satisfies
  //   cand(j, k) >= G[m] + wtmax (|S| - maxcount(S)) - wtmax (k + 1)
  // (shifted, unscaled), S = rows [32(m+1), 32B) inside every span [j, k]: each
  // pixel costs at least Pair(0) = cap - wtmax, and every pixel of S outside the
  // band of the span's mean costs cap (Eq. 4 saturates); maxcount(S) <=
  // max_c (P2[B][c] - P2[m+1][c]) bounds the pixels any one mean's band can hold.
  // The chunk is skipped when that bound exceeds, for every target, the best
  // candidate found so far by any warp (ub, strictly: a skipped candidate can be
  // neither the minimum nor tied with it, so costs and argmins are unchanged).
  auto bulk_chunks = [&](int mend, const Tg& tg, Acc& acc, int Kn) {
    int m = 0;
    if (lane == 0) m = atomicAdd(cs.ctr, 1);
    m = __shfl_sync(0xffffffffu, m, 0);
    auto chunk_of = [&](int q) { return bound ? mend - 1 - q : q; };
    float rr[4 * NR];
    if (m < mend) load_seed(rr, ANg + chunk_of(m) * DP);
    // bound inputs of block B = mend + 1 (this lane: bin c = lane)
    const int p2B = (bound && lane < NBIN) ? p2_at(mend + 1, lane) : 0;
    const int kl = min(Kn + lane, h - 1);
    while (m < mend) {
      const int mc = chunk_of(m);      // this chunk
      int m2 = 0;
      if (lane == 0) m2 = atomicAdd(cs.ctr, 1);
      m2 = __shfl_sync(0xffffffffu, m2, 0);
      float nx[4 * NR];
#pragma unroll
      for (int i = 0; i < 4 * NR; ++i) nx[i] = 0.f;
      if (m2 < mend) load_seed(nx, ANg + chunk_of(m2) * DP);
      bool skip = false;
      if (bound) {
        const int X = __reduce_max_sync(0xffffffffu, cs.ub[lane] + wtmax * (kl + 1));
        if (X < kUBInf) {                // (warp-uniform) some candidate of every target is known
          const int p2n = lane < NBIN ? p2_at(mc + 1, lane) : 0;
          const int maxcount = __reduce_max_sync(0xffffffffu, p2B - p2n);
          skip = cs.gmin[mc] + wtmax * (32 * (mend - mc) - maxcount) > X;
        }
      }
      if (!skip) {
        rect_run(rr, 32 * mc + 1, 32, tg, acc);
        if constexpr (IW) {
          if (bound) {
            // publish this warp's per-target minima (both halves merged): lane l -> target l
            const int o0 = __shfl_xor_sync(0xffffffffu, acc.b0, 16), o1 = __shfl_xor_sync(0xffffffffu, acc.b1, 16);
            atomicMin(cs.ub + lane, hw ? min(acc.b1, o1) : min(acc.b0, o0));
          }
        }
      } else {
        skipped += 32ull * (unsigned)min(32, h - Kn);
      }
#pragma unroll
      for (int i = 0; i < 4 * NR; ++i) rr[i] = nx[i];
      m = m2;
    }
  };

  constexpr int NB = NS / 2;           // f slices per builder warp (warps 1 and 2)
  CT fr[NB];                           // builder warps: W[f][32 bt] for f = lane + 32 (c0 + c)

  // ---------------- backtracking + extraction (a7), warp 0 ------------
  // The list is staged in the W-row ring and the triangle cells (contiguous,
  // >= 2h words), which the next item's prologue A and B leave alone.
  auto backtrack = [&](int item, float lastO, float lastG, float lastS) {
    {
      int c = 0;
      float cost = lastG;
      if (lastO < cost) { c = 1; cost = lastO; }
      if (lastS < cost) { c = 2; cost = lastS; }
      uint2* lst = reinterpret_cast<uint2*>(cs.ring);
      int n = 0;
      if (lane == 0) {
        // the walk reads only the index tables (shared memory); the stixels'
        // disparities are looked up in the parallel write below
        int kb = h - 1;
        while (true) {
          int j, cp;
          if (c == 1) {
            uint16_t x = cs.argO[kb]; j = x & 0xfff; cp = x >> 12;
          } else if (c == 0) {
            j = cs.argG[kb]; cp = j ? 1 : kStart;
          } else {
            uint16_t x = cs.argS[kb]; j = x & 0xfff; cp = x >> 12;
          }
          lst[n] = make_uint2((uint32_t)j | ((uint32_t)kb << 16), (uint32_t)c);
          ++n;
          if (j == 0 || n >= h) break;
          kb = j - 1;
          c = cp;
        }
      }
      n = __shfl_sync(0xffffffffu, n, 0);
      __syncwarp();
      stixel_t* o = a.out + (int64_t)item * a.cap;
      const int nw = min(n, a.cap);
#pragma unroll 1
      for (int i = lane; i < nw; i += 32) {
        uint2 e = lst[n - 1 - i];
        stixel_t s;
        s.bottom = (uint16_t)(e.x & 0xffff);
        s.top = (uint16_t)(e.x >> 16);
        s.cls = (uint8_t)e.y;
        s.pad[0] = s.pad[1] = s.pad[2] = 0;
        // L#19: object -> its mean f, ground -> the ground model at its bottom, sky -> 0
        s.disparity = e.y == 1 ? (float)cs.fpv[s.top]
                    : e.y == 0 ? (float)__ldg(a.dgR + s.bottom) * (1.0f / (1 << kRBits)) : 0.f;
        o[i] = s;
      }
      if (lane == 0) {
        a.count[item] = n;
        if (a.col_cost) a.col_cost[item] = cost * a.cost_scale;
        if (n > a.cap) atomicExch(a.overflow, 1);
      }
      __syncwarp();
    }
  };
  int pend_item = -1;
  float pendO = INF, pendG = INF, pendS = INF;
  for (int item = slot_global; item < a.items; item += gridDim.x * a.cols_per_cta) {
    const uint16_t* col = a.cols + (int64_t)item * h;
    // (diagnostic timeline: the group's third column, past the cold start)
    const bool trace_item = item == slot_global + 2 * gridDim.x * a.cols_per_cta;
    (void)trace_item;
    if (w == 0) STX_STAMP(60, 0);       // item start
    if (w == 0 && pend_item >= 0) {
      backtrack(pend_item, pendO, pendG, pendS);
      pend_item = -1;
    }
    const int ctidA = ctid - 32;         // prologue A: warps 1 .. CW-1
    // ---------------- prologue A (all 4 warps): per-pixel costs (a3-a4) ----------
    float* tG = cs.priv;                 // temporaries in the (idle) priv rows
    float* tS = cs.priv + h;
    uint32_t* tD = reinterpret_cast<uint32_t*>(cs.priv + 2 * h);
    // one row v of prologue A from its reduced value dR (-1 invalid)
    auto prologue_row = [&](int v, int dR, float xg, float xs) {
      const bool valid = dR >= 0;
      // the object model's view of the pixel (L#27): clamped below D - 1/2, so its
      // rounding (the pair-LUT index, L#9) and every span mean lie in [0, D);
      // ground and sky use dR itself (Eq. 4)
      const int dO = min(dR, ((a.D - 1) << kRBits) + (1 << (kRBits - 1)) - 1);
      const int dr = valid ? (dO + (1 << (kRBits - 1))) >> kRBits : -1;   // round half up (L#9)
      if (v < h) {                       // (xg, xs: the row's ground / sky cost, Eq. 4)
        tG[v] = xg; tS[v] = xs;
        tD[v] = valid ? (uint32_t)dO + (1u << (kRBits - 1)) : 0u;
      }
      if (v <= h)                        // static record word of row v: pixel code (ordthr later)
        cs.rec[2 * v + 1].w = (uint32_t)(valid ? dr + 1 : kNoBand) << 16;
      if (v < 2) {                       // padding rows h+1, h+2 and row 0: T = N4 = 0
        cs.rec[2 * (h + 1 + v) + 1] = make_uint4(0, 0, 0, (uint32_t)kNoBand << 16);
        cs.rec[2 * (h + 1 + v)] = make_uint4(0, 0, 0, 0);
        if (v == 0) { cs.rec[1].x = 0; cs.rec[1].y = 0; }
      }
      // E offsets of this row
      int dmr = valid ? a.D - dr : a.dmr_inv;
      int cc = dmr & 3;
      // hi16: E' row of the build -- the byte offset of its window in E copy 0, or
      // (PAIR2D) the row index d of the 2-D table (D + 1 = invalid)
      const uint32_t ehi = PAIR2D ? (uint32_t)(valid ? dr : a.D + 1) : (uint32_t)(dmr * 4);
      cs.eo[v] = (uint32_t)(cc * a.esz * 4 + (dmr - cc) * 4) | (ehi << 16);
    };
    // 4 rows per thread per pass, their loads issued together: the column values
    // and ground-model entries first, then the cost-table entries they index (two
    // memory round trips per pass instead of two per row)
    for (int v0 = ctidA; w > 0 && v0 < h + 2; v0 += 4 * (CW - 1) * 32) {
      int dR[4], dg[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int v = v0 + k * (CW - 1) * 32;
        const uint32_t u = v < h ? __ldg(col + v) : 0xffffu;
        // valid below D (L#23: a caller-made column value >= D * 256 is invalid)
        dR[k] = (u == 0xffffu || u >= ((uint32_t)a.D << kRBits)) ? -1 : (int)u;
        dg[k] = v < h ? __ldg(a.dgR + v) : 0;
      }
      float xg[4], xs[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int v = v0 + k * (CW - 1) * 32;
        xg[k] = capQ; xs[k] = capQ;
        if (dR[k] >= 0) {
          const float* gGv = PAIR2D ? a.gG + v * a.gG_stride : a.gG;   // f2: per-row tables
          xg[k] = __ldg(gGv + min(abs(dR[k] - dg[k]), a.LG - 1));
          xs[k] = __ldg(a.gS + min(dR[k], a.LS - 1));
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int v = v0 + k * (CW - 1) * 32;
        if (v < h + 2) prologue_row(v, dR[k], xg[k], xs[k]);
      }
    }

    for (int i = ctidA; w > 0 && i < DP; i += (CW - 1) * 32) ANg[i] = 0.f;   // W[.][0] = 0
    if (ctidA == 0) *cs.ctr = 0;
    named_bar(bar_col, CW * 32);
    STX_STAMP(63, w);                    // clock calibration (all warps just released)

    if (w == 0) STX_STAMP(60, 3);       // prologue A done
    // ---------------- prologue B (4 warps): prefix sums --------------
    // warp 0: ground PG, warp 1: sky PS, warp 2: disparity T, warp 3: count N4.
    // Two-level: lane l sums its segment of ceil(h/32) consecutive rows, one warp
    // scan of the 32 segment totals, then each lane writes its segment's prefixes
    // (exact integer quanta in exact mode, so the order of the adds is immaterial).
    if (w < 4) {                        // warps 4.. (CW = 8) idle
      const int seg = (h + 31) >> 5;
      const int s0 = min(lane * seg, h), s1 = min(s0 + seg, h);
      if (w < 2) {
        const float* src = (w == 0) ? tG : tS;
        float* dst = (w == 0) ? PGg : PSg;
        float tot = 0.f;
#pragma unroll 1
        for (int v = s0; v < s1; ++v) tot += src[v];
        float acc = warp_incl_scan(tot, lane) - tot;   // exclusive prefix of the totals
        if (lane == 0) dst[0] = 0.f;
#pragma unroll 1
        for (int v = s0; v < s1; ++v) { acc += src[v]; dst[v + 1] = acc; }
      } else {
        uint32_t tot = 0;
#pragma unroll 1
        for (int v = s0; v < s1; ++v) { const uint32_t t = tD[v]; tot += (w == 2) ? t : (t ? 4u : 0u); }
        uint32_t acc = warp_incl_scan(tot, lane) - tot;
#pragma unroll 1
        for (int v = s0; v < s1; ++v) {
          const uint32_t t = tD[v];
          acc += (w == 2) ? t : (t ? 4u : 0u);
          if (w == 2) cs.rec[2 * (v + 1) + 1].x = acc;   // T[v+1]
          else cs.rec[2 * (v + 1) + 1].y = acc;          // N4[v+1]
        }
      }
    }
    named_bar(bar_col, CW * 32);
    if (w == 0) STX_STAMP(60, 4);       // prologue B done

    // build priv W-rows of block bt and the anchor row 32(bt+1): a sequential
    // prefix over rows, per f, so the f slices are independent.  Two
    // warps (w = 1, 2) build them, each half of the slices: lane l owns
    // f = l + 32 (c0 + c), c < NB, so both the E' loads and the priv stores are
    // bank-conflict free.  The row offsets come from lane registers by shuffle;
    // loads of 8 rows are issued before their prefix chain.
    auto build_priv = [&](int bt) {
      const int c0 = (w - 1) * NB;
      const int K0b = bt << 5;
      const int rows = min(32, h - K0b);
      const uint32_t eor = cs.eo[K0b + min(lane, rows - 1)] >> 16;
      const uint32_t dst_s = (uint32_t)__cvta_generic_to_shared(cs.priv) + lane * 4;
      const uint32_t src_s = (uint32_t)__cvta_generic_to_shared(E) + lane * 4;
      // (not unrolled: four copies of this batch of 8 rows, whose shuffles the
      // compiler wraps in collective sequences, cost instruction-cache misses)
#pragma unroll 1
      for (int i0 = 0; i0 < 32; i0 += 8) {
        if (i0 < rows) {
          CT x[8][NB];
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const uint32_t e = __shfl_sync(0xffffffffu, eor, i0 + r);
#pragma unroll
            for (int c = 0; c < NB; ++c) {
              if constexpr (PAIR2D) x[r][c] = __ldg(a.E2g + e * DP + 32 * (c0 + c) + lane);
              else x[r][c] = *shp<const CT>(src_s + e + 128u * (c0 + c));
            }
          }
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            if (i0 + r < rows) {
#pragma unroll
              for (int c = 0; c < NB; c += 2) {
                if constexpr (IW) {
                  fr[c] += x[r][c];
                  fr[c + 1] += x[r][c + 1];
                } else {
                  fadd2_inplace(fr[c], fr[c + 1], x[r][c], x[r][c + 1]);
                }
                *shp<CT>(dst_s + ((i0 + r) * priv_stride<DP>() + 32 * (c0 + c)) * 4u) = fr[c];
                *shp<CT>(dst_s + ((i0 + r) * priv_stride<DP>() + 32 * (c0 + c) + 32) * 4u) = fr[c + 1];
              }
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NB; ++c) reinterpret_cast<CT*>(ANg)[(bt + 1) * DP + 32 * (c0 + c) + lane] = fr[c];
    };
    // triangle cells of block bt: bottom K0+1+j', target K0+k' (k' > j'); their
    // bottoms' W-rows are the block's own priv rows: data term (absolute),
    // f, gravity level.  The 496 cells are spread densely over the column group.
    // Also keeps the W-rows K0+8, K0+16, K0+24 as seeds of block bt+1's newest chunk.
    auto precompute_cells = [&](int bt, int t0, int nthr) {
      const int K0b = bt << 5;
      const int jn = min(K0b + 31, h - 1) - K0b;
      const int ncell = tri_off(jn);
      // {T, N4} of the block's rows K0b+1+l in lane l: the cells' row reads become
      // shuffles (the records' 32-byte stride would make them 8-way bank conflicts)
      const uint2 tnl = tn_at(min(K0b + lane + 1, h));
      if constexpr (IW) {
        // IW: int32 cells for the packed serial chain.  Warp iteration `it` takes
        // bottom rows j' = it (targets k' = it+1+l, lanes l < 31-it) and j' = 30-it
        // (targets k' = l, the other it+1 lanes): 32 cells, two distinct rows.
        // Cell = {data x 32 | code, min(data + gravity prior, BIG) x 32 | code, f,
        // f - ord_margin}, code = j' + 1 (the bottom's place in the block, L#17).
        const int* pv = reinterpret_cast<const int*>(cs.priv);
        int4* cl = reinterpret_cast<int4*>(cells_of(bt));
        const int wq = t0 >> 5, nq = nthr >> 5;       // this warp's index among nq warps
        // (not unrolled: the smaller kernel has fewer instruction-cache misses, +1.5%)
#pragma unroll 1
        for (int it = wq; it < 16; it += nq) {
          const bool lo = lane < 31 - it;
          const int jr = lo ? it : 30 - it;
          const int kp = lo ? it + 1 + lane : lane;
          const uint32_t ryx = __shfl_sync(0xffffffffu, tnl.x, jr), ryy = __shfl_sync(0xffffffffu, tnl.y, jr);
          const uint32_t rkx = __shfl_sync(0xffffffffu, tnl.x, kp), rky = __shfl_sync(0xffffffffu, tnl.y, kp);
          if (kp <= jn) {
            const int f = span_f(rkx - ryx, rky - ryy, smem, Dm1);
            const int d = pv[kp * priv_stride<DP>() + f] - pv[jr * priv_stride<DP>() + f] + capI * (kp - jr);
            const int2 th = thrS[K0b + jr + 1];
            const int pen = (f >= th.x) ? goHiI : ((f < th.y) ? goLoI : goMidI);
            const int code = jr + 1;
            cl[tri_off(jr) + kp - jr - 1] = make_int4(d + code, min(d + pen, kChainBig) + code, f, f - a.ord_margin);
          }
        }
      } else {
      for (int base = t0 - lane; base < ncell; base += nthr) {   // warp-uniform trip count
        const int idx = base + lane;
        const uint32_t jk = tri_jk[min(idx, kTri - 1)];
        const int jp = jk & 0xff, kp = jk >> 8;
        const int k = K0b + kp;
        const uint32_t ryx = __shfl_sync(0xffffffffu, tnl.x, jp), ryy = __shfl_sync(0xffffffffu, tnl.y, jp);
        const uint32_t rkx = __shfl_sync(0xffffffffu, tnl.x, kp), rky = __shfl_sync(0xffffffffu, tnl.y, kp);
        if (idx < ncell && k < h) {
          int f = span_f(rkx - ryx, rky - ryy, smem, Dm1);
          const CT* pv = reinterpret_cast<const CT*>(cs.priv);
          float data = (float)((pv[kp * priv_stride<DP>() + f] - pv[jp * priv_stride<DP>() + f]) / (IW ? kIWS : 1)) + capQ * (float)(kp - jp);
          const int jr = K0b + jp + 1;
          const int2 th = thrS[jr];
          const float pen = (f >= th.x) ? a.kGO_hi : ((f < th.y) ? a.kGO_lo : a.kGO_mid);
          cells_of(bt)[idx] = make_float4(data, data + pen, __int_as_float(f), 0.f);
        }
      }
      }
    };
    // seeds of block bt's newest chunk beyond its first part: W-rows K0 + 32 i / NWN
    // (priv rows 32 i / NWN - 1), i = 1 .. NWN - 1
    constexpr int NWN = newest_warps(CW);
    auto copy_seed = [&](int bt) {
      if ((bt << 5) + 32 < h) {          // only needed if a next block exists
#pragma unroll
        for (int i = 1; i < NWN; ++i) {
          float* sd = cs.seed + ((bt & 1) * (NWN - 1) + i - 1) * DP;
          const float* row = cs.priv + (32 / NWN * i - 1) * priv_stride<DP>();
#pragma unroll 1
          for (int f = lane; f < DP; f += 32) sd[f] = row[f];
        }
      }
    };

    if (w == 1 || w == 2) {
#pragma unroll
      for (int c = 0; c < NB; ++c) fr[c] = 0;
      build_priv(0);
    } else if (bound && w == 3) {
      // chunk-bound tables while warps 1-2 build: P2 at every block boundary (bins
      // of 8 of the pixels' object disparities).  Per block, the lanes (rows) that
      // share a bin find each other with one match; the group's first lane writes
      // the count into a per-bin scratch row (cs.part, free until block 0's merge)
      int* hb = reinterpret_cast<int*>(cs.part);
      int pc = 0;                        // lane c: valid pixels of bin c in rows < 32 bb
#pragma unroll 1
      for (int bb = 0; bb < nb; ++bb) {
        const int v = (bb << 5) + lane;
        const uint32_t code = v < h ? cs.rec[2 * v + 1].w >> 16 : (uint32_t)kNoBand;
        const int bin = code != (uint32_t)kNoBand ? (int)(code - 1) >> 3 : 255;   // round(d) >> 3
        hb[lane] = 0;
        __syncwarp();
        const uint32_t same = __match_any_sync(0xffffffffu, bin);
        if (bin < NBIN && (same & ((1u << lane) - 1)) == 0) hb[bin] = __popc(same);
        __syncwarp();
        pc += hb[lane];
        __syncwarp();
        const int up = __shfl_down_sync(0xffffffffu, pc, 1);
        if (lane < NBIN) P2s[2 * (bb * NBIN + lane)] = (uint16_t)(pc + (lane + 1 < NBIN ? up : 0));
      }
    }
    if (bound && ctid < 32) cs.ub[ctid] = kUBInf;
    named_bar(bar_col, CW * 32);
    if (w == 0) STX_STAMP(60, 5);       // block 0's priv rows built

    // block 0 has only the j = 0 candidate (Eq. 5) and its triangle
    {
      const int kk = lane < h ? lane : h - 1;
      const uint2 rky = tn_at(kk + 1);
      const uint32_t Tk = rky.x, N4k = rky.y;
      const float* pp = cs.priv + kk * priv_stride<DP>();   // lanes past h: the last row's copy
      float rbest = INF;
      int rargj = 0x7fffffff;
      if (w == 1) {
        int f = span_f(Tk, N4k, smem, Dm1);
        rbest = (float)(reinterpret_cast<const CT*>(pp)[f] / (IW ? kIWS : 1)) + a.piFirstO;   // shifted by -cap*(k+1)
        rargj = 0;
      }
      cs.part[w * 32 + lane] = make_float2(rbest, __int_as_float(rargj));
      precompute_cells(0, ctid, CW * 32);
      if (w == 2) copy_seed(0);
    }
    named_bar(bar_col, CW * 32);

    // serial-warp state carried across blocks (warp-uniform): last row's C values,
    // ground / sky running minima (value, argmin) of Eq. 6's G and S rows
    float cCO = INF, cCG = INF;          // C_O[K0-1], C_G[K0-1]
    float MG = a.piFirstG, MS = INF;     // min over bottoms j of (C[j-1] + t - P[j]), j=0 first
    int gj = 0, sj = 0;                  // argmin (j | c' << 12 for sky)
    float lastO = INF, lastG = INF, lastS = INF;

    for (int b = 0; b < nb; ++b) {
      const int K0 = b << 5;
      const int k = K0 + lane;
      const int bn = b + 1;
      const int Kn = bn << 5;
      const bool has_next = bn < nb;
      if (w == 0) STX_STAMP(b, 0);
      if (w == 0) {
        // ============ serial warp: block b's triangle and finalisation ============
        const int kk = k < h ? k : h - 1;
        const uint2 rky = tn_at(kk + 1);
        const uint32_t N4k = rky.y;
        const uint32_t Tk = rky.x;
        const float pg0 = PGg[kk], pg1 = PGg[kk + 1], ps0 = PSg[kk], ps1 = PSg[kk + 1];
        float best = INF;
        int argj = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < CW; ++q) {
          float2 p = cs.part[q * 32 + lane];
          int pj = __float_as_int(p.y);
          if (p.x < best || (p.x == best && pj < argj)) { best = p.x; argj = pj; }
        }
        best += capQ * (float)(k + 1);   // undo the rectangle's per-target shift
        // f and c' of the winner (the rectangle tracked only its j)
        int argf, argc;
        if (argj == 0 || argj >= h) {    // (argj >= h: a lane past h that found no candidate)
          argf = span_f(Tk, N4k, smem, Dm1);
          argc = kStart;
        } else {
          const RowU r = load_row(cs.rec, argj);
          argf = span_f(Tk - r.T, N4k - r.N4, smem, Dm1);
          const int iv = (argf >= r.b1) + (argf >= r.b2) + (argf >= r.b3);   // the step's interval
          argc = (r.cb >> iv) & 1;
        }
        const float kOG = a.kOG;
        const int om = a.ord_margin;
        const int jn = min(K0 + 31, h - 1) - K0;
        // Chain state: C_O, C_G and the object mean of the last finalised target.
        // Target K0: all its bottoms were in the rectangle.
        float mg = (K0 == 0) ? a.piFirstG : fminf(MG, cCO + (kOG - pg0));   // lane 0's value
        mg = __shfl_sync(0xffffffffu, mg, 0);
        int tri_c = 0;                   // IW: the winner's code (0: a bottom before the block)
        if constexpr (IW) {
          // Packed int32 chain (exact mode): costs x 32 with the bottom's code j' + 1
          // in the low 5 bits (0 for the rectangle's winner, whose bottom is lower),
          // so the first-minimum rule of L#17 is one integer min; argc is
          // recovered after the scans.
          int2* pq = reinterpret_cast<int2*>(cs.pgps);
          pq[lane] = make_int2(toI(kOG - pg0), toI(pg1));
          __syncwarp();
          const int oh = toI(a.kOO_hi), ol = toI(a.kOO_lo);
          const int4* cl = reinterpret_cast<const int4*>(cells_of(b));
          int mgI = toI(mg);
          int prevCG = toI(__shfl_sync(0xffffffffu, pg1, 0) + mg);
          int bI = toI(best);
          int afI = argf;
          int prevCO = __shfl_sync(0xffffffffu, bI, 0);
          int prevF = __shfl_sync(0xffffffffu, argf, 0);
          int off = 0;                                  // tri_off(jp)
          STX_STAMP(b, 21);
          for (int jp = 0; jp < jn; ++jp) {
            const int2 q = pq[jp + 1];
            // every lane's cell (bottom j, target K0 + lane); lane jp + 1's is the
            // diagonal, so after the update that lane holds C_O[j] and its f
            {
              const int4 lc = cl[off + lane - jp - 1];  // (lanes <= jp read a dead slot)
              const int cand = min(lc.x + prevCO + ((lc.w > prevF) ? oh : ol), lc.y + prevCG);
              const bool upd = (lane > jp) && (cand < bI);
              bI = upd ? cand : bI;
              afI = upd ? lc.z : afI;
            }
            const int COj = __shfl_sync(0xffffffffu, bI, jp + 1);
            const int Fj = __shfl_sync(0xffffffffu, afI, jp + 1);
            mgI = min(mgI, prevCO + q.x);               // ground chain (value only)
            prevCG = q.y + mgI;
            prevCO = min(COj & ~31, kChainBig);
            prevF = Fj;
            off += 31 - jp;
          }
          best = (bI >= kChainBig) ? INF : (float)(bI >> 5);
          tri_c = bI & 31;
          if (tri_c) { argj = K0 + tri_c; argf = afI; }
        } else {
        // per row j = K0 + lane: {kOG - PG[j], PG[j+1]} for the in-loop ground chain
        cs.pgps[lane] = make_float4(kOG - pg0, pg1, 0.f, 0.f);
        __syncwarp();
        const float oh = opaque(a.kOO_hi), ol = opaque(a.kOO_lo);
        float prevCG = __shfl_sync(0xffffffffu, pg1, 0) + mg;
        float prevCO = __shfl_sync(0xffffffffu, best, 0);
        int prevF = __shfl_sync(0xffffffffu, argf, 0);
        int off = 0;                                    // tri_off(jp)
        STX_STAMP(b, 21);                 // serial: merge + recovery + chain setup done
        for (int jp = 0; jp < jn; ++jp) {
          const int j = K0 + jp + 1;                    // bottom j; target j finalised
          const float4 q = cs.pgps[jp + 1];
          // this lane's cell (bottom j, target k > j) with the same predecessors;
          // lane jp + 1's is the diagonal (the 1-pixel stixel), so after the update
          // that lane holds C_O[j] and its f
          {
            const int idx = off + lane - jp - 1;        // (lanes <= jp read a dead slot)
            const float4 lc = cells_of(b)[idx];
            const float data = lc.x;
            const float dgl = lc.y;
            const int f = __float_as_int(lc.z);
            const float tO = data + (prevCO + ((f > prevF + om) ? oh : ol));
            const float tG = dgl + prevCG;
            const bool pg = tG <= tO;                   // == (aG <= aO): data added to both
            const float cand = pg ? tG : tO;
            const bool upd = (lane > jp) && (cand < best);
            best = upd ? cand : best;
            argj = upd ? j : argj;
            argf = upd ? f : argf;
            argc = upd ? (pg ? 0 : 1) : argc;
          }
          const float COj = __shfl_sync(0xffffffffu, best, jp + 1);
          const int Fj = __shfl_sync(0xffffffffu, argf, jp + 1);
          // ground: GR^j = PG[j+1] + min(.., C_O[j-1] + t - PG[j])  (value only)
          mg = fminf(mg, prevCO + q.x);
          prevCG = q.y + mg;
          prevCO = COj;
          prevF = Fj;
          off += 31 - jp;
        }
        }
        STX_STAMP(b, 22);                 // serial: triangle chain done
        // ---- ground / sky argmins and values of the block's rows, as warp scans ----
        // lane l = row j = K0 + l = target k: candidates at bottom j use C[j-1]
        const float up_best = __shfl_up_sync(0xffffffffu, best, 1);     // all lanes shuffle
        const float COm1 = (lane == 0) ? cCO : up_best;
        float vG = (K0 == 0 && lane == 0) ? a.piFirstG : COm1 + (kOG - pg0);
        int aG = (K0 == 0 && lane == 0) ? 0 : k;
        if (k >= h) { vG = INF; aG = 0x7fffffff; }
        // inclusive prefix min over lanes, ties -> lower lane (first j); carry first
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float v2 = __shfl_up_sync(0xffffffffu, vG, o);
          const int a2 = __shfl_up_sync(0xffffffffu, aG, o);
          if (lane >= o && !(vG < v2)) { vG = v2; aG = a2; }
        }
        if (K0 > 0 && !(vG < MG)) { vG = MG; aG = gj; }
        const float CGk = pg1 + vG;
        const float up_cg = __shfl_up_sync(0xffffffffu, CGk, 1);
        const float CGm1 = (lane == 0) ? cCG : up_cg;
        float v1 = CGm1 + a.kGS - ps0, v2 = COm1 + a.kOS - ps0;    // pred G, pred O
        float vS = (v2 < v1) ? v2 : v1;
        int aS = (v2 < v1) ? (k | (1 << 12)) : k;
        if ((K0 == 0 && lane == 0) || k >= h) { vS = INF; aS = (K0 == 0 && lane == 0) ? (kStart << 12) : 0x7fffffff; }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const float v3 = __shfl_up_sync(0xffffffffu, vS, o);
          const int a3 = __shfl_up_sync(0xffffffffu, aS, o);
          if (lane >= o && !(vS < v3)) { vS = v3; aS = a3; }
        }
        if (K0 > 0 && !(vS < MS)) { vS = MS; aS = sj; }
        const float CSk = ps1 + vS;
        if constexpr (IW) {
          // predecessor class of a triangle winner (bottom j = K0 + tri_c): G iff
          // its G candidate is <= its O candidate (L#17), re-evaluated from the
          // final C_O, C_G and f of row j - 1 (lane tri_c - 1)
          const int src = max(tri_c - 1, 0);
          const float pO = __shfl_sync(0xffffffffu, best, src);
          const float pG = __shfl_sync(0xffffffffu, CGk, src);
          const int pF = __shfl_sync(0xffffffffu, argf, src);
          if (tri_c) {
            const int4 lc = reinterpret_cast<const int4*>(cells_of(b))[tri_off(src) + lane - src - 1];
            const int tO = lc.x + min(toI(pO), kChainBig) + ((lc.w > pF) ? toI(a.kOO_hi) : toI(a.kOO_lo));
            const int tG = lc.y + toI(pG);
            argc = (tG <= tO) ? 0 : 1;
          }
        }
        // carry to the next block: last row of this block (lane 31, or h-1)
        const int L = min(31, h - 1 - K0);
        MG = __shfl_sync(0xffffffffu, vG, L); gj = __shfl_sync(0xffffffffu, aG, L);
        MS = __shfl_sync(0xffffffffu, vS, L); sj = __shfl_sync(0xffffffffu, aS, L);
        cCO = __shfl_sync(0xffffffffu, best, L);
        cCG = __shfl_sync(0xffffffffu, CGk, L);
        if (K0 + 31 >= h - 1) {
          lastO = cCO; lastG = cCG; lastS = __shfl_sync(0xffffffffu, CSk, L);
        }
        STX_STAMP(b, 23);                 // serial: scans + carries done
        // every lane now holds the final values of its target row k: write the
        // record of row k+1 (consumed by later rectangles; predecessor terms
        // shifted by -cap*(k+1)) and the index table
        int gv = 0x7fffffff;
        if (k < h) {
          const float sh = capQ * (float)(k + 1);
          // IW: int32 quanta x 32 with (j - 1) & 31 = k & 31 of row j = k + 1 in the low bits
          auto rb = [&](float x) {
            if constexpr (IW) return (uint32_t)((x >= 16777216.f ? kIWBig : __float2int_rn(x) * kIWS) + (k & 31));
            else return __float_as_uint(x);
          };
          // prior of a candidate with bottom j = k + 1 as a function of its object
          // mean f: O below (ordering: f > argf + om), G below (gravity: f >= thA,
          // diving: f < thB, L#1, L#15), the cheaper of the two (L#17: G on ties)
          const uint32_t AO0 = rb((best + a.kOO_lo) - sh), AO1 = rb((best + a.kOO_hi) - sh);
          const uint32_t AGm = rb((CGk + a.kGO_mid) - sh), AGh = rb((CGk + a.kGO_hi) - sh);
          const uint32_t AGl = rb((CGk + a.kGO_lo) - sh);
          const int2 th = thrS[k + 1];
          const int bO = min(argf + a.ord_margin + 1, 1023);          // f > argf + om
          const int b1 = min(bO, min(th.x, th.y)), b3 = max(bO, max(th.x, th.y));
          const int b2 = max(min(bO, th.x), min(max(bO, th.x), th.y));
          int cb = 0;
          auto step = [&](int f, int i) {
            const uint32_t aO = (f >= bO) ? AO1 : AO0;
            const uint32_t aG = (f >= th.x) ? AGh : ((f >= th.y) ? AGm : AGl);
            bool g;
            if constexpr (IW) g = (int)aG <= (int)aO;
            else g = __uint_as_float(aG) <= __uint_as_float(aO);
            cb |= (g ? 0 : 1) << i;
            return g ? aG : aO;
          };
          const uint32_t V0 = step(b1 - 1, 0), V1 = step(b1, 1), V2 = step(b2, 2), V3 = step(b3, 3);
          cs.rec[2 * (k + 1)] = make_uint4(V0, V1, V2, V3);
          uint32_t* ry = reinterpret_cast<uint32_t*>(cs.rec + 2 * (k + 1) + 1);
          ry[2] = (uint32_t)b1 | ((uint32_t)b2 << 16);
          reinterpret_cast<uint16_t*>(ry + 3)[0] = (uint16_t)(b3 | (cb << 10));   // (drp kept)
          cs.argO[k] = (uint16_t)(argj | (argc << 12));
          cs.argG[k] = (uint16_t)aG;
          cs.argS[k] = (uint16_t)aS;
          cs.fpv[k] = (uint8_t)argf;
          if constexpr (IW)                // chunk bound: min prior term of bottom j = k + 1, + wtmax j
            gv = (min(min((int)V0, (int)V1), min((int)V2, (int)V3)) >> 5) + wtmax * (k + 1);
        }
        if (bound) {
          const int g = __reduce_min_sync(0xffffffffu, gv);   // chunk b = bottoms 32b+1 .. 32b+32
          if (lane == 0) cs.gmin[b] = g;
        }
        STX_STAMP(b, 1);
        if (has_next) named_bar(bar_x, CW * 32);   // block b+1's priv rows are ready
      } else if (has_next) {
        if (w == 1 || w == 2) build_priv(bn);   // block b's priv rows are no longer needed
        if (w == 1) STX_STAMP(b, 2);
        named_bar(bar_rect, (CW - 1) * 32);
        asm volatile("bar.arrive %0, %1;" ::"r"(bar_x), "r"(CW * 32) : "memory");
      }
      // ======== all warps: block b+1, bottoms final before block b ===============
      Acc acc;
      if constexpr (IW) acc = Acc{0x7fffffff, 0x7fffffff, 0x7fffffff, 0x7fffffff};
      else acc = Acc{INF, INF, 0x7fffffff, 0x7fffffff};
      Tg tg{};
      if (has_next) {
        // this lane's target pair t0 = lane & 15, t1 = t0 + 16 of block b+1
        const int t0 = lane & 15, t1 = t0 + 16;
        // (targets past h duplicate the last row: only built priv rows are read)
        const int k0 = min(Kn + t0, h - 1), k1 = min(Kn + t1, h - 1);
        const uint2 r0 = tn_at(k0 + 1), r1 = tn_at(k1 + 1);
        const float* pp0 = cs.priv + (k0 - Kn) * priv_stride<DP>();
        const float* pp1 = cs.priv + (k1 - Kn) * priv_stride<DP>();
        tg = Tg{(uint32_t)__cvta_generic_to_shared(pp0), (uint32_t)__cvta_generic_to_shared(pp1),
                r0.x, r1.x, r0.y, r1.y};
        if (w == 1 && hw == 0) {       // j = 0: first stixel spans 0..k (Eq. 5)
          const CT pf = IW ? (CT)__float2int_rn(a.piFirstO) : (CT)a.piFirstO;
          acc.b0 = reinterpret_cast<const CT*>(pp0)[span_f(r0.x, r0.y, smem, Dm1)] / (IW ? kIWS : 1) + pf;
          acc.b1 = reinterpret_cast<const CT*>(pp1)[span_f(r1.x, r1.y, smem, Dm1)] / (IW ? kIWS : 1) + pf;
          acc.a0 = acc.a1 = 0;
        }
        if (CW == 8 && w >= NWN) {
          // latency plan: block b+1's triangle cells (into the other cell buffer)
          // and newest-chunk seeds now, so the newest phase is the 4 x 8-row run alone
          precompute_cells(bn, ctid - 32 * NWN, (CW - NWN) * 32);
          if (w == NWN) copy_seed(bn);
        }
        // full chunks m <= b-1: their records (rows <= 32 b) were final before block b
        bulk_chunks(b, tg, acc, Kn);
      }
      // warp 0's newest-chunk seed W[.][K0] from L2, prefetched before the barrier
      float rs0[4 * NR];
      if (w == 0 && has_next) load_seed(rs0, ANg + b * DP);
      STX_STAMP(b, 3 + w);
      named_bar(bar_col, CW * 32);
      if (w == 0) STX_STAMP(b, 11);
      if (has_next) {
        // newest chunk (bottoms K0+1 .. K0+32, final after block b's triangle):
        // warps 0 .. NWN-1 take 32/NWN rows each, seeded from W-rows K0 (anchor)
        // and K0 + 32 i / NWN (copied seeds), while the other warps precompute
        // block b+1's triangle cells
        if (w < NWN) {
          float rr[4 * NR];
          if (w == 0) {
#pragma unroll
            for (int i = 0; i < 4 * NR; ++i) rr[i] = rs0[i];
          } else {
            load_seed(rr, cs.seed + ((b & 1) * (NWN - 1) + w - 1) * DP);   // W-row K0 + 32 w / NWN
          }
          rect_run(rr, K0 + 1 + 32 / NWN * w, 32 / NWN, tg, acc);
        } else if (CW != 8) {
          precompute_cells(bn, ctid - 32 * NWN, (CW - NWN) * 32);
          if (w == NWN) copy_seed(bn);
        }
        cs.part[w * 32 + lane] = merge_part(acc);
        if (ctid == 0) *cs.ctr = 0;
        if (bound && ctid < 32) cs.ub[ctid] = kUBInf;   // (read again only after the next bar_col)
      }
      STX_STAMP(b, 12 + w);
      named_bar(bar_col, CW * 32);
      if (w == 0) STX_STAMP(b, 20);
    }

    if (w == 0) STX_STAMP(60, 1);       // blocks done
    // backtracking of this column: by warp 0 at the start of the next item, while
    // the other warps run that item's prologue A
    if (w == 0) { pend_item = item; pendO = lastO; pendG = lastG; pendS = lastS; }
  }
  if (w == 0 && pend_item >= 0) backtrack(pend_item, pendO, pendG, pendS);
  if (bound && a.skipped && lane == 0 && skipped) atomicAdd(a.skipped, skipped);
}

}  // namespace stx
