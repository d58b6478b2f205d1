// kernels.cuh -- sm_100a device code of the stixel hot path.
//
// K1 reduce_kernel : column reduction + transpose, HBM-bound.
// K3 dp_kernel     : per-column prefix sums and object-LUT rows (P:163-177,
//                    P:207-219), the Eq. 5-6 min-plus DP (P:129-157,
//                    P:221-235) and fused backtracking.
//
// Design: one WARP per column, lanes own targets k in
// blocks of 32 ("lanes own targets"), bottoms j iterate warp-uniformly.  The
// object LUT LUT_object[f][v] (D x (h+1) per column, 220 KiB at 1024x440,
// P:209 "too large to fit into Shared Memory") is never materialised: the 32
// rows LUT[.][k+1] of the current target block live in shared memory ("priv"),
// and the row LUT[.][j] of the current bottom is carried incrementally in a
// 4-deep shared ring (row_{j+1} = row_j + Pair[.][d_j]).  Costs are fp32; in
// exact mode (L#22) they are integer quanta < 2^24, so every add and min is
// exact and decisions match the double-precision oracle bit for bit.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/stixels.h"

namespace stx {

constexpr int kRBits = 8;       // reduced disparities in units of 1/256 (L#8)
constexpr int kMaxH = 1024;
constexpr int kStart = 3;       // start marker class (first stixel)

// ---------------------------------------------------------------------------
// K1: column reduction + transpose.
// One CTA = a tile of kRedRows image rows x (tc reduced columns) of one frame.
// Rows are read coalesced into shared memory; each thread then emits one
// reduced value (c, v), consecutive threads -> consecutive v (coalesced,
// transposed writes).
// ---------------------------------------------------------------------------
constexpr int kRedRows = 32;
constexpr int kRedThreads = 256;

struct ReduceArgs {
  const uint8_t* disp;
  int64_t pitch;        // bytes
  int W, H, n_cols, s, tc, q_bits, D, bpp;
  uint32_t invalid;
  uint16_t* out;        // [batch][n_cols][H], 0xFFFF = invalid
};

__global__ void __launch_bounds__(kRedThreads) reduce_kernel(ReduceArgs a) {
  extern __shared__ uint16_t tile[];             // [kRedRows][tpx + 1]
  const int frame = blockIdx.z;
  const int r0 = blockIdx.y * kRedRows;
  const int c0 = blockIdx.x * a.tc;
  const int ncl = min(a.tc, a.n_cols - c0);
  const int tpx = a.tc * a.s;                    // pixels per tile row
  const int px = ncl * a.s;
  const int stride = tpx + 1;
  const int nrows = min(kRedRows, a.H - r0);
  const uint8_t* base = a.disp + (int64_t)frame * a.H * a.pitch + (int64_t)r0 * a.pitch;
  if (a.bpp == 2) {
    for (int i = threadIdx.x; i < nrows * px; i += kRedThreads) {
      int r = i / px, x = i - r * px;
      const uint16_t* row = reinterpret_cast<const uint16_t*>(base + (int64_t)r * a.pitch);
      tile[r * stride + x] = __ldg(row + c0 * a.s + x);
    }
  } else {
    for (int i = threadIdx.x; i < nrows * px; i += kRedThreads) {
      int r = i / px, x = i - r * px;
      tile[r * stride + x] = __ldg(base + (int64_t)r * a.pitch + c0 * a.s + x);
    }
  }
  __syncthreads();
  const uint32_t lim = (uint32_t)a.D << a.q_bits;
  for (int i = threadIdx.x; i < ncl * kRedRows; i += kRedThreads) {
    int cl = i / kRedRows, rr = kRedRows - 1 - (i - cl * kRedRows);  // v ascending
    if (rr >= nrows) continue;
    const uint16_t* p = tile + rr * stride + cl * a.s;
    uint32_t sum = 0, n = 0;
    for (int x = 0; x < a.s; ++x) {
      uint32_t u = p[x];
      bool ok = (u != a.invalid) && (u < lim);
      sum += ok ? u : 0u;
      n += ok ? 1u : 0u;
    }
    uint16_t val = 0xFFFF;
    if (n) {
      // round half up of 2^R*sum/(2^Q*n) = floor((sum*2^(R+1-Q) + n) / (2n))
      uint64_t num = ((uint64_t)sum << (kRBits + 1 - a.q_bits)) + n;
      val = (uint16_t)(num / (2ull * n));
    }
    int r = r0 + rr;
    int v = a.H - 1 - r;
    a.out[((int64_t)frame * a.n_cols + c0 + cl) * a.H + v] = val;
  }
}

// ---------------------------------------------------------------------------
// K3: DP kernel (prefix sums + object-LUT rows + Eq. 5-6 DP + backtracking).
//
// Work unit: one column, handled by a "column group" of kCW = 4 warps with its
// own named barrier.  Lanes own targets k = K0 + lane of a 32-row block b
// (K0 = 32 b).  The object LUT LUT_object[f][v] (D x (h+1)) is never
// materialised; per block, the 32 target rows priv_b[i][f] = LUT[f][K0+i+1]
// live in shared memory (double-buffered), and the bottom row LUT[.][j] is
// carried incrementally in a per-warp ring seeded from an anchor row
// (row_{j+1} = row_j + Pair[.][d_j]).
//
// Roles.  Warp 0 (the "serial" warp) runs, per block, the part of Eq. 6 that is
// inherently sequential: targets K0 < j <= k in the same block need C[.][j-1]
// of the step before (the paper's barrier per step), done here in
// registers with warp shuffles.  Warps 1-3 (the "rectangle" warps) compute,
// for the NEXT block b+1 and while warp 0 works on block b, every cell whose
// bottom j is already final: its 32 target rows, and bottoms j <= K0 in 32-row
// chunks.  Only the newest chunk (bottoms of block b) waits for warp 0, and is
// split three ways.  The serial warp also finalises each target: ground and
// sky running minima (their data term does not depend on the predecessor, so
// GR^k = PG[k+1] + min_j (C_O[j-1] + t - PG[j])), the index table and
// the 32-byte record of row k+1 that later rectangles read.
// Exact mode (L#22): all costs are integer quanta < 2^24 carried in fp32, so
// adds/mins are exact and every decision matches the oracle.
// ---------------------------------------------------------------------------
constexpr int kCW = 4;                 // warps per column

struct DPArgs {
  const uint16_t* cols;    // [items][h] reduced columns (model order), 0xFFFF invalid
  stixel_t* out;           // [items][cap]
  int32_t* count;          // [items]
  float* col_cost;         // [items] or null
  float* scratch;          // [grid*cols_per_cta][2][h+1]  ground / sky prefix sums
  const float* E;          // [4][esz] object pair-cost windows (host built)
  const uint32_t* M2;      // [h+1] magic reciprocals ceil(2^31/n)
  const float* gG;         // ground cost by |dR - dgR|, length LG (last = cap)
  const float* gS;         // sky cost by dR, length LS (last = cap)
  const int* dgR;          // [h] ground model, 1/256 units
  int* overflow;
  int h, D, n_cols, items, cap, LG, LS, esz, dmr_inv, ord_margin, cols_per_cta;
  int col_bytes, shared_bytes;   // smem layout
  float capQ, cost_scale;
  float piFirstO, piFirstG;      // first-stixel priors (incl. BIC)
  float kOO_lo, kOO_hi;          // O above O: trans + ordering (lo: no violation)
  float kGO_mid, kGO_hi, kGO_lo; // O above G: trans + gravity level
  float kOG, kGS, kOS;           // G above O, S above G, S above O
  uint32_t thr[kMaxH];           // per row j: (thrA[j]+1) | thrB[j] << 16, both
                                 // clamped to [0, 65535]: f >= lo16 <=> floating,
                                 // f < hi16 <=> below ground (unsigned compares)
};

struct ColSmem {
  float* priv;      // [32][DP+1]     priv[i][f] = LUT_object[f][32b+i+1] of the block being built
  float* seed;      // [2][2][DP]     LUT rows 32b+12, 32b+24 of block b (parity b & 1)
  float* anchor;    // [nb+1][DP]     anchor[m][f] = LUT_object[f][32m]
  float* ring;      // [3][4][DP]     rectangle warps' rings of LUT_object[.][j]
  float* cbd;       // [496]          triangle cells (bottom K0+1+j', target K0+k' > j'), packed
  uint16_t* cbf;    // [496]          ... f | gravity level << 12
  uint4* rec;       // [h+1][2]       row j: {AO0,AO1,AGm,AGh} {AGl, T[j], N4[j]|ordthr<<16, thr}
  uint32_t* eo;     // [h+2]          lo16: ring window byte offset; hi16: E0 byte offset
  uint16_t* argO;   // [h]            j | c'<<12
  uint16_t* argG;   // [h]            j (pred class O, or start if j == 0)
  uint16_t* argS;   // [h]            j | c'<<12
  uint8_t* fpv;     // [h]            f of the last stixel of the best O-ending segmentation
  float2* part;     // [3][32]        rectangle partial minima {cost, argj}
  float4* pgps;     // [32]           serial warp: {PG[k], PG[k+1], PS[k], PS[k+1]}
};

constexpr int kTri = 496;              // cells of a 32-row triangle: sum_{j'<31} (31 - j')
__host__ __device__ constexpr int tri_off(int jp) { return 31 * jp - (jp * (jp - 1)) / 2; }

__host__ __device__ inline int al16(int x) { return (x + 15) & ~15; }

template <int DP>
__host__ __device__ inline int col_smem_bytes(int h) {
  const int nb = (h + 31) >> 5;
  int b = 0;
  b += al16(32 * (DP + 1) * 4);
  b += al16(4 * DP * 4);
  b += al16((nb + 1) * DP * 4);
  b += al16(3 * 4 * DP * 4);                      // rings, then cells (contiguous:
  b += al16(kTri * 4) + al16(kTri * 2);           //  prologue temporaries reuse both)
  b += al16((h + 1) * 32);
  b += al16((h + 2) * 4);
  b += al16(h * 2) * 3;
  b += al16(h);
  b += al16(3 * 32 * 8);
  b += al16(32 * 16);
  return b;
}

template <int DP>
__device__ inline ColSmem carve(uint8_t* p, int h) {
  const int nb = (h + 31) >> 5;
  ColSmem w;
  w.priv = reinterpret_cast<float*>(p); p += al16(32 * (DP + 1) * 4);
  w.seed = reinterpret_cast<float*>(p); p += al16(4 * DP * 4);
  w.anchor = reinterpret_cast<float*>(p); p += al16((nb + 1) * DP * 4);
  w.ring = reinterpret_cast<float*>(p); p += al16(3 * 4 * DP * 4);
  w.cbd = reinterpret_cast<float*>(p); p += al16(kTri * 4);
  w.cbf = reinterpret_cast<uint16_t*>(p); p += al16(kTri * 2);
  w.rec = reinterpret_cast<uint4*>(p); p += al16((h + 1) * 32);
  w.eo = reinterpret_cast<uint32_t*>(p); p += al16((h + 2) * 4);
  w.argO = reinterpret_cast<uint16_t*>(p); p += al16(h * 2);
  w.argG = reinterpret_cast<uint16_t*>(p); p += al16(h * 2);
  w.argS = reinterpret_cast<uint16_t*>(p); p += al16(h * 2);
  w.fpv = p; p += al16(h);
  w.part = reinterpret_cast<float2*>(p); p += al16(3 * 32 * 8);
  w.pgps = reinterpret_cast<float4*>(p);
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

// Gravity penalty by level (0 mid, 1 floating, 2 below ground) as two selects.
__device__ __forceinline__ float pen3(int lvl, float mid, float hi, float lo) {
  float r;
  asm("{\n\t.reg .pred p1, p2;\n\t.reg .f32 t;\n\t"
      "setp.eq.s32 p1, %1, 1;\n\tsetp.eq.s32 p2, %1, 2;\n\t"
      "selp.f32 t, %3, %2, p1;\n\tselp.f32 %0, %4, t, p2;\n\t}"
      : "=f"(r) : "r"(lvl), "f"(mid), "f"(hi), "f"(lo));
  return r;
}

__device__ __forceinline__ void named_bar(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Object model value f of span [j, k] from prefix differences:
// f = floor(t / (256 n)), t = sum(d + 128) over valid pixels: the exact half-up
// rounded mean (L#10), via a multiply-high by ceil(2^31/n) (exact for t < 2^28),
// clamped to D-1.  M2 sits at shared offset 0; n4 = 4n is its byte offset.
__device__ __forceinline__ int span_f(uint32_t t, uint32_t n4, const uint8_t* smem0, int Dm1) {
  uint32_t y = t >> (kRBits - 1);
  uint32_t M = *reinterpret_cast<const uint32_t*>(smem0 + n4);
  return min((int)__umulhi(y, M), Dm1);
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float ldsf(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

// Per-row uniform values of record j for the cell evaluation.
struct RowU {
  float AO0, AO1, AGm, AGh, AGl;
  uint32_t T, N4;
  int ordthr, thrA1, thrB;
};
__device__ __forceinline__ RowU load_row(const uint4* rec, int j) {
  const uint32_t ra = (uint32_t)__cvta_generic_to_shared(rec + 2 * j);
  uint4 x = lds128(ra), y = lds128(ra + 16);
  RowU u;
  u.AO0 = __uint_as_float(x.x); u.AO1 = __uint_as_float(x.y);
  u.AGm = __uint_as_float(x.z); u.AGh = __uint_as_float(x.w);
  u.AGl = __uint_as_float(y.x);
  u.T = y.y; u.N4 = y.z & 0xffffu; u.ordthr = (int)(y.z >> 16);
  u.thrA1 = (int)(y.w & 0xffffu); u.thrB = (int)(y.w >> 16);
  return u;
}

// Plain (compiler-visible) version: records are read-only while a rectangle runs.
__device__ __forceinline__ RowU load_row_c(const uint4* rec, int j) {
  const uint4 x = rec[2 * j], y = rec[2 * j + 1];
  RowU u;
  u.AO0 = __uint_as_float(x.x); u.AO1 = __uint_as_float(x.y);
  u.AGm = __uint_as_float(x.z); u.AGh = __uint_as_float(x.w);
  u.AGl = __uint_as_float(y.x);
  u.T = y.y; u.N4 = y.z & 0xffffu; u.ordthr = (int)(y.z >> 16);
  u.thrA1 = (int)(y.w & 0xffffu); u.thrB = (int)(y.w >> 16);
  return u;
}

template <int DP>
__global__ void __launch_bounds__(32 * kCW * 4, 1) dp_kernel(const __grid_constant__ DPArgs a) {
  constexpr int NR = DP / 128;         // LDS.128 ring windows per lane
  constexpr int NS = DP / 32;          // 32-wide f slices
  constexpr int NSW = (NS + 2) / 3;    // f slices per rectangle warp (at most)
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  // Warp roles: the C serial warps take the highest warp ids (the issue arbiter
  // prefers high ids; SMSP = wid % 4), the 3C rectangle warps the rest, spread so
  // that a column's warps sit on different SM sub-partitions where possible.
  const int C = a.cols_per_cta;
  int cslot, w;
  if (wid >= 3 * C) {
    cslot = wid - 3 * C; w = 0;
  } else if (C == 4) {
    cslot = ((wid & 3) + (wid >> 2) + 1) & 3; w = 1 + (wid >> 2);
  } else {
    cslot = wid % C; w = 1 + wid / C;
  }
  const int rw = w - 1;                // rectangle warp index 0..2, -1 for the serial warp
  const int ctid = w * 32 + lane;      // thread index within the column group
  const int h = a.h;
  const int Dm1 = a.D - 1;
  const int nb = (h + 31) >> 5;
  const int bar_col = 1 + cslot;       // 128 threads: whole column group
  const int bar_rect = 1 + C + cslot;  // 96 threads: rectangle warps

  // CTA-shared tables: M2 at offset 0, then 4 shifted copies of the object
  // pair-cost window E (Pair[f][d] = E[f - d + D]).
  uint32_t* M2s = reinterpret_cast<uint32_t*>(smem);
  float* E = reinterpret_cast<float*>(smem + al16((h + 1) * 4));
  uint16_t* tri_jk = reinterpret_cast<uint16_t*>(smem + al16((h + 1) * 4) + 4 * a.esz * 4);
  for (int i = threadIdx.x; i <= h; i += blockDim.x) M2s[i] = a.M2[i];
  for (int i = threadIdx.x; i < 4 * a.esz; i += blockDim.x) E[i] = a.E[i];
  for (int jp = 0; jp < 31; ++jp)                 // triangle cell index -> (j', k')
    for (int kp = jp + 1 + (int)threadIdx.x; kp < 32; kp += blockDim.x)
      tri_jk[tri_off(jp) + kp - jp - 1] = (uint16_t)(jp | (kp << 8));
  __syncthreads();
  const uint8_t* Eb = reinterpret_cast<const uint8_t*>(E);

  ColSmem cs = carve<DP>(smem + a.shared_bytes + cslot * a.col_bytes, h);
  float* ringw = cs.ring + (rw < 0 ? 0 : rw) * 4 * DP;
  const float INF = __int_as_float(0x7f800000);
  const int slot_global = blockIdx.x * a.cols_per_cta + cslot;
  float* PGg = a.scratch + (int64_t)slot_global * 2 * (h + 1);
  float* PSg = PGg + (h + 1);

  // ---- rectangle-warp helpers ---------------------------------------------
  // one ring step: rr += Pair[.][d_src] for f = 4*lane.. (+128 r); store to slot
  auto ring_step = [&](float (&rr)[4 * NR], int row_src, int slot) {
    uint32_t e = cs.eo[row_src] & 0xffffu;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      float4 x = *reinterpret_cast<const float4*>(Eb + e + 16 * lane + 512 * r);
      rr[4 * r + 0] += x.x; rr[4 * r + 1] += x.y; rr[4 * r + 2] += x.z; rr[4 * r + 3] += x.w;
      *reinterpret_cast<float4*>(ringw + slot * DP + 4 * lane + 128 * r) =
          make_float4(rr[4 * r + 0], rr[4 * r + 1], rr[4 * r + 2], rr[4 * r + 3]);
    }
  };
  // Bottoms j0 .. j0+nsteps-1 (j0 = 1 mod 4, nsteps = 0 mod 4, last record read
  // j0+nsteps+1 <= h) for this warp's targets (priv row pp); `seed` is the LUT
  // row LUT[.][j0-1].  Software-pipelined: the next pair's records and object
  // means are computed before the current pair's table loads.
  auto rect_run = [&](const float* seed, int j0, int nsteps, const float* pp, uint32_t Tk,
                      uint32_t N4k, float& best, int& argj) {
    float rr[4 * NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      float4 x = make_float4(seed[4 * lane + 128 * r], seed[4 * lane + 128 * r + 1],
                             seed[4 * lane + 128 * r + 2], seed[4 * lane + 128 * r + 3]);
      rr[4 * r + 0] = x.x; rr[4 * r + 1] = x.y; rr[4 * r + 2] = x.z; rr[4 * r + 3] = x.w;
    }
    ring_step(rr, j0 - 1, 1);
    ring_step(rr, j0, 2);
    RowU r0 = load_row_c(cs.rec, j0), r1 = load_row_c(cs.rec, j0 + 1);
    int f0 = span_f(Tk - r0.T, N4k - r0.N4, smem, Dm1);
    int f1 = span_f(Tk - r1.T, N4k - r1.N4, smem, Dm1);
    __syncwarp();
#pragma unroll 1
    for (int jj = 0; jj < nsteps; jj += 4) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int jA = j0 + jj + 2 * half;          // slots (jA & 3) = 1 + 2 half
        // prefetch the next pair (rows jA+2, jA+3; static fields only matter for f)
        // (clamped: the pair after the last one is loaded but not used)
        const RowU n0 = load_row_c(cs.rec, min(jA + 2, h)), n1 = load_row_c(cs.rec, min(jA + 3, h));
        const int g0 = span_f(Tk - n0.T, N4k - n0.N4, smem, Dm1);
        const int g1 = span_f(Tk - n1.T, N4k - n1.N4, smem, Dm1);
        const float* ra = ringw + ((1 + 2 * half) & 3) * DP;
        const float* rb = ringw + ((2 + 2 * half) & 3) * DP;
        {
          float data = pp[f0] - ra[f0];
          float aO = (f0 > r0.ordthr) ? r0.AO1 : r0.AO0;
          float aG = (f0 >= r0.thrA1) ? r0.AGh : ((f0 < r0.thrB) ? r0.AGl : r0.AGm);
          float cand = data + fminf(aO, aG);
          if (cand < best) { best = cand; argj = jA; }
        }
        {
          float data = pp[f1] - rb[f1];
          float aO = (f1 > r1.ordthr) ? r1.AO1 : r1.AO0;
          float aG = (f1 >= r1.thrA1) ? r1.AGh : ((f1 < r1.thrB) ? r1.AGl : r1.AGm);
          float cand = data + fminf(aO, aG);
          if (cand < best) { best = cand; argj = jA + 1; }
        }
        ring_step(rr, jA + 1, (3 + 2 * half) & 3);
        ring_step(rr, jA + 2, (4 + 2 * half) & 3);
        r0 = n0; r1 = n1; f0 = g0; f1 = g1;
        __syncwarp();
      }
    }
  };

  float fr[NSW];                       // rectangle warps: LUT_object[f][32 bt] of their f slices

  for (int item = slot_global; item < a.items; item += gridDim.x * a.cols_per_cta) {
    const uint16_t* col = a.cols + (int64_t)item * h;
    // ---------------- prologue A (all 4 warps): per-pixel costs (a3-a4) ----------
    float* tG = cs.ring;                 // temporaries in the (idle) ring + cell area
    float* tS = cs.ring + h;
    uint32_t* tD = reinterpret_cast<uint32_t*>(cs.ring + 2 * h);
    for (int v = ctid; v < h + 2; v += kCW * 32) {
      int dR = -1;
      if (v < h) {
        uint32_t u = col[v];
        dR = (u == 0xffffu) ? -1 : (int)u;
      }
      bool valid = dR >= 0;
      if (v < h) {
        float xg = a.capQ, xs = a.capQ;
        if (valid) {
          xg = __ldg(a.gG + min(abs(dR - __ldg(a.dgR + v)), a.LG - 1));
          xs = __ldg(a.gS + min(dR, a.LS - 1));
        }
        tG[v] = xg; tS[v] = xs;
        tD[v] = valid ? (uint32_t)dR + (1u << (kRBits - 1)) : 0u;
        cs.rec[2 * v + 3].w = a.thr[v + 1 < h ? v + 1 : h - 1];
      }
      // object pixel disparity rounded half up (L#9) -> E offsets of this row
      int dmr = valid ? a.D - ((dR + (1 << (kRBits - 1))) >> kRBits) : a.dmr_inv;
      int cc = dmr & 3;
      cs.eo[v] = (uint32_t)(cc * a.esz * 4 + (dmr - cc) * 4) | ((uint32_t)(dmr * 4) << 16);
    }
    for (int i = ctid; i < DP; i += kCW * 32) cs.anchor[i] = 0.f;   // anchor 0 = LUT[.][0] = 0
    named_bar(bar_col, kCW * 32);

    // build priv rows of block bt (rectangle warps, f slices rw, rw+3, ...) and the
    // anchor row 32(bt+1): a sequential prefix over rows, per f.  The
    // row offsets come from lane registers by shuffle; loads of 8 rows are issued
    // before their prefix chain.
    auto build_priv = [&](int bt) {
      const int K0b = bt << 5;
      const int rows = min(32, h - K0b);
      const uint32_t eor = cs.eo[K0b + min(lane, rows - 1)] >> 16;
      const int nq = (NS - rw + 2) / 3;            // slices of this warp (warp-uniform)
      for (int i0 = 0; i0 < rows; i0 += 8) {
        float x[8][NSW];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const uint32_t e = __shfl_sync(0xffffffffu, eor, (i0 + r) & 31);
          const float* src = reinterpret_cast<const float*>(Eb + e) + 32 * rw + lane;
#pragma unroll
          for (int q = 0; q < NSW; ++q) x[r][q] = (q < nq) ? src[96 * q] : 0.f;
        }
        const int rn = min(8, rows - i0);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          if (r < rn) {
            float* dst = cs.priv + (i0 + r) * (DP + 1) + 32 * rw + lane;
#pragma unroll
            for (int q = 0; q < NSW; ++q) {
              fr[q] += x[r][q];
              if (q < nq) dst[96 * q] = fr[q];
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < NSW; ++q)
        if (q < nq) cs.anchor[(bt + 1) * DP + 32 * rw + 96 * q + lane] = fr[q];
    };
    // triangle cells of block bt: bottom K0+1+j', target K0+k' (k' > j'); their
    // bottoms' LUT rows are the block's own priv rows: data, f, gravity level.
    // The 496 cells are spread densely over the 96 rectangle threads.  Also keeps
    // the LUT rows K0+12 and K0+24 as seeds for block bt+1's newest chunk.
    auto precompute_cells = [&](int bt) {
      const int K0b = bt << 5;
      const int jn = min(K0b + 31, h - 1) - K0b;
      const int ncell = tri_off(jn);
      for (int idx = rw * 32 + lane; idx < ncell; idx += 96) {
        const uint32_t jk = tri_jk[idx];
        const int jp = jk & 0xff, kp = jk >> 8;
        const int k = K0b + kp;
        if (k < h) {
          const uint4 ry = cs.rec[2 * (K0b + jp + 1) + 1];
          const uint4 rk = cs.rec[2 * (k + 1) + 1];
          int f = span_f(rk.y - ry.y, (rk.z & 0xffffu) - (ry.z & 0xffffu), smem, Dm1);
          float data = cs.priv[kp * (DP + 1) + f] - cs.priv[jp * (DP + 1) + f];
          int lvl = (f >= (int)(ry.w & 0xffffu)) ? 1 : ((f < (int)(ry.w >> 16)) ? 2 : 0);
          cs.cbd[idx] = data;
          cs.cbf[idx] = (uint16_t)(f | (lvl << 12));
        }
      }
      if (rw < 2 && K0b + 32 < h) {     // seeds (only needed if a next block exists)
        float* sd = cs.seed + ((bt & 1) * 2 + rw) * DP;
        const float* row = cs.priv + (12 * rw + 11) * (DP + 1);
        for (int f = lane; f < DP; f += 32) sd[f] = row[f];
      }
    };

    // ---------------- prologue B (warp 0): prefix sums ---------------
    // meanwhile the rectangle warps build block 0's priv rows
    if (w == 0) {
      float cg = 0.f, cs_ = 0.f;
      uint32_t ct = 0, cn = 0;
      if (lane == 0) { PGg[0] = 0.f; PSg[0] = 0.f; }
      for (int v0 = 0; v0 < h; v0 += 32) {
        int v = v0 + lane;
        float xg = 0.f, xs = 0.f;
        uint32_t xt = 0, xn = 0;
        if (v < h) {
          xg = tG[v]; xs = tS[v]; xt = tD[v]; xn = xt ? 4u : 0u;
        }
        float ig = warp_incl_scan(xg, lane) + cg;
        float is = warp_incl_scan(xs, lane) + cs_;
        uint32_t it = warp_incl_scan(xt, lane) + ct;
        uint32_t in = warp_incl_scan(xn, lane) + cn;
        if (v < h) {
          PGg[v + 1] = ig; PSg[v + 1] = is;
          cs.rec[2 * (v + 1) + 1].y = it;            // T[v+1]
          cs.rec[2 * (v + 1) + 1].z = in;            // N4[v+1]
        }
        cg = __shfl_sync(0xffffffffu, ig, 31);
        cs_ = __shfl_sync(0xffffffffu, is, 31);
        ct = __shfl_sync(0xffffffffu, it, 31);
        cn = __shfl_sync(0xffffffffu, in, 31);
      }
      __threadfence_block();
    } else {
#pragma unroll
      for (int q = 0; q < NSW; ++q) fr[q] = 0.f;
      build_priv(0);
    }
    named_bar(bar_col, kCW * 32);

    // rectangle warps: block 0 has only the j = 0 candidate (Eq. 5) and its triangle
    float rbest = INF;
    int rargj = 0x7fffffff;
    if (w != 0) {
      const int kk = lane < h ? lane : h - 1;
      const uint4 rky = cs.rec[2 * (kk + 1) + 1];
      const uint32_t Tk = rky.y, N4k = rky.z & 0xffffu;
      const float* pp = cs.priv + lane * (DP + 1);
      if (rw == 0) {
        int f = span_f(Tk, N4k, smem, Dm1);
        rbest = pp[f] + a.piFirstO;
        rargj = 0;
      }
      cs.part[rw * 32 + lane] = make_float2(rbest, __int_as_float(rargj));
      precompute_cells(0);
    }
    named_bar(bar_col, kCW * 32);

    // serial-warp state: running minima of ground / sky (warp-uniform), last C values
    float MG = a.piFirstG, MS = INF;
    int gj = 0, sj = 0, sc = kStart;
    float prevCO = INF, prevCG = INF, lastO = INF, lastG = INF, lastS = INF;
    int prevF = 0;

    for (int b = 0; b < nb; ++b) {
      const int K0 = b << 5;
      const int k = K0 + lane;
      if (w == 0) {
        // ============ serial warp: block b's triangle and finalisation ============
        const int kk = k < h ? k : h - 1;
        const uint4 rky = cs.rec[2 * (kk + 1) + 1];
        const uint32_t N4k = rky.z & 0xffffu;
        const uint32_t Tk = rky.y;
        const float pg0 = PGg[kk], pg1 = PGg[kk + 1], ps0 = PSg[kk], ps1 = PSg[kk + 1];
        float best = INF;
        int argj = 0x7fffffff;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          float2 p = cs.part[q * 32 + lane];
          int pj = __float_as_int(p.y);
          if (p.x < best || (p.x == best && pj < argj)) { best = p.x; argj = pj; }
        }
        // f and c' of the winner (the rectangle tracked only its j); packed
        // index-table entry: j | c' << 12 | f << 14
        int argf, argc;
        if (argj == 0) {
          argf = span_f(Tk, N4k, smem, Dm1);
          argc = kStart;
        } else {
          const RowU r = load_row(cs.rec, argj);
          argf = span_f(Tk - r.T, N4k - r.N4, smem, Dm1);
          float aO = (argf > r.ordthr) ? r.AO1 : r.AO0;
          float aG = (argf >= r.thrA1) ? r.AGh : ((argf < r.thrB) ? r.AGl : r.AGm);
          argc = (aG <= aO) ? 0 : 1;
        }
        int pack = argj | (argc << 12) | (argf << 14);
        cs.pgps[lane] = make_float4(pg0, pg1, ps0, ps1);
        __syncwarp();
        const float oh = opaque(a.kOO_hi), ol = opaque(a.kOO_lo);
        const float gh = opaque(a.kGO_hi), gl = opaque(a.kGO_lo), gm = opaque(a.kGO_mid);
        const int om = a.ord_margin;

        float myCG = 0.f;
        int myG = 0, myS = 0;
        // ground / sky running minima for target kf from C[kf-1] (warp-uniform)
        auto ground_sky = [&](int kf, float4 q) {
          if (kf == 0) {
            MG = a.piFirstG; gj = 0; MS = INF; sj = 0; sc = kStart;
          } else {
            float vG = prevCO + a.kOG - q.x;
            if (vG < MG) { MG = vG; gj = kf; }
            float v1 = prevCG + a.kGS - q.z;
            if (v1 < MS) { MS = v1; sj = kf; sc = 0; }
            float v2 = prevCO + a.kOS - q.z;
            if (v2 < MS) { MS = v2; sj = kf; sc = 1; }
          }
          float CGk = q.y + MG, CSk = q.w + MS;
          if (lane == kf - K0) { myCG = CGk; myG = gj; myS = sj | (sc << 12); }
          if (kf == h - 1) { lastG = CGk; lastS = CSk; }
          return CGk;
        };

        {  // target K0: all its bottoms were in the rectangle
          float COk = __shfl_sync(0xffffffffu, best, 0);
          int pk = __shfl_sync(0xffffffffu, pack, 0);
          float CGk = ground_sky(K0, cs.pgps[0]);
          prevCO = COk; prevCG = CGk; prevF = pk >> 14;
          if (K0 == h - 1) lastO = COk;
        }
        const int jn = min(K0 + 31, h - 1) - K0;
        // running minimum (over bottoms < j) of the next target to finalise
        float rB = __shfl_sync(0xffffffffu, best, 1);
        int rP = __shfl_sync(0xffffffffu, pack, 1);
        int off = 0;                                    // tri_off(jp)
        for (int jp = 0; jp < jn; ++jp) {
          const int j = K0 + jp + 1;                    // bottom j; target j finalised
          const float4 q = cs.pgps[jp + 1];
          // diagonal cell (bottom j, target j), evaluated redundantly by all lanes
          const float dd = cs.cbd[off];
          const int dfl = cs.cbf[off];
          const int df = dfl & 0xfff, dl = dfl >> 12;
          const float daO = prevCO + ((df > prevF + om) ? oh : ol);
          const float daG = prevCG + pen3(dl, gm, gh, gl);
          const bool dpg = daG <= daO;
          const float dc = dd + (dpg ? daG : daO);
          const bool take = dc < rB;
          const float COj = take ? dc : rB;
          const int Pj = take ? (j | ((dpg ? 0 : 1) << 12) | (df << 14)) : rP;
          // this lane's cell (bottom j, target k > j) with the same predecessors
          if (lane > jp) {
            const int idx = off + lane - jp - 1;
            const float data = cs.cbd[idx];
            const int fl = cs.cbf[idx];
            const int f = fl & 0xfff, lvl = fl >> 12;
            const float aO = prevCO + ((f > prevF + om) ? oh : ol);
            const float aG = prevCG + pen3(lvl, gm, gh, gl);
            const bool pg = aG <= aO;
            const float cand = data + (pg ? aG : aO);
            if (cand < best) { best = cand; pack = j | ((pg ? 0 : 1) << 12) | (f << 14); }
          }
          rB = __shfl_sync(0xffffffffu, best, (jp + 2) & 31);
          rP = __shfl_sync(0xffffffffu, pack, (jp + 2) & 31);
          const float CGj = ground_sky(j, q);
          prevCO = COj; prevCG = CGj; prevF = Pj >> 14;
          if (j == h - 1) lastO = COj;
          off += 31 - jp;
        }
        // every lane now holds the final values of its target row k: write the
        // record of row k+1 (consumed by later rectangles) and the index table
        if (k < h) {
          const int af = pack >> 14;
          cs.rec[2 * (k + 1)] = make_uint4(__float_as_uint(best + a.kOO_lo), __float_as_uint(best + a.kOO_hi),
                                           __float_as_uint(myCG + a.kGO_mid), __float_as_uint(myCG + a.kGO_hi));
          uint32_t* ry = reinterpret_cast<uint32_t*>(cs.rec + 2 * (k + 1) + 1);
          ry[0] = __float_as_uint(myCG + a.kGO_lo);
          ry[2] = N4k | ((uint32_t)(af + a.ord_margin) << 16);
          cs.argO[k] = (uint16_t)(pack & 0x3fff);
          cs.argG[k] = (uint16_t)myG;
          cs.argS[k] = (uint16_t)myS;
          cs.fpv[k] = (uint8_t)af;
        }
      }
      // ======== rectangle warps: block b+1, bottoms final before block b ========
      const int bn = b + 1;
      const int Kn = bn << 5;
      const bool has_next = bn < nb;
      uint32_t Tn = 0, N4n = 0;
      const float* ppn = cs.priv + lane * (DP + 1);
      if (w != 0 && has_next) {
        build_priv(bn);                  // block b's priv rows are no longer needed
        named_bar(bar_rect, 3 * 32);
        const int kk = Kn + lane < h ? Kn + lane : h - 1;
        const uint4 rky = cs.rec[2 * (kk + 1) + 1];
        Tn = rky.y; N4n = rky.z & 0xffffu;
        rbest = INF; rargj = 0x7fffffff;
        if (rw == 0) {                 // j = 0: first stixel spans 0..k (Eq. 5)
          int f = span_f(Tn, N4n, smem, Dm1);
          rbest = ppn[f] + a.piFirstO;
          rargj = 0;
        }
        // full chunks m <= b-1: their records (rows <= 32 b) were final before block b
        for (int m = rw; m <= b - 1; m += 3)
          rect_run(cs.anchor + m * DP, 32 * m + 1, 32, ppn, Tn, N4n, rbest, rargj);
      }
      named_bar(bar_col, kCW * 32);
      if (w != 0 && has_next) {
        // newest chunk (bottoms K0+1 .. K0+32, final after block b's triangle),
        // split 12 / 12 / 8 rows, seeded from LUT rows K0, K0+12, K0+24
        const int j0 = K0 + 1 + 12 * rw;
        const int ns = (rw == 2) ? 8 : 12;
        const float* seed = (rw == 0) ? cs.anchor + b * DP : cs.seed + ((b & 1) * 2 + rw - 1) * DP;
        rect_run(seed, j0, ns, ppn, Tn, N4n, rbest, rargj);
        cs.part[rw * 32 + lane] = make_float2(rbest, __int_as_float(rargj));
        precompute_cells(bn);
      }
      named_bar(bar_col, kCW * 32);
    }

    // ---------------- backtracking + extraction (a7), warp 0 ------------
    if (w == 0) {
      int c = 0;
      float cost = lastG;
      if (lastO < cost) { c = 1; cost = lastO; }
      if (lastS < cost) { c = 2; cost = lastS; }
      uint2* lst = reinterpret_cast<uint2*>(cs.priv);    // scratch (priv rows are dead)
      float* lsd = cs.priv + 2 * h;
      int n = 0;
      if (lane == 0) {
        int kb = h - 1;
        while (true) {
          int j, cp;
          float d;
          if (c == 1) {
            uint16_t x = cs.argO[kb]; j = x & 0xfff; cp = x >> 12; d = (float)cs.fpv[kb];
          } else if (c == 0) {
            j = cs.argG[kb]; cp = j ? 1 : kStart;
            d = (float)__ldg(a.dgR + j) * (1.0f / (1 << kRBits));
          } else {
            uint16_t x = cs.argS[kb]; j = x & 0xfff; cp = x >> 12; d = 0.f;
          }
          lst[n] = make_uint2((uint32_t)j | ((uint32_t)kb << 16), (uint32_t)c);
          lsd[n] = d;
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
      for (int i = lane; i < nw; i += 32) {
        uint2 e = lst[n - 1 - i];
        stixel_t s;
        s.bottom = (uint16_t)(e.x & 0xffff);
        s.top = (uint16_t)(e.x >> 16);
        s.cls = (uint8_t)e.y;
        s.pad[0] = s.pad[1] = s.pad[2] = 0;
        s.disparity = lsd[n - 1 - i];
        o[i] = s;
      }
      if (lane == 0) {
        a.count[item] = n;
        if (a.col_cost) a.col_cost[item] = cost * a.cost_scale;
        if (n > a.cap) atomicExch(a.overflow, 1);
      }
      __syncwarp();
    }
    named_bar(bar_col, kCW * 32);
  }
}

}  // namespace stx
