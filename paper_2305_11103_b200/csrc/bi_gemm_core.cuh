// Shared K1 machinery: the 128-byte-swizzled shared-memory tile layout, the
// DMMA.8x8x4 k-tile compute with permuted k-slots, and the fused epilogue.
// Both K1 paths -- TMA (bi_gemm_tma.cu) and cp.async (bi_gemm.cu) -- stage
// tiles in exactly this layout and run exactly this compute, so every path
// sums in the same order: results are bitwise identical whichever path a
// launch takes (and therefore across lanes, batches and rank counts).
//
// Layout per stage (CTA tile 128 x 128, k-tile 16):
//   A: 128 rows [m] of 16 doubles (128 B), 16-byte chunk c of row r stored at
//      chunk c ^ (r & 7)                           (== TMA SWIZZLE_128B)
//   B: 8 boxes of 16 columns; box row k (16 doubles) chunk c stored at
//      c ^ (k & 7)
// The four k-slots of DMMA k-step s use the permuted k sets
//   S0={0,3,12,15} S1={2,1,14,13} S2={4,7,8,11} S3={6,5,10,9}
// which make every A and B fragment load bank-conflict free in this layout.
#pragma once

#include "bi_common.cuh"

namespace bi {

constexpr int kK1Warps = 16;  // 4 x 4 warps of 32 x 32
constexpr int kK1Threads = kK1Warps * 32;
constexpr int kK1BoxB = 16 * 16 * 8;         // one B box: 16 k-rows x 16 doubles
constexpr int kK1StageA = kBM * kBK * 8;     // 16 KB
constexpr int kK1StageB = kBK * kBN * 8;     // 16 KB
constexpr int kK1Stage = kK1StageA + kK1StageB;

__device__ __forceinline__ int k1_kslot(int s, int j) {
  constexpr unsigned long long tbl = 0x9a56b874de12fc30ull;  // 4 bits per entry, [s][j]
  return (int)((tbl >> (4 * (s * 4 + j))) & 15);
}

// byte offset of A element (row r, k) / B element (k, n) inside a stage
__device__ __forceinline__ int k1_a_off(int r, int k) {
  return r * 128 + ((((k >> 1) ^ r) & 7) << 4) + ((k & 1) << 3);
}
__device__ __forceinline__ int k1_b_off(int k, int n) {
  const int nn = n & 15;
  return kK1StageA + (n >> 4) * kK1BoxB + k * 128 + ((((nn >> 1) ^ k) & 7) << 4) + ((nn & 1) << 3);
}

struct K1Frag {
  int aoff[4];
  int boff[4][2];
};

__device__ __forceinline__ void k1_frag_init(K1Frag& f, int fr, int fc) {
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int k = k1_kslot(s, fc);
    f.aoff[s] = ((((k >> 1) ^ fr) & 7) << 4) + ((k & 1) << 3);
#pragma unroll
    for (int h = 0; h < 2; ++h) f.boff[s][h] = k * 128 + ((((h * 4 + (fr >> 1)) ^ k) & 7) << 4) + ((fr & 1) << 3);
  }
}

__device__ __forceinline__ void k1_dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// One k-tile of DMMA on a stage (warp tile 32 x 32 at (wm, wn)).  StageA is
// the byte size of the stage's A part (tile rows x 128 B); B follows it.
template <int StageA = kK1StageA>
__device__ __forceinline__ void k1_compute(const uint8_t* stage, const K1Frag& f, int wm, int wn, int fr,
                                           double (&acc)[4][4][2]) {
  const uint8_t* sa = stage + (wm * 32 + fr) * 128;
  const uint8_t* sb = stage + StageA + (wn * 2) * kK1BoxB;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    double af[4], bf[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) af[i] = *reinterpret_cast<const double*>(sa + i * 8 * 128 + f.aoff[s]);
#pragma unroll
    for (int j = 0; j < 4; ++j) bf[j] = *reinterpret_cast<const double*>(sb + (j >> 1) * kK1BoxB + f.boff[s][j & 1]);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) k1_dmma(acc[i][j], af[i], bf[j]);
  }
}

// The same k-tile on a 64 x 32 warp tile (rows wm*64 .. +63): the two 32-row
// halves are exactly the 32 x 32 tiles (2wm, wn) and (2wm+1, wn) of
// k1_compute, with the same fragments and k-step order per accumulator --
// bitwise the same sums -- but each B fragment feeds 8 DMMAs instead of 4
// (0.375 instead of 0.5 shared loads per DMMA, half the warps per SM).
template <int StageA = kK1StageA>
__device__ __forceinline__ void k1_compute_64x32(const uint8_t* stage, const K1Frag& f, int wm, int wn, int fr,
                                                 double (&acc)[2][4][4][2]) {
  const uint8_t* sa = stage + (wm * 64 + fr) * 128;
  const uint8_t* sb = stage + StageA + (wn * 2) * kK1BoxB;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    double af[8], bf[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) af[i] = *reinterpret_cast<const double*>(sa + i * 8 * 128 + f.aoff[s]);
#pragma unroll
    for (int j = 0; j < 4; ++j) bf[j] = *reinterpret_cast<const double*>(sb + (j >> 1) * kK1BoxB + f.boff[s][j & 1]);
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) k1_dmma(acc[h][i][j], af[4 * h + i], bf[j]);
  }
}

// D = [C] + sign * acc with the output column remap; all C loads before any
// D store (C may alias D).  Every C load of the thread is issued before the
// first use, so the 16 loads overlap instead of paying one L2/DRAM latency
// each; full tiles with 16-byte-aligned, even-strided C/D and an even skip
// window (column pairs never straddle it) take branch-free 16-byte accesses.
template <int TM = kBM, int TN = kBN>
__device__ __forceinline__ void k1_epilogue(const GemmDesc& d, int bz, int m0, int n0, int wm, int wn, int fr, int fc,
                                            double (&acc)[4][4][2]) {
  pdl_trigger();
  const int mrem = d.M - m0, nrem = d.N - n0;
  const double* C = d.C ? d.C + bz * d.sC : nullptr;
  double* D = d.D + bz * d.sD;
  const double sgn = d.neg ? -1.0 : 1.0;
  const int skip_at = d.skip_at, skip_len = d.skip_len;
  auto pcol = [&](int g) { return g < skip_at ? g : g + skip_len; };
  const bool full = mrem >= TM && nrem >= TN && ((skip_at | skip_len) & 1) == 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc[i][j][0] *= sgn;
      acc[i][j][1] *= sgn;
    }
  if (C) {
    const bool vec = full && ((d.ldc & 1) == 0) && ((((uintptr_t)C) & 15) == 0);
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // two rounds of 8 loads in flight (register budget)
      double2 cv[2][4];
#pragma unroll
      for (int ii = 0; ii < 2; ++ii) {
        const int r = wm * 32 + (2 * h + ii) * 8 + fr;
        const int64_t row = m0 + r;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int cl = wn * 32 + j * 8 + 2 * fc;
          if (vec) {
            cv[ii][j] = __ldg(reinterpret_cast<const double2*>(C + row * d.ldc + pcol(n0 + cl)));
          } else {
            cv[ii][j] = make_double2(0.0, 0.0);
            if (r < mrem && cl < nrem) cv[ii][j].x = __ldg(C + row * d.ldc + pcol(n0 + cl));
            if (r < mrem && cl + 1 < nrem) cv[ii][j].y = __ldg(C + row * d.ldc + pcol(n0 + cl + 1));
          }
        }
      }
#pragma unroll
      for (int ii = 0; ii < 2; ++ii)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[2 * h + ii][j][0] += cv[ii][j].x;
          acc[2 * h + ii][j][1] += cv[ii][j].y;
        }
    }
  }
  if (full && ((d.ldd & 1) == 0) && ((((uintptr_t)D) & 15) == 0)) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t row = m0 + wm * 32 + i * 8 + fr;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<double2*>(D + row * d.ldd + pcol(n0 + wn * 32 + j * 8 + 2 * fc)) =
            make_double2(acc[i][j][0], acc[i][j][1]);
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = wm * 32 + i * 8 + fr;
    const int64_t row = m0 + r;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cl = wn * 32 + j * 8 + 2 * fc;
      if (r >= mrem || cl >= nrem) continue;
      const int p0 = pcol(n0 + cl), p1 = pcol(n0 + cl + 1);
      double* dp = D + row * d.ldd + p0;
      if (cl + 1 < nrem && p1 == p0 + 1 && (((uintptr_t)dp) & 15) == 0) {
        *reinterpret_cast<double2*>(dp) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        dp[0] = acc[i][j][0];
        if (cl + 1 < nrem) D[row * d.ldd + p1] = acc[i][j][1];
      }
    }
  }
}

// tile index -> (descriptor, batch item, tile origin)
struct K1Tile {
  int desc, bz, m0, n0;
};

#ifndef BI_K1_GROUP_M
#define BI_K1_GROUP_M 16
#endif
constexpr int kGroupM = BI_K1_GROUP_M;  // tile-rows per rasterisation group

template <int TM = kBM, int TN = kBN>
__device__ __forceinline__ K1Tile k1_locate(const GemmDesc* table, int count, int tile) {
  int lo = 0, hi = count - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (table[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
  }
  const GemmDesc& d = table[lo];
  const int local = tile - d.tile_begin;
  const int per = d.tiles_m * d.tiles_n;
  const int bz = local / per;
  const int rem = local - bz * per;
  // Grouped rasterisation: consecutive tiles walk kGroupM tile-rows down a
  // column of tiles before moving right, so the ~300 co-resident CTAs share
  // ~kGroupM A row-panels and ~300/kGroupM B column-panels in L2 instead of a
  // few A panels and EVERY B panel (row-major order re-read B from DRAM once
  // per tile-row: 61.5 GB for two 8192^3 products, ncu r02).  Only which CTA
  // computes a tile changes, so results are bitwise unchanged.
  const int first_m = (rem / (kGroupM * d.tiles_n)) * kGroupM;
  const int rows = min(d.tiles_m - first_m, kGroupM);
  const int r2 = rem - first_m * d.tiles_n;
  const int tm = first_m + r2 % rows;
  return K1Tile{lo, bz, tm * TM, (r2 / rows) * TN};
}

}  // namespace bi
