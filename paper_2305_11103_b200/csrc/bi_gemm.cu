// K1: FP64 block GEMM on the sm_100a FP64 tensor pipe (DMMA.8x8x4).
//
// Replaces the reference's only matrix-product kernel, core._mm_acc
// (/root/reference/pkg/src/blockinv/core.py:115-139), and every caller of it
// on the hot path: multiply / schur_accumulate (core.py:142-192),
// fox_block_multiply (engine.py:202-249) and the up/down assembly products
// (engine.py:414-437).
//
//   D = [C] + sign * A * B        (row-major, arbitrary ld, strided batched,
//                                  grouped over descriptors)
//
// tcgen05.mma has no f64 kind on sm_100a, so the FP64 tensor path is the
// warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4; measured 37.0 TF/s chip
// peak, profiles/r01_fp64_dmma_dfma_microbench.txt).  Tiles: 128x128x16 per
// CTA, 8 warps of 64x32, 4-stage cp.async ring in padded shared memory (row
// pads of 4 doubles make every fragment load bank-conflict free).
#include "bi_common.cuh"

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace bi {

thread_local int g_launch_priority = 0;
thread_local int g_gemm_grid_cap = 0;

int high_launch_priority() {
  static int prio = [] {
    int least = 0, greatest = 0;
    if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) return 0;
    return greatest;
  }();
  return prio;
}

namespace {

// Kernel configuration: WMW x WNW warps, each owning a WTM x WTN accumulator
// tile; CTA tile kBM x kBN (128 x 128); BK-deep k-tiles, STAGES-deep ring.
template <int WMW, int WNW, int WTM, int WTN, int BK, int STAGES>
struct Cfg {
  static constexpr int kThreads = WMW * WNW * 32;
  static constexpr int kFM = WTM / 8, kFN = WTN / 8;  // 8x8 DMMA fragments per warp
  static constexpr int kALd = BK + 4;   // A tile stored [m][k] (pad 4: conflict-free fragment loads)
  static constexpr int kBLd = kBN + 4;  // B tile stored [k][n]
  static constexpr int kAStage = kBM * kALd;
  static constexpr int kBStage = BK * kBLd;
  static constexpr int kSmem = STAGES * (kAStage + kBStage) * (int)sizeof(double);
  static_assert(WMW * WTM == kBM && WNW * WTN == kBN, "CTA tile must be 128 x 128");
  static_assert(kSmem <= 227 * 1024, "shared memory");
};

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

template <int WMW, int WNW, int WTM, int WTN, int BK, int STAGES>
__device__ __forceinline__ void gemm_tile(const GemmLaunch& L, const int tile, double* smem) {
  using C_ = Cfg<WMW, WNW, WTM, WTN, BK, STAGES>;
  constexpr int kThreads = C_::kThreads, kFM = C_::kFM, kFN = C_::kFN;
  constexpr int kALd = C_::kALd, kBLd = C_::kBLd, kAStage = C_::kAStage, kBStage = C_::kBStage;
  double* sA = smem;
  double* sB = smem + STAGES * kAStage;

  // ---- locate this tile's (descriptor, batch item, tile) ------------------
  const GemmDesc* table = (L.count <= kGemmInline) ? L.inl : L.descs;
  int lo = 0, hi = L.count - 1;
  while (lo < hi) {  // last descriptor whose tile_begin <= tile
    int mid = (lo + hi + 1) >> 1;
    if (table[mid].tile_begin <= tile) lo = mid; else hi = mid - 1;
  }
  const GemmDesc& d = table[lo];
  const int local = tile - d.tile_begin;
  const int per = d.tiles_m * d.tiles_n;
  const int bz = local / per;
  const int rem = local - bz * per;
  const int tm = rem / d.tiles_n;
  const int tn = rem - tm * d.tiles_n;
  const int m0 = tm * kBM, n0 = tn * kBN;
  const int mrem = d.M - m0, nrem = d.N - n0, K = d.K;
  const int64_t lda = d.lda, ldb = d.ldb;
  const double* __restrict__ A = d.A + bz * d.sA + (int64_t)m0 * lda;
  const double* __restrict__ B = d.B + bz * d.sB + n0;
  const bool al16 = ((((uintptr_t)A) | ((uintptr_t)B)) & 15) == 0 && ((lda | ldb) & 1) == 0;

  const int tid = threadIdx.x;
  // Interior tiles with aligned operands take the fast path: per-thread copy
  // pointers are computed once and advanced by BK per k-tile, no bounds checks.
  constexpr int kAChunks = (kBM * BK / 2) / kThreads, kBChunks = (BK * kBN / 2) / kThreads;
  constexpr int kAChunksRow = BK / 2, kBChunksRow = kBN / 2;
  const bool fast = al16 && mrem >= kBM && nrem >= kBN && (K % BK) == 0;
  const double* a_src[kAChunks];
  const double* b_src[kBChunks];
  int a_dst[kAChunks], b_dst[kBChunks];
#pragma unroll
  for (int i = 0; i < kAChunks; ++i) {
    const int q = tid + i * kThreads, row = q / kAChunksRow, cc = q % kAChunksRow;
    a_src[i] = A + (int64_t)row * lda + 2 * cc;
    a_dst[i] = row * kALd + 2 * cc;
  }
#pragma unroll
  for (int i = 0; i < kBChunks; ++i) {
    const int q = tid + i * kThreads, row = q / kBChunksRow, cc = q % kBChunksRow;
    b_src[i] = B + (int64_t)row * ldb + 2 * cc;
    b_dst[i] = row * kBLd + 2 * cc;
  }
  const int64_t b_step = (int64_t)BK * ldb;
  auto load_a_fast = [&](int stage, int kt) {
    double* as = sA + stage * kAStage;
#pragma unroll
    for (int i = 0; i < kAChunks; ++i) cp_async16(as + a_dst[i], a_src[i] + kt * BK, 16);
  };
  auto load_b_fast = [&](int stage, int kt) {
    double* bs = sB + stage * kBStage;
#pragma unroll
    for (int i = 0; i < kBChunks; ++i) cp_async16(bs + b_dst[i], b_src[i] + kt * b_step, 16);
  };
  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * BK;
    double* as = sA + stage * kAStage;
    double* bs = sB + stage * kBStage;
    if (al16) {
#pragma unroll
      for (int i = 0; i < kAChunks; ++i) {
        const int q = tid + i * kThreads;
        const int row = q / kAChunksRow, cc = q % kAChunksRow, kk = k0 + 2 * cc;
        int bytes = 0;
        const double* src = A;
        if (row < mrem && kk < K) {
          bytes = min(2, K - kk) * 8;
          src = A + (int64_t)row * lda + kk;
        }
        cp_async16(as + row * kALd + 2 * cc, src, bytes);
      }
#pragma unroll
      for (int i = 0; i < kBChunks; ++i) {
        const int q = tid + i * kThreads;
        const int row = q / kBChunksRow, cc = q % kBChunksRow, kk = k0 + row;
        int bytes = 0;
        const double* src = B;
        if (kk < K && 2 * cc < nrem) {
          bytes = min(2, nrem - 2 * cc) * 8;
          src = B + (int64_t)kk * ldb + 2 * cc;
        }
        cp_async16(bs + row * kBLd + 2 * cc, src, bytes);
      }
    } else {
#pragma unroll
      for (int i = 0; i < (kBM * BK) / kThreads; ++i) {
        const int q = tid + i * kThreads;
        const int row = q / BK, kc = q % BK, kk = k0 + kc;
        const bool ok = row < mrem && kk < K;
        cp_async8(as + row * kALd + kc, ok ? A + (int64_t)row * lda + kk : A, ok ? 8 : 0);
      }
#pragma unroll
      for (int i = 0; i < (BK * kBN) / kThreads; ++i) {
        const int q = tid + i * kThreads;
        const int row = q / kBN, nc = q % kBN, kk = k0 + row;
        const bool ok = kk < K && nc < nrem;
        cp_async8(bs + row * kBLd + nc, ok ? B + (int64_t)kk * ldb + nc : B, ok ? 8 : 0);
      }
    }
  };

  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp / WNW, wn = warp % WNW;
  const int fr = lane >> 2, fc = lane & 3;

  double acc[kFM][kFN][2];
#pragma unroll
  for (int i = 0; i < kFM; ++i)
#pragma unroll
    for (int j = 0; j < kFN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) {
      if (fast) {
        load_a_fast(s, s);
        load_b_fast(s, s);
      } else {
        load_stage(s, s);
      }
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nk = kt + STAGES - 1;
    const bool pre = nk < KT;
    const int nstage = nk % STAGES;
    const double* as = sA + (kt % STAGES) * kAStage + (wm * WTM + fr) * kALd + fc;
    const double* bs = sB + (kt % STAGES) * kBStage + fc * kBLd + wn * WTN + fr;
    if (pre && !fast) load_stage(nstage, nk);
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double af[kFM], bf[kFN];
#pragma unroll
      for (int i = 0; i < kFM; ++i) af[i] = as[i * 8 * kALd + ks * 4];
#pragma unroll
      for (int j = 0; j < kFN; ++j) bf[j] = bs[ks * 4 * kBLd + j * 8];
#pragma unroll
      for (int i = 0; i < kFM; ++i)
#pragma unroll
        for (int j = 0; j < kFN; ++j) dmma(acc[i][j], af[i], bf[j]);
      // spread the next stage's copies between k-steps (fast path)
      if (fast && pre) {
        if (ks == 0) load_a_fast(nstage, nk);
        if (ks == 1) load_b_fast(nstage, nk);
      }
    }
    cp_async_commit();
  }

  // ---- epilogue: D = [C] + sign * acc, with the optional column remap ----
  // All C loads are issued before any D store (C may alias D, so the
  // compiler cannot reorder them itself; interleaving would serialize one
  // DRAM round trip per fragment).
  const double* C = d.C ? d.C + bz * d.sC : nullptr;
  double* D = d.D + bz * d.sD;
  const int64_t ldc = d.ldc, ldd = d.ldd;
  const double sgn = d.neg ? -1.0 : 1.0;
  const int skip_at = d.skip_at, skip_len = d.skip_len;
  auto pcol = [&](int g) { return g < skip_at ? g : g + skip_len; };
#pragma unroll
  for (int i = 0; i < kFM; ++i)
#pragma unroll
    for (int j = 0; j < kFN; ++j) {
      acc[i][j][0] *= sgn;
      acc[i][j][1] *= sgn;
    }
  if (C) {
#pragma unroll
    for (int i = 0; i < kFM; ++i) {
      const int r = wm * WTM + i * 8 + fr;
      const int64_t row = m0 + r;
#pragma unroll
      for (int j = 0; j < kFN; ++j) {
        const int cl = wn * WTN + j * 8 + 2 * fc;
        if (r >= mrem || cl >= nrem) continue;
        const int p0 = pcol(n0 + cl), p1 = pcol(n0 + cl + 1);
        const double* cp = C + row * ldc + p0;
        if (cl + 1 < nrem && p1 == p0 + 1 && (((uintptr_t)cp) & 15) == 0) {
          const double2 cv = __ldg(reinterpret_cast<const double2*>(cp));
          acc[i][j][0] += cv.x;
          acc[i][j][1] += cv.y;
        } else {
          acc[i][j][0] += cp[0];
          if (cl + 1 < nrem) acc[i][j][1] += C[row * ldc + p1];
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kFM; ++i) {
    const int r = wm * WTM + i * 8 + fr;
    const int64_t row = m0 + r;
#pragma unroll
    for (int j = 0; j < kFN; ++j) {
      const int cl = wn * WTN + j * 8 + 2 * fc;
      if (r >= mrem || cl >= nrem) continue;
      const int p0 = pcol(n0 + cl), p1 = pcol(n0 + cl + 1);
      double* dp = D + row * ldd + p0;
      if (cl + 1 < nrem && p1 == p0 + 1 && (((uintptr_t)dp) & 15) == 0) {
        *reinterpret_cast<double2*>(dp) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        dp[0] = acc[i][j][0];
        if (cl + 1 < nrem) D[row * ldd + p1] = acc[i][j][1];
      }
    }
  }
}

// Persistent over tiles: a launch may use fewer CTAs than tiles (the engine
// caps GEMM grids to keep SMs free for the latency-bound leaf chains).
template <int WMW, int WNW, int WTM, int WTN, int BK, int STAGES>
__global__ void __launch_bounds__(WMW* WNW * 32, 1) gemm_dmma_kernel(const __grid_constant__ GemmLaunch L) {
  extern __shared__ __align__(128) double smem[];
  for (int tile = blockIdx.x; tile < L.total_tiles; tile += gridDim.x) {
    gemm_tile<WMW, WNW, WTM, WTN, BK, STAGES>(L, tile, smem);
    __syncthreads();  // the next tile's prologue reuses the stage ring
  }
}

// Variants (selected by BI_GEMM_VARIANT for tuning).  Default 4 = the TMA +
// mbarrier kernel of bi_gemm_tma.cu (16 warps of 32x32), falling back to
// variant 2 (cp.async, same warp layout) when operands are not 16-byte aligned
// or a launch has more than kGemmInline descriptors.
#define BI_GEMM_VARIANTS(X)                \
  X(0, 2, 4, 64, 32, 16, 4) /* 8 warps */  \
  X(1, 2, 4, 64, 32, 32, 3)                \
  X(2, 4, 4, 32, 32, 16, 4) /* 16 warps */ \
  X(3, 4, 4, 32, 32, 32, 3)

int g_variant = -1;

}  // namespace
bool launch_gemm_tma(const GemmDesc* h, int count, int grid_cap, cudaStream_t stream, cudaError_t* err);
namespace {

int gemm_variant() {
  if (g_variant < 0) {
    const char* v = getenv("BI_GEMM_VARIANT");
    g_variant = v ? atoi(v) : 4;
    if (g_variant < 0 || g_variant > 4) g_variant = 4;
  }
  return g_variant;
}

std::once_flag g_attr_once;
cudaError_t g_attr_err = cudaSuccess;

}  // namespace

int finalize_descs(GemmDesc* d, int count) {
  int t = 0;
  for (int i = 0; i < count; ++i) {
    const bool empty = d[i].M <= 0 || d[i].N <= 0 || d[i].batch <= 0;
    d[i].tiles_m = empty ? 0 : (d[i].M + kBM - 1) / kBM;
    d[i].tiles_n = empty ? 1 : (d[i].N + kBN - 1) / kBN;
    d[i].tile_begin = t;
    t += empty ? 0 : d[i].tiles_m * d[i].tiles_n * d[i].batch;
  }
  return t;
}

cudaError_t gemm_init_attributes() {
  std::call_once(g_attr_once, [] {
    cudaError_t e = cudaSuccess;
#define BI_SET_ATTR(id, a, b, c, d_, e_, f)                                                       \
  if (e == cudaSuccess)                                                                       \
    e = cudaFuncSetAttribute(gemm_dmma_kernel<a, b, c, d_, e_, f>,                            \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<a, b, c, d_, e_, f>::kSmem);
    BI_GEMM_VARIANTS(BI_SET_ATTR)
#undef BI_SET_ATTR
    g_attr_err = e;
  });
  return g_attr_err;
}

cudaError_t launch_gemm(const GemmDesc* h_descs, const GemmDesc* d_descs, int count,
                        cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  cudaError_t e = gemm_init_attributes();
  if (e != cudaSuccess) return e;
  const GemmDesc& last = h_descs[count - 1];
  const int total =
      last.tile_begin + ((last.M <= 0 || last.N <= 0 || last.batch <= 0) ? 0 : last.tiles_m * last.tiles_n * last.batch);
  if (total == 0) return cudaSuccess;
  GemmLaunch L{};
  L.count = count;
  L.total_tiles = total;
  if (count <= kGemmInline) {
    for (int i = 0; i < count; ++i) L.inl[i] = h_descs[i];
    L.descs = nullptr;
  } else {
    if (!d_descs) return cudaErrorInvalidValue;
    L.descs = d_descs;
  }
  const int grid = (g_gemm_grid_cap > 0 && g_gemm_grid_cap < total) ? g_gemm_grid_cap : total;
  if (gemm_variant() == 4) {
    cudaError_t te = cudaSuccess;
    if (launch_gemm_tma(h_descs, count, g_gemm_grid_cap, stream, &te)) return te;
  }
  switch (gemm_variant() == 4 ? 2 : gemm_variant()) {
#define BI_LAUNCH(id, a, b, c, d_, e_, f)                                                          \
  case id:                                                                                     \
    e = launch_kernel(gemm_dmma_kernel<a, b, c, d_, e_, f>, dim3(grid),                         \
                      dim3(Cfg<a, b, c, d_, e_, f>::kThreads), Cfg<a, b, c, d_, e_, f>::kSmem, stream, 1u, \
                      L);                                                                      \
    break;
    BI_GEMM_VARIANTS(BI_LAUNCH)
#undef BI_LAUNCH
  }
  return e;
}

}  // namespace bi
