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
// warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4; measured 36.98 TF/s chip
// peak, profiles/r01_fp64_dmma_dfma_microbench.txt).  Two feeders share one
// swizzled tile layout and one compute/epilogue (bi_gemm_core.cuh):
//   * TMA + mbarrier ring (bi_gemm_tma.cu) -- default when every operand is
//     16-byte aligned with even leading dimensions;
//   * this file's cp.async ring -- any alignment (8-byte copies when needed),
//     any number of descriptors.
// Both are persistent over tiles (the engine may cap the grid).
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "bi_gemm_core.cuh"

namespace bi {

thread_local int g_launch_priority = 0;
thread_local int g_launch_pdl = 0;
thread_local int g_gemm_grid_cap = 0;

int carveout_percent() {
  static const int v = [] {
    const char* e = getenv("BI_CARVEOUT");
    return e ? atoi(e) : -1;
  }();
  return v;
}

int high_launch_priority() {
  static int prio = [] {
    int least = 0, greatest = 0;
    if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) return 0;
    return greatest;
  }();
  return prio;
}

bool launch_gemm_tma(const GemmDesc* h, int count, int grid_cap, cudaStream_t stream, cudaError_t* err);

namespace {

constexpr int kStages = 4;

// Tile configurations of the cp.async feeder: TM x TN CTA tile of 32 x 32
// warp tiles.  128 x 128 (16 warps) is the throughput tile; 64 x 64 (4 warps)
// is the latency tile for the small trailing updates of K3, where one FP64 SM
// (~250 GF/s) would otherwise spend >4 us on a single 128 x 128 x 32 tile.
// Both sum every element in the same order (same k-tile / k-slot sequence per
// warp tile), so results do not depend on the tile shape.
template <int TM, int TN>
struct K1Cfg {
  static constexpr int kWN = TN / 32;
  static constexpr int kThreads = (TM / 32) * kWN * 32;
  static constexpr int kStageA = TM * kBK * 8;
  static constexpr int kStage = kStageA + kBK * TN * 8;
  static constexpr int kSmem = kStages * kStage + 1024;
  static constexpr int kMinBlocks = (TM == 128 && TN == 64) ? 2 : 1;  // 128 x 64: two CTAs per SM
};

__device__ __forceinline__ void cp_async16(uint8_t* smem, const double* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(uint8_t* smem, const double* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int TM, int TN>
__device__ __forceinline__ void gemm_tile(const GemmLaunch& L, const int tile, uint8_t* smem, const K1Frag& f,
                                          int wm, int wn, int fr, int fc) {
  using Cfg = K1Cfg<TM, TN>;
  constexpr int kThr = Cfg::kThreads;
  const GemmDesc* table = (L.count <= kGemmInline) ? L.inl : L.descs;
  const K1Tile tc = k1_locate<TM, TN>(table, L.count, tile);
  const GemmDesc& d = table[tc.desc];
  const int mrem = d.M - tc.m0, nrem = d.N - tc.n0, K = d.K;
  const int64_t lda = d.lda, ldb = d.ldb;
  const double* __restrict__ A = d.A + tc.bz * d.sA + (int64_t)tc.m0 * lda;
  const double* __restrict__ B = d.B + tc.bz * d.sB + tc.n0;
  const bool al16 = ((((uintptr_t)A) | ((uintptr_t)B)) & 15) == 0 && ((lda | ldb) & 1) == 0;
  const int tid = threadIdx.x;
  auto b_chunk = [&](int k, int cc) {  // byte offset of B chunk (k-row k, 16-byte chunk cc)
    return Cfg::kStageA + (cc >> 3) * kK1BoxB + k * 128 + (((cc & 7) ^ (k & 7)) << 4);
  };

  // copy one k-tile into a stage of the swizzled layout
  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * kBK;
    uint8_t* st = smem + stage * Cfg::kStage;
    if (al16) {
#pragma unroll
      for (int i = 0; i < (TM * kBK / 2) / kThr; ++i) {  // A: TM rows x 8 chunks
        const int q = tid + i * kThr;
        const int row = q >> 3, c = q & 7, kk = k0 + 2 * c;
        int bytes = 0;
        const double* src = A;
        if (row < mrem && kk < K) {
          bytes = min(2, K - kk) * 8;
          src = A + (int64_t)row * lda + kk;
        }
        cp_async16(st + row * 128 + ((c ^ (row & 7)) << 4), src, bytes);
      }
#pragma unroll
      for (int i = 0; i < (kBK * TN / 2) / kThr; ++i) {  // B: 16 rows x TN/2 chunks
        const int q = tid + i * kThr;
        const int k = q / (TN / 2), cc = q % (TN / 2), kk = k0 + k;
        int bytes = 0;
        const double* src = B;
        if (kk < K && 2 * cc < nrem) {
          bytes = min(2, nrem - 2 * cc) * 8;
          src = B + (int64_t)kk * ldb + 2 * cc;
        }
        cp_async16(st + b_chunk(k, cc), src, bytes);
      }
    } else {
#pragma unroll
      for (int i = 0; i < (TM * kBK) / kThr; ++i) {
        const int e = tid + i * kThr;
        const int row = e >> 4, kc = e & 15, kk = k0 + kc;
        const bool ok = row < mrem && kk < K;
        cp_async8(st + k1_a_off(row, kc), ok ? A + (int64_t)row * lda + kk : A, ok ? 8 : 0);
      }
#pragma unroll
      for (int i = 0; i < (kBK * TN) / kThr; ++i) {
        const int e = tid + i * kThr;
        const int k = e / TN, n = e % TN, kk = k0 + k;
        const bool ok = kk < K && n < nrem;
        cp_async8(st + b_chunk(k, n >> 1) + ((n & 1) << 3), ok ? B + (int64_t)kk * ldb + n : B, ok ? 8 : 0);
      }
    }
  };

  // interior tiles with aligned operands: no bounds checks
  const bool fast = al16 && mrem >= TM && nrem >= TN && (K % kBK) == 0;
  auto load_fast = [&](int stage, int kt) {
    uint8_t* st = smem + stage * Cfg::kStage;
#pragma unroll
    for (int i = 0; i < (TM * kBK / 2) / kThr; ++i) {
      const int q = tid + i * kThr, row = q >> 3, c = q & 7;
      cp_async16(st + row * 128 + ((c ^ (row & 7)) << 4), A + (int64_t)row * lda + kt * kBK + 2 * c, 16);
    }
#pragma unroll
    for (int i = 0; i < (kBK * TN / 2) / kThr; ++i) {
      const int q = tid + i * kThr, k = q / (TN / 2), cc = q % (TN / 2);
      cp_async16(st + b_chunk(k, cc), B + (int64_t)(kt * kBK + k) * ldb + 2 * cc, 16);
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = (K + kBK - 1) / kBK;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < KT) {
      if (fast) load_fast(s, s); else load_stage(s, s);
    }
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    const int nk = kt + kStages - 1;
    if (nk < KT) {
      if (fast) load_fast(nk % kStages, nk); else load_stage(nk % kStages, nk);
    }
    cp_async_commit();
    k1_compute<Cfg::kStageA>(smem + (kt % kStages) * Cfg::kStage, f, wm, wn, fr, acc);
  }
  k1_epilogue<TM, TN>(d, tc.bz, tc.m0, tc.n0, wm, wn, fr, fc, acc);
}

template <int TM, int TN>
__global__ void __launch_bounds__(K1Cfg<TM, TN>::kThreads, K1Cfg<TM, TN>::kMinBlocks)
    gemm_dmma_kernel(const __grid_constant__ GemmLaunch L) {
  pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp / K1Cfg<TM, TN>::kWN, wn = warp % K1Cfg<TM, TN>::kWN, fr = lane >> 2, fc = lane & 3;
  K1Frag f;
  k1_frag_init(f, fr, fc);
  for (int tile = blockIdx.x; tile < L.total_tiles; tile += gridDim.x) {
    gemm_tile<TM, TN>(L, tile, smem, f, wm, wn, fr, fc);
    cp_async_wait<0>();
    __syncthreads();  // the next tile's prologue reuses the stage ring
  }
}


// BI_GEMM_SMALL_TILES: 128-tile count below which a launch runs on the 64 x 64
// cp.async latency tiles.  Default 0 (off): since the TMA kernel runs 128 x 64
// tiles two CTAs per SM, it is as good on small launches and better in the
// engine (bench 29.1 -> 28.0 ms; profiles/r01_k1_variants.txt).
int small_tile_threshold() {
  static const int v = [] {
    const char* e = getenv("BI_GEMM_SMALL_TILES");
    return e ? atoi(e) : 0;
  }();
  return v;
}

int use_tma() {
  static const int v = [] {
    const char* e = getenv("BI_GEMM_TMA");
    return e ? atoi(e) : 1;
  }();
  return v;
}

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
  static PerDeviceOnce once;
  return once.run([] {
    cudaError_t e = cudaFuncSetAttribute(gemm_dmma_kernel<kBM, kBN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         K1Cfg<kBM, kBN>::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_dmma_kernel<64, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               K1Cfg<64, 64>::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_dmma_kernel<128, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               K1Cfg<128, 64>::kSmem);
    if (e == cudaSuccess) e = set_carveout(gemm_dmma_kernel<128, 64>);
    if (e == cudaSuccess) e = set_carveout(gemm_dmma_kernel<kBM, kBN>);
    if (e == cudaSuccess) e = set_carveout(gemm_dmma_kernel<64, 64>);
    return e;
  });
}

cudaError_t launch_gemm_small_n(const GemmDesc* h, int count, cudaStream_t stream);

cudaError_t launch_gemm(const GemmDesc* h_descs, const GemmDesc* d_descs, int count, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  cudaError_t e = gemm_init_attributes();
  if (e != cudaSuccess) return e;
  const GemmDesc& last = h_descs[count - 1];
  const int total =
      last.tile_begin + ((last.M <= 0 || last.N <= 0 || last.batch <= 0) ? 0 : last.tiles_m * last.tiles_n * last.batch);
  if (total == 0) return cudaSuccess;
  // Optional latency tiles for launches whose 128-tile grid cannot fill the GPU.
  if (count <= kGemmInline && total < small_tile_threshold()) return launch_gemm_small_n(h_descs, count, stream);
  if (use_tma()) {
    cudaError_t te = cudaSuccess;
    if (launch_gemm_tma(h_descs, count, g_gemm_grid_cap, stream, &te)) return te;
  }
  GemmLaunch L{};
  L.count = count;
  L.total_tiles = total;
  static const int cp_tn = [] {  // BI_GEMM_CP_TN: cp.async tile width (64: two CTAs per SM; 128)
    const char* v = getenv("BI_GEMM_CP_TN");
    return (v && atoi(v) == 128) ? 128 : 64;
  }();
  if (count <= kGemmInline && cp_tn == 64) {  // inline descriptors: re-tile for 128 x 64
    int t = 0;
    for (int i = 0; i < count; ++i) {
      GemmDesc d = h_descs[i];
      const bool empty = d.M <= 0 || d.N <= 0 || d.batch <= 0;
      d.tiles_m = empty ? 0 : (d.M + kBM - 1) / kBM;
      d.tiles_n = empty ? 1 : (d.N + 63) / 64;
      d.tile_begin = t;
      t += empty ? 0 : d.tiles_m * d.tiles_n * d.batch;
      L.inl[i] = d;
    }
    L.descs = nullptr;
    L.total_tiles = t;
    const int cap2 = g_gemm_grid_cap > 0 ? 2 * g_gemm_grid_cap : 0;
    const int grid2 = (cap2 > 0 && cap2 < t) ? cap2 : t;
    return launch_kernel(gemm_dmma_kernel<128, 64>, dim3(grid2), dim3(K1Cfg<128, 64>::kThreads),
                         (size_t)K1Cfg<128, 64>::kSmem, stream, 1u, L);
  }
  if (count <= kGemmInline) {
    for (int i = 0; i < count; ++i) L.inl[i] = h_descs[i];
    L.descs = nullptr;
  } else {
    if (!d_descs) return cudaErrorInvalidValue;
    L.descs = d_descs;
  }
  const int grid = (g_gemm_grid_cap > 0 && g_gemm_grid_cap < total) ? g_gemm_grid_cap : total;
  return launch_kernel(gemm_dmma_kernel<kBM, kBN>, dim3(grid), dim3(K1Cfg<kBM, kBN>::kThreads),
                       (size_t)K1Cfg<kBM, kBN>::kSmem, stream, 1u, L);
}

// Latency path: <= kGemmInline descriptors on 64 x 64 tiles, one CTA per tile
// (4x the CTAs of the 128 x 128 tiling).  Same summation order as launch_gemm.
cudaError_t launch_gemm_small_n(const GemmDesc* h, int count, cudaStream_t stream) {
  cudaError_t e = gemm_init_attributes();
  if (e != cudaSuccess) return e;
  if (count <= 0 || count > kGemmInline) return cudaErrorInvalidValue;
  GemmLaunch L{};
  L.count = count;
  L.descs = nullptr;
  int t = 0;
  for (int i = 0; i < count; ++i) {
    GemmDesc d = h[i];
    const bool empty = d.M <= 0 || d.N <= 0 || d.batch <= 0;
    d.tiles_m = empty ? 0 : (d.M + 63) / 64;
    d.tiles_n = empty ? 1 : (d.N + 63) / 64;
    d.tile_begin = t;
    t += empty ? 0 : d.tiles_m * d.tiles_n * d.batch;
    L.inl[i] = d;
  }
  L.total_tiles = t;
  if (t == 0) return cudaSuccess;
  return launch_kernel(gemm_dmma_kernel<64, 64>, dim3(t), dim3(K1Cfg<64, 64>::kThreads),
                       (size_t)K1Cfg<64, 64>::kSmem, stream, 1u, L);
}

cudaError_t launch_gemm_small(const GemmDesc& h, cudaStream_t stream) { return launch_gemm_small_n(&h, 1, stream); }

}  // namespace bi
