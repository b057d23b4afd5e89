// K1P: FP64 DMMA GEMM whose left operand is gathered along K straight from
// the peers' memory -- the sharded scheduler's all-gather fused into K1.
//
//   D = [C] + sign * [A_0 | A_1 | ... | A_{s-1}] * B
//
// A_i (M x k_i, leading dimension lda_i) may live on any GPU that has peer
// access to this one (UVA over NVLink: the TMA ring of bi_gemm_tma.cu, one
// tensor map per owner, or -- for unaligned views -- this file's cp.async
// ring reads the peer's HBM directly), so the column slabs of the inverted pivot block, B/C, L and R
// that a global level of the column-sharded schedule needs (distributed.py,
// SURVEY 8e) are never copied into a gathered buffer: each k-tile is fetched
// from its owner while the previous stages are multiplied, so the transfer
// overlaps the math tile by tile.  This replaces the reference's Fox
// broadcast-multiply (engine.py:202-249) across GPUs.
//
// Segment boundaries lie on k-tile (16) boundaries, so every k-tile comes
// from one owner and the k-tile / k-slot sequence -- and with it every
// rounding -- is exactly K1's: the result is bitwise identical to bi_gemm on
// the gathered operand (tested), hence to every rank count.
#include <cstdlib>

#include "bi_gemm_core.cuh"

namespace bi {

bool launch_gemm_kseg_tma(const GemmDesc& d, int nseg, const double* const* a, const int64_t* lda,
                          const int64_t* kseg, int grid_cap, cudaStream_t stream, cudaError_t* err);

namespace {

bool use_tma_feeder() {
  static const int v = [] {
    const char* e = getenv("BI_GEMM_TMA");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

constexpr int kPM = 128, kPN = 64;                   // CTA tile, 8 warps of 32 x 32
constexpr int kPThreads = (kPM / 32) * (kPN / 32) * 32;
constexpr int kPStages = 4;
constexpr int kPStageA = kPM * kBK * 8;              // 16 KB
constexpr int kPStage = kPStageA + kBK * kPN * 8;    // + 8 KB
constexpr int kPSmem = kPStages * kPStage + 1024;

struct KSegLaunch {
  GemmDesc d;                // B, C, D, ld*, M, N, K, neg; A unused
  const double* a[kMaxKSeg];
  int64_t lda[kMaxKSeg];
  int kt0[kMaxKSeg];         // first k-tile of each segment
  int nseg;
  int tiles_n, total_tiles;
};

__device__ __forceinline__ void cp16(uint8_t* smem, const double* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp8(uint8_t* smem, const double* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}

__global__ void __launch_bounds__(kPThreads, 2) gemm_kseg_kernel(const __grid_constant__ KSegLaunch L) {
  pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp / (kPN / 32), wn = warp % (kPN / 32), fr = lane >> 2, fc = lane & 3;
  K1Frag f;
  k1_frag_init(f, fr, fc);
  const GemmDesc& d = L.d;
  const int K = d.K, KT = (K + kBK - 1) / kBK;
  bool al16 = (((uintptr_t)d.B) & 15) == 0 && (d.ldb & 1) == 0;
  for (int s = 0; s < L.nseg; ++s) al16 = al16 && (((uintptr_t)L.a[s]) & 15) == 0 && (L.lda[s] & 1) == 0;

  for (int tile = blockIdx.x; tile < L.total_tiles; tile += gridDim.x) {
    const int m0 = (tile / L.tiles_n) * kPM, n0 = (tile % L.tiles_n) * kPN;
    const int mrem = d.M - m0, nrem = d.N - n0;
    const double* __restrict__ B = d.B + n0;
    auto b_chunk = [&](int k, int cc) {
      return kPStageA + (cc >> 3) * kK1BoxB + k * 128 + (((cc & 7) ^ (k & 7)) << 4);
    };
    // one k-tile into a stage; its A columns come from the segment (owner) holding them
    auto load_stage = [&](int stage, int kt) {
      int s = 0;
#pragma unroll 1
      while (s + 1 < L.nseg && L.kt0[s + 1] <= kt) ++s;
      const int64_t lda = L.lda[s];
      const int kloc = (kt - L.kt0[s]) * kBK;  // column of this k-tile inside segment s
      const double* __restrict__ A = L.a[s] + (int64_t)m0 * lda + kloc;
      const int k0 = kt * kBK;
      uint8_t* st = smem + stage * kPStage;
      if (al16) {
#pragma unroll
        for (int i = 0; i < (kPM * kBK / 2) / kPThreads; ++i) {
          const int q = tid + i * kPThreads, row = q >> 3, c = q & 7, kk = k0 + 2 * c;
          int bytes = 0;
          const double* src = L.a[s];
          if (row < mrem && kk < K) {
            bytes = min(2, K - kk) * 8;
            src = A + (int64_t)row * lda + 2 * c;
          }
          cp16(st + row * 128 + ((c ^ (row & 7)) << 4), src, bytes);
        }
#pragma unroll
        for (int i = 0; i < (kBK * kPN / 2) / kPThreads; ++i) {
          const int q = tid + i * kPThreads, k = q / (kPN / 2), cc = q % (kPN / 2), kk = k0 + k;
          int bytes = 0;
          const double* src = d.B;
          if (kk < K && 2 * cc < nrem) {
            bytes = min(2, nrem - 2 * cc) * 8;
            src = B + (int64_t)kk * d.ldb + 2 * cc;
          }
          cp16(st + b_chunk(k, cc), src, bytes);
        }
      } else {
#pragma unroll
        for (int i = 0; i < (kPM * kBK) / kPThreads; ++i) {
          const int e = tid + i * kPThreads, row = e >> 4, kc = e & 15;
          const bool ok = row < mrem && k0 + kc < K;
          cp8(st + k1_a_off(row, kc), ok ? A + (int64_t)row * lda + kc : L.a[s], ok ? 8 : 0);
        }
#pragma unroll
        for (int i = 0; i < (kBK * kPN) / kPThreads; ++i) {
          const int e = tid + i * kPThreads, k = e / kPN, n = e % kPN, kk = k0 + k;
          const bool ok = kk < K && n < nrem;
          cp8(st + b_chunk(k, n >> 1) + ((n & 1) << 3), ok ? B + (int64_t)kk * d.ldb + n : d.B, ok ? 8 : 0);
        }
      }
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int s = 0; s < kPStages - 1; ++s) {
      if (s < KT) load_stage(s, s);
      asm volatile("cp.async.commit_group;\n" ::);
    }
    for (int kt = 0; kt < KT; ++kt) {
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kPStages - 2));
      __syncthreads();
      const int nk = kt + kPStages - 1;
      if (nk < KT) load_stage(nk % kPStages, nk);
      asm volatile("cp.async.commit_group;\n" ::);
      k1_compute<kPStageA>(smem + (kt % kPStages) * kPStage, f, wm, wn, fr, acc);
    }
    k1_epilogue<kPM, kPN>(d, 0, m0, n0, wm, wn, fr, fc, acc);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();  // the next tile's prologue reuses the stage ring
  }
}

}  // namespace

cudaError_t launch_gemm_kseg(const GemmDesc& d, int nseg, const double* const* a, const int64_t* lda,
                             const int64_t* kseg, cudaStream_t stream) {
  static PerDeviceOnce once;
  cudaError_t e = once.run([] {
    cudaError_t r = cudaFuncSetAttribute(gemm_kseg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem);
    if (r == cudaSuccess) r = set_carveout(gemm_kseg_kernel);
    return r;
  });
  if (e != cudaSuccess) return e;
  if (nseg < 1 || nseg > kMaxKSeg) return cudaErrorInvalidValue;
  if (use_tma_feeder()) {  // TMA ring (default); cp.async below for unaligned operands
    cudaError_t te = cudaSuccess;
    if (launch_gemm_kseg_tma(d, nseg, a, lda, kseg, g_gemm_grid_cap, stream, &te)) return te;
  }
  KSegLaunch L{};
  L.d = d;
  L.nseg = nseg;
  int64_t k0 = 0;
  for (int s = 0; s < nseg; ++s) {
    if (k0 % kBK) return cudaErrorInvalidValue;  // segments start on k-tile boundaries
    L.a[s] = a[s];
    L.lda[s] = lda[s];
    L.kt0[s] = (int)(k0 / kBK);
    k0 += kseg[s];
  }
  if (k0 != d.K) return cudaErrorInvalidValue;
  if (d.M <= 0 || d.N <= 0) return cudaSuccess;
  L.tiles_n = (d.N + kPN - 1) / kPN;
  L.total_tiles = ((d.M + kPM - 1) / kPM) * L.tiles_n;
  const int grid = (g_gemm_grid_cap > 0 && 2 * g_gemm_grid_cap < L.total_tiles) ? 2 * g_gemm_grid_cap : L.total_tiles;
  return launch_kernel(gemm_kseg_kernel, dim3(grid), dim3(kPThreads), (size_t)kPSmem, stream, 1u, L);
}

}  // namespace bi
