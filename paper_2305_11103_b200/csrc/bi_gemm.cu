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
#include <mutex>

namespace bi {
namespace {

constexpr int kStages = 4;
constexpr int kThreads = 256;
constexpr int kALd = kBK + 4;  // 20 doubles: A tile stored [m][k]
constexpr int kBLd = kBN + 4;  // 132 doubles: B tile stored [k][n]
constexpr int kAStage = kBM * kALd;
constexpr int kBStage = kBK * kBLd;
constexpr int kSmemBytes = kStages * (kAStage + kBStage) * (int)sizeof(double);

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

__global__ void __launch_bounds__(kThreads, 1) gemm_dmma_kernel(const __grid_constant__ GemmLaunch L) {
  extern __shared__ __align__(128) double smem[];
  double* sA = smem;
  double* sB = smem + kStages * kAStage;

  // ---- locate this CTA's (descriptor, batch item, tile) -------------------
  const int tile = blockIdx.x;
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
  auto load_stage = [&](int stage, int kt) {
    const int k0 = kt * kBK;
    double* as = sA + stage * kAStage;
    double* bs = sB + stage * kBStage;
    if (al16) {
#pragma unroll
      for (int i = 0; i < (kBM * kBK / 2) / kThreads; ++i) {  // A: 128 rows x 8 chunks
        const int q = tid + i * kThreads;
        const int row = q >> 3, cc = q & 7, kk = k0 + 2 * cc;
        int bytes = 0;
        const double* src = A;
        if (row < mrem && kk < K) {
          bytes = min(2, K - kk) * 8;
          src = A + (int64_t)row * lda + kk;
        }
        cp_async16(as + row * kALd + 2 * cc, src, bytes);
      }
#pragma unroll
      for (int i = 0; i < (kBK * kBN / 2) / kThreads; ++i) {  // B: 16 rows x 64 chunks
        const int q = tid + i * kThreads;
        const int row = q >> 6, cc = q & 63, kk = k0 + row;
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
      for (int i = 0; i < (kBM * kBK) / kThreads; ++i) {
        const int q = tid + i * kThreads;
        const int row = q >> 4, kc = q & 15, kk = k0 + kc;
        const bool ok = row < mrem && kk < K;
        cp_async8(as + row * kALd + kc, ok ? A + (int64_t)row * lda + kk : A, ok ? 8 : 0);
      }
#pragma unroll
      for (int i = 0; i < (kBK * kBN) / kThreads; ++i) {
        const int q = tid + i * kThreads;
        const int row = q >> 7, nc = q & 127, kk = k0 + row;
        const bool ok = kk < K && nc < nrem;
        cp_async8(bs + row * kBLd + nc, ok ? B + (int64_t)kk * ldb + nc : B, ok ? 8 : 0);
      }
    }
  };

  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps, 64 x 32 each
  const int fr = lane >> 2, fc = lane & 3;

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int KT = (K + kBK - 1) / kBK;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const int nk = kt + kStages - 1;
      if (nk < KT) load_stage(nk % kStages, nk);
      cp_async_commit();
    }
    const double* as = sA + (kt % kStages) * kAStage + (wm * 64 + fr) * kALd + fc;
    const double* bs = sB + (kt % kStages) * kBStage + fc * kBLd + wn * 32 + fr;
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      double af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = as[i * 8 * kALd + ks * 4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[ks * 4 * kBLd + j * 8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
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
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc[i][j][0] *= sgn;
      acc[i][j][1] *= sgn;
    }
  if (C) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = wm * 64 + i * 8 + fr;
      const int64_t row = m0 + r;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int cl = wn * 32 + j * 8 + 2 * fc;
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
  for (int i = 0; i < 8; ++i) {
    const int r = wm * 64 + i * 8 + fr;
    const int64_t row = m0 + r;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cl = wn * 32 + j * 8 + 2 * fc;
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
    g_attr_err = cudaFuncSetAttribute(gemm_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSmemBytes);
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
  gemm_dmma_kernel<<<total, kThreads, kSmemBytes, stream>>>(L);
  return cudaGetLastError();
}

}  // namespace bi
