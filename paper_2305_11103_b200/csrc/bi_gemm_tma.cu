// K1, TMA variant: D = [C] + sign * A * B with TMA-fed shared memory and an
// mbarrier ring (no CTA-wide barrier in the main loop).
//
// Two ring managements (same tile, layout and summation order):
//   gemm_tma_refill_kernel (default): the warp that releases a stage last
//     refills it with the k-tile kStages ahead -- possibly the next tile's --
//     so refills leave as early as possible and no warp waits for the
//     slowest one;
//   gemm_tma_kernel (BI_GEMM_REFILL=0): thread 0 produces kStages-1 ahead,
//     waiting on per-stage "empty" barriers.
// Measured on the same box (profiles/r01_k1_variants.txt): equal on plain
// GEMMs, +0.9 % on accumulating ones, +0.5 % on the engine's K1 phase; a
// deeper ring (6, 7 stages) did not help.
//
// Tile: 128 x 64 with 8 warps (4-stage ring, 97 KB) and TWO CTAs per SM is
// the default (BI_GEMM_TN=128 selects the 16-warp 128 x 128 CTA): one CTA's
// epilogue and ring refill run under the other CTA's main loop, which the
// single 16-warp CTA cannot do.  Same box: 2048^3 x 8 33.2 -> 34.3 TF/s,
// C += AB 32.9 -> 34.1 (99 % of cuBLAS), 512^3 x 32 27.7 -> 32.6; engine K1
// phase 32.5 -> 33.5 TF/s.
//
// sm_100a has no tcgen05 FP64 kind; the FP64 tensor path is DMMA.8x8x4
// (mma.sync.m8n8k4.f64).  This variant feeds it the Blackwell way: one thread
// issues cp.async.bulk.tensor (TMA) loads of 128-byte-swizzled tiles into a
// 5-stage ring; full/empty mbarriers replace __syncthreads, so the 16 consumer
// warps drift freely inside the ring and the per-thread address arithmetic of
// cp.async disappears from the DMMA issue stream.
//
// Bank conflicts: with SWIZZLE_128B the natural m8n8k4 fragment pattern
// conflicts 2-way.  The four k-slots of DMMA k-step s are therefore mapped to
// the permuted k sets S0={0,3,12,15}, S1={2,1,14,13}, S2={4,7,8,11},
// S3={6,5,10,9} of the 16-wide k-tile (the same permutation on A and B, i.e. a
// reordering of the sum).  For both the A box ([m][k], 128 B rows) and the B
// boxes ([k][16 n], 128 B rows) every half-warp then touches 16 distinct
// 8-byte bank pairs.
//
// Replaces core._mm_acc / multiply / schur_accumulate (core.py:115-192) like
// the cp.async variant in bi_gemm.cu; selected when every operand is 16-byte
// aligned with even leading dimensions and the launch has <= 4 descriptors.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "bi_gemm_core.cuh"

namespace bi {
namespace {

// Ring-stage release by the consumer warps (lane 0 after __syncwarp, which
// orders the warp's shared-memory reads of the stage before it): a
// release/acquire pair around the counter, so every warp's generic-proxy
// reads of the stage happen-before the last warp's async-proxy (TMA) refill
// of it (fence.proxy.async follows in fill()).  Returns true for the last warp.
__device__ __forceinline__ bool release_stage(unsigned* counter, unsigned warps) {
  __threadfence_block();  // release: this warp's reads of the stage
  if (atomicAdd(counter, 1u) != warps - 1) return false;
  __threadfence_block();  // acquire: every other warp's reads
  return true;
}


constexpr int kWarps = kK1Warps;
constexpr int kThreads = kK1Threads;
constexpr int kBoxBBytes = kK1BoxB;
constexpr int kStageA = kK1StageA;
constexpr int kStageBytes = kK1Stage;
template <int S>
constexpr int smem_bytes() { return S * kStageBytes + 1024; }  // + alignment slack

// Up to kTmaInline descriptors ride in the kernel parameters (2 tensor maps +
// the descriptor each: ~3.2 KB for 8; sm_100 allows 32 KB of parameters).
constexpr int kTmaInline = 8;
struct alignas(64) TmaLaunch {
  CUtensorMap ta[kTmaInline];
  CUtensorMap tb[kTmaInline];
  GemmDesc d[kTmaInline];
  int count, total_tiles;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

template <int kStages>
__global__ void __launch_bounds__(kThreads, 1) gemm_tma_kernel(const __grid_constant__ TmaLaunch L) {
  pdl_enter();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int fr = lane >> 2, fc = lane & 3;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  K1Frag f;
  k1_frag_init(f, fr, fc);

  unsigned prod_it = 0;  // producer's k-tile counter (thread 0 only)
  unsigned cons_it = 0;  // consumers' k-tile counter
  auto issue = [&](const K1Tile& tc, int kt) {
    const int stage = prod_it % kStages;
    if (prod_it >= (unsigned)kStages) mbar_wait(&empty[stage], ((prod_it / kStages) - 1) & 1);
    uint8_t* sa = smem + stage * kStageBytes;
    uint8_t* sb = sa + kStageA;
    mbar_expect_tx(&full[stage], kStageBytes);
    tma_load_3d(sa, &L.ta[tc.desc], &full[stage], kt * kBK, tc.m0, tc.bz);
#pragma unroll
    for (int j = 0; j < kBN / 16; ++j)
      tma_load_3d(sb + j * kBoxBBytes, &L.tb[tc.desc], &full[stage], tc.n0 + 16 * j, kt * kBK, tc.bz);
    ++prod_it;
  };

  for (int tile = blockIdx.x; tile < L.total_tiles; tile += gridDim.x) {
    const K1Tile tc = k1_locate(L.d, L.count, tile);
    const GemmDesc& d = L.d[tc.desc];
    const int KT = (d.K + kBK - 1) / kBK;
    if (tid == 0) {
      for (int kt = 0; kt < KT && kt < kStages - 1; ++kt) issue(tc, kt);
    }
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < KT; ++kt) {
      if (tid == 0 && kt + kStages - 1 < KT) issue(tc, kt + kStages - 1);
      const int stage = cons_it % kStages;
      mbar_wait(&full[stage], (cons_it / kStages) & 1);
      k1_compute(smem + stage * kStageBytes, f, wm, wn, fr, acc);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      ++cons_it;
    }

    k1_epilogue(d, tc.bz, tc.m0, tc.n0, wm, wn, fr, fc, acc);
  }
}

// Variant: no producer thread.  Each warp's lane 0 counts itself out of a
// stage after consuming it; the warp that releases a stage last refills it
// with the k-tile kStages ahead in the CTA's sequence (possibly the next
// tile's).  Refills go out the moment a slot frees, nobody blocks on the
// slowest warp, and the next tile's first loads overlap this tile's tail.
// TN = 128: 16 warps, one CTA per SM.  TN = 64: 8 warps on a 128 x 64 tile,
// two CTAs per SM, so one CTA's epilogue runs under the other's main loop.
// Fat = true: 4 warps of 64 x 32 on the 128 x 64 tile (k1_compute_64x32),
// the shape cuBLAS's DGEMM uses on sm_100 (ncu: 128 threads, 220 registers,
// two CTAs per SM); same summation order as the 8-warp tile.
// TM = 64: 64 x 64 tiles of 4 warps (32 x 32), three CTAs per SM -- the
// shape cuBLAS picks for short-K batches (ncu at 256^3 x 64: 128 threads,
// 126 registers, 65.5 KB, grid 1024): twice the tiles of 128 x 64, so the
// small products of the first levels fill more waves.
template <int TN, bool Fat = false, int TM = kBM>
struct RefillCfg {
  static constexpr int kWarpsT = Fat ? 4 : (TM / 32) * (TN / 32);
  static constexpr int kThr = kWarpsT * 32;
  static constexpr int kStageA = TM * kBK * 8;
  static constexpr int kStageB = kBK * TN * 8;
  static constexpr int kStage = kStageA + kStageB;
  static constexpr int kMinBlocks = TM == 64 ? 3 : (TN == 64 ? 2 : 1);
};
template <int kStages, int TN, int TM = kBM>
constexpr int refill_smem() { return kStages * RefillCfg<TN, false, TM>::kStage + 1024; }

template <int kStages, int TN, bool Fat = false, int TM = kBM>
__global__ void __launch_bounds__(RefillCfg<TN, Fat, TM>::kThr, RefillCfg<TN, Fat, TM>::kMinBlocks)
    gemm_tma_refill_kernel(const __grid_constant__ TmaLaunch L) {
  pdl_enter();
  using Cfg = RefillCfg<TN, Fat, TM>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ unsigned released[kStages];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = Fat ? warp >> 1 : warp / (TN / 32), wn = Fat ? warp & 1 : warp % (TN / 32);
  const int fr = lane >> 2, fc = lane & 3;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  K1Frag f;
  k1_frag_init(f, fr, fc);

  // fill `stage` with the k-tile `ahead` positions past k-tile 0 of (tile, tc, KT)
  auto fill = [&](int stage, int tile, K1Tile tc, int KT, int ahead) {
    while (ahead >= KT) {
      ahead -= KT;
      tile += gridDim.x;
      if (tile >= L.total_tiles) return;
      tc = k1_locate<TM, TN>(L.d, L.count, tile);
      KT = (L.d[tc.desc].K + kBK - 1) / kBK;
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic reads before async writes
    uint8_t* sa = smem + stage * Cfg::kStage;
    uint8_t* sb = sa + Cfg::kStageA;
    mbar_expect_tx(&full[stage], Cfg::kStage);
    tma_load_3d(sa, &L.ta[tc.desc], &full[stage], ahead * kBK, tc.m0, tc.bz);
#pragma unroll
    for (int j = 0; j < TN / 16; ++j)
      tma_load_3d(sb + j * kBoxBBytes, &L.tb[tc.desc], &full[stage], tc.n0 + 16 * j, ahead * kBK, tc.bz);
  };
  if (tid == 0 && (int)blockIdx.x < L.total_tiles) {
    const K1Tile t0 = k1_locate<TM, TN>(L.d, L.count, blockIdx.x);
    const int KT0 = (L.d[t0.desc].K + kBK - 1) / kBK;
    for (int s = 0; s < kStages; ++s) fill(s, blockIdx.x, t0, KT0, s);
  }

  unsigned cons_it = 0;
  for (int tile = blockIdx.x; tile < L.total_tiles; tile += gridDim.x) {
    const K1Tile tc = k1_locate<TM, TN>(L.d, L.count, tile);
    const GemmDesc& d = L.d[tc.desc];
    const int KT = (d.K + kBK - 1) / kBK;
    constexpr int H = Fat ? 2 : 1;  // 32-row halves of the warp tile
    double acc[H][4][4][2];
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[h][i][j][0] = acc[h][i][j][1] = 0.0;

    for (int kt = 0; kt < KT; ++kt) {
      const int stage = cons_it % kStages;
      mbar_wait(&full[stage], (cons_it / kStages) & 1);
      if constexpr (Fat) {
        k1_compute_64x32<Cfg::kStageA>(smem + stage * Cfg::kStage, f, wm, wn, fr, acc);
      } else {
        k1_compute<Cfg::kStageA>(smem + stage * Cfg::kStage, f, wm, wn, fr, acc[0]);
      }
      __syncwarp();
      if (lane == 0 && release_stage(&released[stage], Cfg::kWarpsT)) {
        released[stage] = 0;
        fill(stage, tile, tc, KT, kt + kStages);
      }
      ++cons_it;
    }

#pragma unroll
    for (int h = 0; h < H; ++h) k1_epilogue<TM, TN>(d, tc.bz, tc.m0, tc.n0, H * wm + h, wn, fr, fc, acc[h]);
  }
}

// K1P on TMA: the refill ring above with a single descriptor whose A operand
// is K-segmented over up to kMaxKSeg owners (one tensor map each; a map may
// describe a peer GPU's memory -- TMA reads it over NVLink).  Segment
// boundaries lie on k-tiles, so every stage is filled from one owner and the
// summation order is K1's (bitwise equal to bi_gemm on the gathered A).
struct alignas(64) TmaSegLaunch {
  CUtensorMap ta[kMaxKSeg];
  CUtensorMap tb;
  GemmDesc d;
  int kt0[kMaxKSeg];
  int nseg, tiles_n, total_tiles;
};

template <int kStages, int TN>
__global__ void __launch_bounds__(RefillCfg<TN>::kThr, RefillCfg<TN>::kMinBlocks)
    gemm_tma_kseg_kernel(const __grid_constant__ TmaSegLaunch L) {
  pdl_enter();
  using Cfg = RefillCfg<TN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ unsigned released[kStages];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp / (TN / 32), wn = warp % (TN / 32);
  const int fr = lane >> 2, fc = lane & 3;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  K1Frag f;
  k1_frag_init(f, fr, fc);
  const GemmDesc& d = L.d;
  const int KT = (d.K + kBK - 1) / kBK;

  // fill `stage` with k-tile `ahead` of `tile` (or of a later tile of this CTA)
  auto fill = [&](int stage, int tile, int ahead) {
    tile += (ahead / KT) * gridDim.x;
    ahead %= KT;
    if (tile >= L.total_tiles) return;
    int s = 0;
    while (s + 1 < L.nseg && L.kt0[s + 1] <= ahead) ++s;
    const int m0 = (tile / L.tiles_n) * kBM, n0 = (tile % L.tiles_n) * TN;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic reads before async writes
    uint8_t* sa = smem + stage * Cfg::kStage;
    uint8_t* sb = sa + kStageA;
    mbar_expect_tx(&full[stage], Cfg::kStage);
    tma_load_3d(sa, &L.ta[s], &full[stage], (ahead - L.kt0[s]) * kBK, m0, 0);
#pragma unroll
    for (int j = 0; j < TN / 16; ++j) tma_load_3d(sb + j * kBoxBBytes, &L.tb, &full[stage], n0 + 16 * j, ahead * kBK, 0);
  };
  if (tid == 0 && (int)blockIdx.x < L.total_tiles)
    for (int s = 0; s < kStages; ++s) fill(s, blockIdx.x, s);

  unsigned cons_it = 0;
  for (int tile = blockIdx.x; tile < L.total_tiles; tile += gridDim.x) {
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < KT; ++kt) {
      const int stage = cons_it % kStages;
      mbar_wait(&full[stage], (cons_it / kStages) & 1);
      k1_compute<kStageA>(smem + stage * Cfg::kStage, f, wm, wn, fr, acc);
      __syncwarp();
      if (lane == 0 && release_stage(&released[stage], Cfg::kWarpsT)) {
        released[stage] = 0;
        fill(stage, tile, kt + kStages);
      }
      ++cons_it;
    }
    k1_epilogue<kBM, TN>(d, 0, (tile / L.tiles_n) * kBM, (tile % L.tiles_n) * TN, wm, wn, fr, fc, acc);
  }
}

// K1P with TMA multicast across a thread-block cluster of CS CTAs that share
// one A row block (consecutive 64-column tiles): the cluster's leader loads
// the A k-tile once and multicasts it into every CTA of the cluster, so each A
// element -- a peer's slab, read over NVLink -- is fetched once per cluster
// instead of once per column tile (remote reads are not cached in the reading
// GPU's L2; at the K1 rate one column tile per A fetch needs ~2 TB/s, with
// CS = 4 about 0.5 TB/s, under one NVLink 5 direction).  A stage is refilled
// only when every CTA of the cluster released it (cluster-wide `empty`
// barriers, below).  Same stage layout, k order and epilogue as K1: bitwise
// equal.  Measured on one B200 (local segments): 30.5 / 29.4 / 26.7 TF/s at
// CS = 2 / 4 / 8 against 33.4 without a cluster (per-CTA slices + all-to-all
// empty arrives had given 28.6 / 25.5 / 17.9; profiles/r01_kseg_fused_gather.txt).
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, unsigned cta) {
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                               unsigned short mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

// Leader-issued A: CTA rank 0 multicasts the whole 128-row A k-tile to the
// cluster once every CTA released the stage (one remote arrive per CTA on the
// leader's `empty` barrier; the leader's warps poll it, in order, before each
// k-step and while spinning on a `full` barrier -- no warp blocks on the
// cluster).  Each CTA refills its own B boxes the moment its own warps
// released the stage.  Iteration u of a CTA is stage u % kStages of tile
// cid + (u / KT) * ncl, k-tile u % KT.
template <int kStages, int CS>
__global__ void __launch_bounds__(RefillCfg<64>::kThr, RefillCfg<64>::kMinBlocks)
    gemm_tma_kseg_mc_kernel(const __grid_constant__ TmaSegLaunch L) {
  pdl_enter();
  constexpr int TN = 64;
  using Cfg = RefillCfg<TN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ unsigned released[kStages];
  __shared__ unsigned next_fill;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp / (TN / 32), wn = warp % (TN / 32);
  const int fr = lane >> 2, fc = lane & 3;
  const unsigned crank = cluster_ctarank();
  const bool leader = crank == 0;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CS);
      released[s] = 0;
    }
    next_fill = kStages;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  cluster_sync_all();  // every CTA's barriers exist before any remote arrive or multicast

  K1Frag f;
  k1_frag_init(f, fr, fc);
  const GemmDesc& d = L.d;
  const int KT = (d.K + kBK - 1) / kBK;
  const int groups_n = (L.tiles_n + CS - 1) / CS;
  const int total_ct = ((d.M + kBM - 1) / kBM) * groups_n;
  const int cid = blockIdx.x / CS, ncl = gridDim.x / CS;
  const unsigned iters = cid < total_ct ? (unsigned)((total_ct - cid + ncl - 1) / ncl) * (unsigned)KT : 0u;
  const unsigned short mask = (unsigned short)((1u << CS) - 1);

  auto fill_b = [&](unsigned u) {  // this CTA's B boxes (+ the stage's expected bytes)
    const int stage = u % kStages, ct = cid + (int)(u / KT) * ncl, ahead = u % KT;
    const int n0 = ((ct % groups_n) * CS + (int)crank) * TN;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    uint8_t* sb = smem + stage * Cfg::kStage + kStageA;
    mbar_expect_tx(&full[stage], Cfg::kStage);  // the multicast A k-tile + this CTA's B boxes
#pragma unroll
    for (int j = 0; j < TN / 16; ++j) tma_load_3d(sb + j * kBoxBBytes, &L.tb, &full[stage], n0 + 16 * j, ahead * kBK, 0);
  };
  auto fill_a = [&](unsigned u) {  // leader: the A k-tile into every CTA of the cluster
    const int stage = u % kStages, ct = cid + (int)(u / KT) * ncl, ahead = u % KT;
    int s = 0;
    while (s + 1 < L.nseg && L.kt0[s + 1] <= ahead) ++s;
    tma_load_3d_mc(smem + stage * Cfg::kStage, &L.ta[s], &full[stage], (ahead - L.kt0[s]) * kBK,
                   (ct / groups_n) * kBM, 0, mask);
  };
  auto poll = [&]() {  // leader lane 0s: next A refill once the whole cluster released its stage
    const unsigned u = *reinterpret_cast<volatile unsigned*>(&next_fill);
    if (u < iters && mbar_test(&empty[u % kStages], ((u / kStages) - 1) & 1) && atomicCAS(&next_fill, u, u + 1) == u)
      fill_a(u);
  };
  if (tid == 0)
    for (unsigned u = 0; u < (unsigned)kStages && u < iters; ++u) {
      fill_b(u);
      if (leader) fill_a(u);
    }

  unsigned cons_it = 0;
  for (int ct = cid; ct < total_ct; ct += ncl) {
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < KT; ++kt) {
      const int stage = cons_it % kStages;
      const unsigned par = (cons_it / kStages) & 1;
      if (leader && lane == 0) poll();
      while (!mbar_test(&full[stage], par)) {
        if (leader && lane == 0) poll();
      }
      k1_compute<kStageA>(smem + stage * Cfg::kStage, f, wm, wn, fr, acc);
      __syncwarp();
      if (lane == 0 && release_stage(&released[stage], Cfg::kWarpsT)) {
        released[stage] = 0;
        if (cons_it + kStages < iters) {  // a refill follows (same test in every CTA)
          mbar_arrive_remote(&empty[stage], 0);
          fill_b(cons_it + kStages);
          if (leader) poll();
        }
      }
      ++cons_it;
    }
    const int m0 = (ct / groups_n) * kBM, n0 = ((ct % groups_n) * CS + (int)crank) * TN;
    k1_epilogue<kBM, TN>(d, 0, m0, n0, wm, wn, fr, fc, acc);  // n0 >= N (cluster padding): stores nothing
  }
  cluster_sync_all();  // no CTA exits while a peer may still arrive on its barriers
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_tma_once;
cudaError_t g_tma_err = cudaSuccess;

cudaError_t tma_init() {
  std::call_once(g_tma_once, [] {  // the driver entry point: once per process
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) {
      g_tma_err = e != cudaSuccess ? e : cudaErrorNotSupported;
      return;
    }
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (g_tma_err != cudaSuccess) return g_tma_err;
  static PerDeviceOnce attrs;  // kernel attributes: once per device
  return attrs.run([] {
    cudaError_t e =
        cudaFuncSetAttribute(gemm_tma_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<5>());
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_tma_refill_kernel<5, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               refill_smem<5, 128>());
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_tma_refill_kernel<4, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               refill_smem<4, 64>());
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_tma_refill_kernel<4, 64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               refill_smem<4, 64>());
    if (e == cudaSuccess) e = set_carveout(gemm_tma_refill_kernel<4, 64, true>);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_tma_refill_kernel<4, 64, false, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               refill_smem<4, 64, 64>());
    if (e == cudaSuccess) e = set_carveout(gemm_tma_refill_kernel<4, 64, false, 64>);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_tma_kseg_kernel<4, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               refill_smem<4, 64>());
    if (e == cudaSuccess) e = set_carveout(gemm_tma_kseg_kernel<4, 64>);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_tma_kseg_mc_kernel<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               refill_smem<4, 64>());
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_tma_kseg_mc_kernel<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               refill_smem<4, 64>());
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_tma_kseg_mc_kernel<4, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               refill_smem<4, 64>());
    if (e == cudaSuccess) e = set_carveout(gemm_tma_kernel<5>);
    if (e == cudaSuccess) e = set_carveout(gemm_tma_refill_kernel<5, 128>);
    if (e == cudaSuccess) e = set_carveout(gemm_tma_refill_kernel<4, 64>);
    return e;
  });
}

bool encode_3d(CUtensorMap* map, const double* base, uint64_t inner, uint64_t outer, uint64_t batch, int64_t ld,
               int64_t bstride, uint32_t box_inner, uint32_t box_outer) {
  cuuint64_t dims[3] = {inner, outer, batch};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)(batch > 1 ? bstride : ld * (int64_t)outer) * 8};
  cuuint32_t box[3] = {box_inner, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

// K1P on TMA; false when the operands do not qualify (16-byte aligned bases,
// even leading dimensions) and the caller takes the cp.async K1P kernel.
bool launch_gemm_kseg_tma(const GemmDesc& d, int nseg, const double* const* a, const int64_t* lda,
                          const int64_t* kseg, int grid_cap, cudaStream_t stream, cudaError_t* err) {
  *err = cudaSuccess;
  if (nseg < 1 || nseg > kMaxKSeg || d.K <= 0 || tma_init() != cudaSuccess) return false;
  if ((((uintptr_t)d.B) & 15) || (d.ldb & 1)) return false;
  // BI_KSEG_CLUSTER: CTAs per cluster sharing A by TMA multicast (1: no cluster,
  // default -- fastest on one GPU: 33.4 / 30.5 / 29.4 / 26.7 TF/s for 1 / 2 / 4 / 8
  // at 8192 x 4096 x 8192; 2, 4, 8 cut the peer reads per A element by that factor)
  static const int cs = [] {
    const char* e = getenv("BI_KSEG_CLUSTER");
    const int v = e ? atoi(e) : 1;
    return (v == 2 || v == 4 || v == 8) ? v : 1;
  }();
  TmaSegLaunch L;
  std::memset(&L, 0, sizeof(L));
  int64_t k0 = 0;
  int used = 0;
  for (int s = 0; s < nseg; ++s) {
    if (kseg[s] == 0) continue;  // empty segments own no k-tile
    if ((((uintptr_t)a[s]) & 15) || (lda[s] & 1) || k0 % kBK) return false;
    if (!encode_3d(&L.ta[used], a[s], (uint64_t)kseg[s], (uint64_t)d.M, 1, lda[s], 0, kBK, kBM)) return false;
    L.kt0[used++] = (int)(k0 / kBK);
    k0 += kseg[s];
  }
  if (!encode_3d(&L.tb, d.B, (uint64_t)d.N, (uint64_t)d.K, 1, d.ldb, 0, 16, kBK)) return false;
  L.d = d;
  L.nseg = used;
  L.tiles_n = (d.N + 63) / 64;
  L.total_tiles = ((d.M + kBM - 1) / kBM) * L.tiles_n;
  if (d.M <= 0 || d.N <= 0) return true;
  const int cap2 = grid_cap > 0 ? 2 * grid_cap : 0;
  if (cs > 1) {
    const int groups = ((d.M + kBM - 1) / kBM) * ((L.tiles_n + cs - 1) / cs);
    const int clusters = (cap2 > 0 && cap2 / cs < groups) ? std::max(1, cap2 / cs) : groups;
    auto k = cs == 2 ? gemm_tma_kseg_mc_kernel<4, 2> : cs == 8 ? gemm_tma_kseg_mc_kernel<4, 8> : gemm_tma_kseg_mc_kernel<4, 4>;
    *err = launch_kernel(k, dim3(clusters * cs), dim3(RefillCfg<64>::kThr), (size_t)refill_smem<4, 64>(), stream,
                         (unsigned)cs, L);
    return true;
  }
  const int grid = (cap2 > 0 && cap2 < L.total_tiles) ? cap2 : L.total_tiles;
  *err = launch_kernel(gemm_tma_kseg_kernel<4, 64>, dim3(grid), dim3(RefillCfg<64>::kThr),
                       (size_t)refill_smem<4, 64>(), stream, 1u, L);
  return true;
}

// Returns true when the launch was issued with the TMA kernel; false when the
// descriptors do not qualify (caller falls back to the cp.async kernel).
bool launch_gemm_tma(const GemmDesc* h, int count, int grid_cap, cudaStream_t stream, cudaError_t* err) {
  *err = cudaSuccess;
  if (count <= 0 || count > kTmaInline) return false;
  if (tma_init() != cudaSuccess) return false;
  TmaLaunch L;
  std::memset(&L, 0, sizeof(L));
  L.count = count;
  int total = 0;
  for (int i = 0; i < count; ++i) {
    const GemmDesc& d = h[i];
    const bool ok = (((uintptr_t)d.A | (uintptr_t)d.B) & 15) == 0 && ((d.lda | d.ldb) & 1) == 0 &&
                    (d.batch <= 1 || ((d.sA | d.sB) & 1) == 0) && d.sA >= 0 && d.sB >= 0 && d.K > 0;
    if (!ok) return false;
    const uint64_t batch = d.batch > 0 ? (uint64_t)d.batch : 1;
    if (!encode_3d(&L.ta[i], d.A, (uint64_t)d.K, (uint64_t)d.M, batch, d.lda, d.sA, kBK, kBM)) return false;
    if (!encode_3d(&L.tb[i], d.B, (uint64_t)d.N, (uint64_t)d.K, batch, d.ldb, d.sB, 16, kBK)) return false;
    L.d[i] = d;
    total = d.tile_begin + ((d.M <= 0 || d.N <= 0 || d.batch <= 0) ? 0 : d.tiles_m * d.tiles_n * d.batch);
  }
  L.total_tiles = total;
  if (total == 0) return true;
  const int grid = (grid_cap > 0 && grid_cap < total) ? grid_cap : total;
  static const int refill = [] {
    const char* e = getenv("BI_GEMM_REFILL");
    return e ? atoi(e) : 1;
  }();
  static const int tn = [] {  // BI_GEMM_TN: 64 (8 warps, 2 CTAs/SM; default) or 128 (16 warps, 1 CTA/SM)
    const char* e = getenv("BI_GEMM_TN");
    return (e && atoi(e) == 128) ? 128 : 64;
  }();
  // BI_GEMM_TM: 128 (default) or 64; BI_GEMM_TM=0 = 64 when every descriptor
  // has K < BI_GEMM_TM64_K (512) and the 128 x 64 tiling has fewer than
  // BI_GEMM_TM64_TILES (1200, ~4 waves of 296) tiles.  64 x 64 wins alone on
  // short-K batches (256^3 x 64: 26.6 -> 28.0 TF/s; K3's 8-leaf K = 128 outer
  // update 14.6 -> 17.1) but not inside the engine (cfg4 394.7 -> 395.4 ms,
  // cfg2 26.9 -> 26.9; profiles/r02_k1_tiles.txt), so it stays opt-in.
  static const int tm_env = [] {
    const char* e = getenv("BI_GEMM_TM");
    return e ? atoi(e) : 128;
  }();
  static const int tm64_k = [] {
    const char* e = getenv("BI_GEMM_TM64_K");
    return e ? atoi(e) : 512;
  }();
  static const int tm64_tiles = [] {
    const char* e = getenv("BI_GEMM_TM64_TILES");
    return e ? atoi(e) : 1200;
  }();
  int kmax = 0, t128 = 0;
  for (int i = 0; i < count; ++i) {
    const GemmDesc& d = L.d[i];
    kmax = std::max(kmax, d.K);
    if (d.M > 0 && d.N > 0 && d.batch > 0) t128 += ((d.M + kBM - 1) / kBM) * ((d.N + 63) / 64) * d.batch;
  }
  const int tm = tm_env == 64 || tm_env == 128 ? tm_env : (kmax < tm64_k && t128 < tm64_tiles ? 64 : 128);
  if (refill && tn == 64 && tm == 64) {
    int t = 0;
    for (int i = 0; i < count; ++i) {
      GemmDesc& d = L.d[i];
      const bool empty = d.M <= 0 || d.N <= 0 || d.batch <= 0;
      d.tiles_m = empty ? 0 : (d.M + 63) / 64;
      d.tiles_n = empty ? 1 : (d.N + 63) / 64;
      d.tile_begin = t;
      t += empty ? 0 : d.tiles_m * d.tiles_n * d.batch;
      const uint64_t batch = d.batch > 0 ? (uint64_t)d.batch : 1;
      if (!encode_3d(&L.ta[i], d.A, (uint64_t)d.K, (uint64_t)d.M, batch, d.lda, d.sA, kBK, 64)) return false;
    }
    L.total_tiles = t;
    const int cap3 = grid_cap > 0 ? 3 * grid_cap : 0;
    const int grid3 = (cap3 > 0 && cap3 < t) ? cap3 : t;
    *err = launch_kernel(gemm_tma_refill_kernel<4, 64, false, 64>, dim3(grid3),
                         dim3(RefillCfg<64, false, 64>::kThr), (size_t)refill_smem<4, 64, 64>(), stream, 1u, L);
    return true;
  }
  if (refill && tn == 64) {
    // re-tile the descriptors for 128 x 64 tiles
    int t = 0;
    for (int i = 0; i < count; ++i) {
      GemmDesc& d = L.d[i];
      const bool empty = d.M <= 0 || d.N <= 0 || d.batch <= 0;
      d.tiles_m = empty ? 0 : (d.M + kBM - 1) / kBM;
      d.tiles_n = empty ? 1 : (d.N + 63) / 64;
      d.tile_begin = t;
      t += empty ? 0 : d.tiles_m * d.tiles_n * d.batch;
    }
    L.total_tiles = t;
    const int cap2 = grid_cap > 0 ? 2 * grid_cap : 0;
    const int grid2 = (cap2 > 0 && cap2 < t) ? cap2 : t;
    // BI_GEMM_WARPS: 8 = 32 x 32 warp tiles, 4 = 64 x 32 (the cuBLAS shape),
    // unset = 4 when every descriptor has K >= 1024 (see below).  Measured (tools/gemm_sweep.py,
    // profiles/r02_k1_fat_warps.txt): 4 warps win on long k loops (8192^3 34.50 ->
    // 35.41 TF/s, cuBLAS 35.48; 1024^3 x 16 33.93 -> 34.30) and lose on short ones
    // (512^3 x 32 32.8 -> 28.8; K3's K = 128 updates 22.5 -> 18.6), where fewer
    // warps per CTA hide less of each tile's prologue and epilogue.
    static const int warps_env = [] {
      const char* e = getenv("BI_GEMM_WARPS");
      return e ? atoi(e) : 0;
    }();
    // ... and at least BI_GEMM_FAT_TILES (default 1184 = four waves of 2 x 148) tiles:
    // with fewer, an SM often holds ONE 4-warp CTA (one warp per scheduler,
    // which cannot keep the DMMA pipe busy: 34.0 vs 36.98 TF/s in the
    // microbench) -- cfg3's 1000-wide via_d products lost 0.65 ms that way.
    static const int fat_tiles = [] {
      const char* e = getenv("BI_GEMM_FAT_TILES");
      return e ? atoi(e) : 4 * 2 * 148;
    }();
    int kmin = INT32_MAX;
    for (int i = 0; i < count; ++i) kmin = std::min(kmin, L.d[i].K);
    const bool fat = warps_env == 4 || (warps_env != 8 && kmin >= 1024 && t >= fat_tiles);
    if (fat)
      *err = launch_kernel(gemm_tma_refill_kernel<4, 64, true>, dim3(grid2), dim3(RefillCfg<64, true>::kThr),
                           (size_t)refill_smem<4, 64>(), stream, 1u, L);
    else
      *err = launch_kernel(gemm_tma_refill_kernel<4, 64>, dim3(grid2), dim3(RefillCfg<64>::kThr),
                           (size_t)refill_smem<4, 64>(), stream, 1u, L);
    return true;
  }
  if (refill) {
    *err = launch_kernel(gemm_tma_refill_kernel<5, 128>, dim3(grid), dim3(RefillCfg<128>::kThr),
                         (size_t)refill_smem<5, 128>(), stream, 1u, L);
    return true;
  }
  *err = launch_kernel(gemm_tma_kernel<5>, dim3(grid), dim3(kThreads), (size_t)smem_bytes<5>(), stream, 1u, L);
  return true;
}

}  // namespace bi
