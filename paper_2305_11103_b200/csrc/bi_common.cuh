// Shared definitions for the B200 blockwise-inversion library (sm_100a only).
#pragma once

#include <mutex>
#include <vector>

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libblockinv_b200 is built for sm_100a only"
#endif

namespace bi {

// ---------------------------------------------------------------------------
// error plumbing (C-ABI status codes, see include/blockinv_b200.h)
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
const char* get_error();

struct Status {
  int code = 0;
  static Status ok() { return Status{}; }
};

#define BI_CUDA_TRY(expr)                                                          \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ::bi::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));        \
      return 3;                                                                    \
    }                                                                              \
  } while (0)

#define BI_REQUIRE(cond, msg)                                                      \
  do {                                                                             \
    if (!(cond)) {                                                                 \
      ::bi::set_error(msg);                                                        \
      return 2;                                                                    \
    }                                                                              \
  } while (0)

// ---------------------------------------------------------------------------
// K1 descriptors: D = beta*C + sign*A*B, strided batched, optional output
// column remap (the Gauss-Jordan trailing update skips the panel columns).
// ---------------------------------------------------------------------------
struct GemmDesc {
  const double* A;
  const double* B;
  const double* C;  // may be null (beta = 0) or equal to D
  double* D;
  int64_t lda, ldb, ldc, ldd;
  int64_t sA, sB, sC, sD;  // batch strides in elements
  int M, N, K, batch;
  int neg;       // 1: alpha = -1
  int skip_at;   // output column n >= skip_at is stored at n + skip_len
  int skip_len;
  int tiles_m, tiles_n;  // filled by finalize_descs
  int tile_begin;        // prefix over descriptors (filled by finalize_descs)
};

constexpr int kGemmInline = 4;  // descriptors passed by value in kernel params

struct GemmLaunch {
  const GemmDesc* descs;  // device array when count > kGemmInline
  int count;
  int total_tiles;
  GemmDesc inl[kGemmInline];
};

// Tile sizes of the DMMA kernel.
constexpr int kBM = 128, kBN = 128, kBK = 16;

// Fills tiles_m/tiles_n/tile_begin; returns total tiles.
int finalize_descs(GemmDesc* d, int count);
// Launch on `stream`. `d_descs` may be null when count <= kGemmInline.
cudaError_t launch_gemm(const GemmDesc* h_descs, const GemmDesc* d_descs, int count,
                        cudaStream_t stream);
// One descriptor on 64 x 64 tiles (latency path; same summation order).
cudaError_t launch_gemm_small(const GemmDesc& h, cudaStream_t stream);
// K1P (bi_gemm_peer.cu): A gathered along K from up to kMaxKSeg owners (peer memory).
constexpr int kMaxKSeg = 8;
cudaError_t launch_gemm_kseg(const GemmDesc& d, int nseg, const double* const* a, const int64_t* lda,
                             const int64_t* kseg, cudaStream_t stream);

// Run `fn` once per CUDA device and cache its status: kernel attributes
// (dynamic shared memory limits, carveouts, cluster permissions) are per
// device, so a process driving several GPUs must set them on each.
struct PerDeviceOnce {
  std::mutex mu;
  std::vector<int> status;  // -1 unset, else the cudaError_t of the first run
  template <typename F>
  cudaError_t run(F fn) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    if ((int)status.size() <= dev) status.resize(dev + 1, -1);
    if (status[dev] < 0) status[dev] = (int)fn();
    return (cudaError_t)status[dev];
  }
};

// Preferred L1/shared carveout (percent) applied to every kernel of the
// library, from BI_CARVEOUT (default -1 = driver default).
int carveout_percent();
template <typename K>
cudaError_t set_carveout(K kernel) {
  const int c = carveout_percent();
  return c < 0 ? cudaSuccess : cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, c);
}

// ---------------------------------------------------------------------------
// K3 batched pivoted Gauss-Jordan, one group of equal-order blocks.
// Blocks are addressed either by pointer arrays (device) or base + stride.
// ---------------------------------------------------------------------------
struct InvGroup {
  int n;      // block order
  int count;  // number of blocks
  const double* src_base;
  int64_t src_stride, ld_src;
  const double* const* src_ptrs;  // optional device array [count]
  const int64_t* src_lds;         // optional device array [count]
  double* dst_base;
  int64_t dst_stride, ld_dst;
  double* const* dst_ptrs;  // optional
  const int64_t* dst_lds;   // optional
  // scratch (device), laid out by inv_group_layout
  double* W;        // count * n * ldw
  int64_t ldw;
  double* tmp;      // count * 128 * ldw  (sub-panel pivot rows: the inner updates' B)
  double* tmpo;     // count * 128 * ldw  (outer-panel pivot rows: the outer updates' B)
  int* perm;        // count * n
  int* flags;       // count * n
  unsigned long long* maxabs;  // count (bit pattern of max|.|)
  int* info;        // count (device; caller-visible)
  // blocks above 8192 (pivot-A recursion with K3 leaves, launch_inv_group):
  // host mirrors of pointer tables (required with src_ptrs / dst_ptrs) and scratch
  const double* const* h_src_ptrs;
  const int64_t* h_src_lds;
  double* const* h_dst_ptrs;
  const int64_t* h_dst_lds;
  double* big_tmp;         // (n - n/2)^2 doubles
  void* big_leaf_scratch;  // K3 scratch for one leaf
  int* big_info;           // leaf status slots
};
// Largest order the K3 panel kernels take directly (one cluster of 16 x 512 rows).
constexpr int kInvMaxDirect = 8192;

int64_t inv_group_scratch_bytes(int n, int count);
// Assign scratch pointers from `base` (needs inv_group_scratch_bytes bytes).
void inv_group_layout(InvGroup& g, void* base);
// Kernel launches (total incl. K1 updates) and K1 launches of one group.
void inv_group_launch_counts(const InvGroup& g, int64_t* kernels, int64_t* gemms);
// Full inversion of the group on `stream`: init, load, panels + updates, store.
cudaError_t launch_inv_group(const InvGroup& g, cudaStream_t stream);
cudaError_t inv_init_attributes_public();
// Destroy K3's helper streams/events (the optional lookahead path); safe to call anytime.
cudaError_t inv_release_helpers();

// ---------------------------------------------------------------------------
// K4 residual
// ---------------------------------------------------------------------------
cudaError_t launch_residual(int64_t n, int batch, const double* a, int64_t lda, int64_t sa,
                            const double* x, int64_t ldx, int64_t sx, double* out,
                            double* scratch, cudaStream_t stream);

// Launch priority applied to every kernel the calling thread launches
// (cudaLaunchAttributePriority; 0 = default).  The engine raises it around
// the latency-bound leaf inversions so their CTAs win freed SMs from the
// throughput-bound GEMMs of the other lane.
extern thread_local int g_launch_priority;
// Programmatic dependent launch for the calling thread's launches
// (cudaLaunchAttributeProgrammaticStreamSerialization; 0 = off).  Set around
// the K3 chain: each kernel's CTAs may be scheduled while its predecessor in
// the stream still runs and wait in pdl_enter() for its completion, so the
// chain's next launch holds its SM slots instead of queueing behind the
// throughput GEMMs of other lanes at every kernel boundary.
extern thread_local int g_launch_pdl;
struct PdlScope {
  int saved;
  explicit PdlScope(int on) : saved(g_launch_pdl) { g_launch_pdl = on; }
  ~PdlScope() { g_launch_pdl = saved; }
};
// First statement of every kernel that can sit in a PDL chain: wait for the
// predecessor grid (a no-op when launched without the attribute).
__device__ __forceinline__ void pdl_enter() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// Let the successor launch: called where a kernel's remaining work is short
// (panel epilogue, K1 tile epilogue), so the successor's CTAs are being
// placed during the tail instead of idling on SM slots for the whole run.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
// Upper bound on K1 grid size (0 = one CTA per tile); K1 is persistent over
// tiles, so a capped launch still covers every tile.
extern thread_local int g_gemm_grid_cap;
struct GemmCapScope {
  int saved;
  explicit GemmCapScope(int c) : saved(g_gemm_grid_cap) { g_gemm_grid_cap = c; }
  ~GemmCapScope() { g_gemm_grid_cap = saved; }
};
struct PriorityScope {
  int saved;
  explicit PriorityScope(int p) : saved(g_launch_priority) { g_launch_priority = p; }
  ~PriorityScope() { g_launch_priority = saved; }
};
int high_launch_priority();

template <typename... KArgs, typename... Args>
cudaError_t launch_kernel_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                             unsigned cluster, bool force_cluster, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[3];
  unsigned na = 0;
  if (cluster > 1 || force_cluster) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (g_launch_priority != 0) {
    attr[na].id = cudaLaunchAttributePriority;
    attr[na].val.priority = g_launch_priority;
    ++na;
  }
  if (g_launch_pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Args&&>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_kernel(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                          unsigned cluster, Args&&... args) {
  return launch_kernel_ex(kernel, grid, block, smem, stream, cluster, false, static_cast<Args&&>(args)...);
}

// Set kernel attributes (dynamic smem, cluster sizes) once per process.
cudaError_t init_attributes();

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

}  // namespace bi
