// extern "C" entry points of libblockinv_b200.so (declared in
// include/blockinv_b200.h) plus the single-level Schur paths, the in-place
// pivot-A recursion and the K4 residual kernel.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/blockinv_b200.h"
#include "bi_common.cuh"

namespace bi {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
const char* get_error() { return g_last_error.c_str(); }

cudaError_t gemm_init_attributes();

// ---------------------------------------------------------------------------
// K4: squared Frobenius norm and max-abs of (P - I) for a column panel
// P = A * X[:, c0:c0+w] computed by K1 into `panel` (n x w, ld w).
// ---------------------------------------------------------------------------
__global__ void residual_reduce_kernel(const double* panel, int64_t n, int64_t w, int64_t c0,
                                       double* out) {
  double s = 0.0, mx = 0.0;
  const int64_t total = n * w;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / w, c = e - r * w;
    double v = panel[e];
    if (r == c0 + c) v -= 1.0;
    s = fma(v, v, s);
    mx = fmax(mx, fabs(v));
  }
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __shared__ double ss[32], sm[32];
  if ((threadIdx.x & 31) == 0) {
    ss[threadIdx.x >> 5] = s;
    sm[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
      s += ss[i];
      mx = fmax(mx, sm[i]);
    }
    atomicAdd(out, s);
    atomicMax(reinterpret_cast<unsigned long long*>(out + 1), (unsigned long long)__double_as_longlong(mx));
  }
}

static int64_t residual_panel_width(int64_t n) {
  const int64_t cap = (int64_t)1 << 27;  // 1 GiB of panel scratch at most
  int64_t w = std::max<int64_t>(128, cap / std::max<int64_t>(n, 1));
  w = std::min(w, n);
  return round_up(w, 4);
}

cudaError_t launch_residual(int64_t n, int batch, const double* a, int64_t lda, int64_t sa, const double* x,
                            int64_t ldx, int64_t sx, double* out, double* scratch, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double) * 2 * batch, stream);
  if (e != cudaSuccess) return e;
  const int64_t w = residual_panel_width(n);
  for (int b = 0; b < batch; ++b) {
    for (int64_t c0 = 0; c0 < n; c0 += w) {
      const int64_t cw = std::min(w, n - c0);
      GemmDesc d{};
      d.A = a + b * sa;
      d.lda = lda;
      d.B = x + b * sx + c0;
      d.ldb = ldx;
      d.C = nullptr;
      d.D = scratch;
      d.ldd = cw;
      d.M = (int)n;
      d.N = (int)cw;
      d.K = (int)n;
      d.batch = 1;
      d.skip_at = INT32_MAX;
      finalize_descs(&d, 1);
      if ((e = launch_gemm(&d, nullptr, 1, stream)) != cudaSuccess) return e;
      residual_reduce_kernel<<<592, 256, 0, stream>>>(scratch, n, cw, c0, out + 2 * b);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

cudaError_t init_attributes() {
  cudaError_t e = gemm_init_attributes();
  if (e == cudaSuccess) e = inv_init_attributes_public();
  return e;
}

static GemmDesc make_gemm(int64_t M, int64_t N, int64_t K, int neg, const double* A, int64_t lda,
                          const double* B, int64_t ldb, const double* C, int64_t ldc, double* D, int64_t ldd) {
  GemmDesc d{};
  d.A = A;
  d.lda = lda;
  d.B = B;
  d.ldb = ldb;
  d.C = C;
  d.ldc = C ? ldc : 0;
  d.D = D;
  d.ldd = ldd;
  d.M = (int)M;
  d.N = (int)N;
  d.K = (int)K;
  d.batch = 1;
  d.neg = neg;
  d.skip_at = INT32_MAX;
  d.skip_len = 0;
  finalize_descs(&d, 1);
  return d;
}

static cudaError_t gemm1(int64_t M, int64_t N, int64_t K, int neg, const double* A, int64_t lda, const double* B,
                         int64_t ldb, const double* C, int64_t ldc, double* D, int64_t ldd, cudaStream_t s) {
  GemmDesc d = make_gemm(M, N, K, neg, A, lda, B, ldb, C, ldc, D, ldd);
  return launch_gemm(&d, nullptr, 1, s);
}

// One K3 inversion of a single n x n block (src -> dst) with its scratch at `scratch`.
static cudaError_t inv1(int64_t n, const double* src, int64_t lds, double* dst, int64_t ldd, void* scratch,
                        int* info, cudaStream_t s) {
  InvGroup g{};
  g.n = (int)n;
  g.count = 1;
  g.src_base = src;
  g.ld_src = lds;
  g.dst_base = dst;
  g.ld_dst = ldd;
  inv_group_layout(g, scratch);
  g.info = info;
  return launch_inv_group(g, s);
}

}  // namespace bi

using namespace bi;

static int64_t a256(int64_t v) { return round_up(v, 256); }

extern "C" int bi_version(void) { return 1; }
extern "C" const char* bi_last_error(void) { return bi::get_error(); }

static std::vector<int> g_init_devices;
static std::mutex g_init_mu;

extern "C" int bi_init(int ndev, const int* dev_ids) {
  BI_REQUIRE(ndev >= 1 && dev_ids, "bi_init needs at least one device id");
  int count = 0, prev = 0;
  BI_CUDA_TRY(cudaGetDeviceCount(&count));
  BI_CUDA_TRY(cudaGetDevice(&prev));
  for (int i = 0; i < ndev; ++i) BI_REQUIRE(dev_ids[i] >= 0 && dev_ids[i] < count, "device id out of range");
  int rc = 0;
  for (int i = 0; i < ndev && rc == 0; ++i) {
    cudaDeviceProp p{};
    cudaError_t e = cudaGetDeviceProperties(&p, dev_ids[i]);
    if (e == cudaSuccess && p.major != 10) {
      set_error("device is not sm_100 (B200): this library is built for sm_100a only");
      rc = 5;
      break;
    }
    if (e == cudaSuccess) e = cudaSetDevice(dev_ids[i]);
    if (e == cudaSuccess) e = init_attributes();
    for (int j = 0; j < ndev && e == cudaSuccess; ++j) {
      if (dev_ids[j] == dev_ids[i]) continue;
      int can = 0;
      e = cudaDeviceCanAccessPeer(&can, dev_ids[i], dev_ids[j]);
      if (e == cudaSuccess && can) {
        e = cudaDeviceEnablePeerAccess(dev_ids[j], 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
          e = cudaSuccess;
        }
      }
    }
    if (e != cudaSuccess) {
      set_error(cudaGetErrorString(e));
      rc = 3;
    }
  }
  cudaSetDevice(prev);
  if (rc == 0) {
    std::lock_guard<std::mutex> lock(g_init_mu);
    for (int i = 0; i < ndev; ++i)
      if (std::find(g_init_devices.begin(), g_init_devices.end(), dev_ids[i]) == g_init_devices.end())
        g_init_devices.push_back(dev_ids[i]);
  }
  return rc;
}

extern "C" int bi_finalize(void) {
  std::vector<int> devs;
  {
    std::lock_guard<std::mutex> lock(g_init_mu);
    devs.swap(g_init_devices);
  }
  int prev = 0;
  BI_CUDA_TRY(cudaGetDevice(&prev));
  for (int d : devs) {
    BI_CUDA_TRY(cudaSetDevice(d));
    BI_CUDA_TRY(cudaDeviceSynchronize());
  }
  BI_CUDA_TRY(bi::inv_release_helpers());
  BI_CUDA_TRY(cudaSetDevice(prev));
  return 0;
}

extern "C" int bi_gemm(int64_t m, int64_t n, int64_t k, int alpha_sign, const double* a, int64_t lda,
                       int64_t stride_a, const double* b, int64_t ldb, int64_t stride_b, const double* cin,
                       int64_t ldc, int64_t stride_c, double* d, int64_t ldd, int64_t stride_d, int batch,
                       void* stream) {
  BI_REQUIRE(m >= 0 && n >= 0 && k >= 0 && batch >= 0, "negative dimension");
  BI_REQUIRE(m < INT32_MAX && n < INT32_MAX && k < INT32_MAX, "dimension too large");
  BI_REQUIRE(alpha_sign == 1 || alpha_sign == -1, "alpha_sign must be +1 or -1");
  if (m == 0 || n == 0 || batch == 0) return 0;
  BI_REQUIRE(d != nullptr && (k == 0 || (a && b)), "null operand");
  BI_REQUIRE(lda >= k && ldb >= n && ldd >= n && (!cin || ldc >= n), "leading dimension too small");
  BI_CUDA_TRY(init_attributes());
  GemmDesc g = make_gemm(m, n, k, alpha_sign < 0 ? 1 : 0, a, lda, b, ldb, cin, ldc, d, ldd);
  g.batch = batch;
  g.sA = stride_a;
  g.sB = stride_b;
  g.sC = stride_c;
  g.sD = stride_d;
  finalize_descs(&g, 1);
  BI_CUDA_TRY(launch_gemm(&g, nullptr, 1, static_cast<cudaStream_t>(stream)));
  return 0;
}

extern "C" int bi_gemm_kseg(int64_t m, int64_t n, int alpha_sign, int nseg, const double* const* a_segs,
                            const int64_t* lda_segs, const int64_t* k_segs, const double* b, int64_t ldb,
                            const double* cin, int64_t ldc, double* d, int64_t ldd, void* stream) {
  BI_REQUIRE(m >= 0 && n >= 0 && m < INT32_MAX && n < INT32_MAX, "bad dimension");
  BI_REQUIRE(alpha_sign == 1 || alpha_sign == -1, "alpha_sign must be +1 or -1");
  BI_REQUIRE(nseg >= 1 && nseg <= kMaxKSeg, "nseg must be in [1, 8]");
  BI_REQUIRE(a_segs && lda_segs && k_segs, "null segment table");
  int64_t k = 0;
  for (int s = 0; s < nseg; ++s) {
    BI_REQUIRE(k_segs[s] >= 0, "negative segment width");
    BI_REQUIRE(k % kBK == 0, "every segment but the last must be a multiple of 16 wide");
    BI_REQUIRE(k_segs[s] == 0 || (a_segs[s] && lda_segs[s] >= k_segs[s]), "bad segment operand");
    k += k_segs[s];
  }
  BI_REQUIRE(k < INT32_MAX, "dimension too large");
  if (m == 0 || n == 0) return 0;
  BI_REQUIRE(d != nullptr && (k == 0 || b), "null operand");
  BI_REQUIRE(ldb >= n && ldd >= n && (!cin || ldc >= n), "leading dimension too small");
  BI_CUDA_TRY(init_attributes());
  GemmDesc g = make_gemm(m, n, k, alpha_sign < 0 ? 1 : 0, nullptr, 0, b, ldb, cin, ldc, d, ldd);
  if (k == 0) {  // D = [C]: route through K1 (zero k-tiles, same epilogue)
    g.A = b;
    finalize_descs(&g, 1);
    BI_CUDA_TRY(launch_gemm(&g, nullptr, 1, static_cast<cudaStream_t>(stream)));
    return 0;
  }
  BI_CUDA_TRY(launch_gemm_kseg(g, nseg, a_segs, lda_segs, k_segs, static_cast<cudaStream_t>(stream)));
  return 0;
}

extern "C" int64_t bi_gemm_grouped_workspace_bytes(int count) {
  if (count < 0) return -1;
  return count <= kGemmInline ? 0 : a256((int64_t)count * (int64_t)sizeof(GemmDesc));
}

extern "C" int bi_gemm_grouped(int count, const bi_gemm_desc* descs, void* workspace, int64_t workspace_bytes,
                               void* stream) {
  BI_REQUIRE(count >= 0, "negative count");
  if (count == 0) return 0;
  BI_REQUIRE(descs != nullptr, "null descriptor array");
  BI_REQUIRE(count <= kGemmInline || (workspace && workspace_bytes >= bi_gemm_grouped_workspace_bytes(count)),
             "workspace too small for the descriptor table");
  std::vector<GemmDesc> gs;
  gs.reserve(count);
  for (int i = 0; i < count; ++i) {
    const bi_gemm_desc& x = descs[i];
    BI_REQUIRE(x.m >= 0 && x.n >= 0 && x.k >= 0 && x.batch >= 0, "negative dimension");
    BI_REQUIRE(x.m < INT32_MAX && x.n < INT32_MAX && x.k < INT32_MAX, "dimension too large");
    BI_REQUIRE(x.alpha_sign == 1 || x.alpha_sign == -1, "alpha_sign must be +1 or -1");
    BI_REQUIRE(x.d != nullptr && (x.k == 0 || (x.a && x.b)), "null operand");
    BI_REQUIRE(x.lda >= x.k && x.ldb >= x.n && x.ldd >= x.n && (!x.cin || x.ldc >= x.n),
               "leading dimension too small");
    GemmDesc g = make_gemm(x.m, x.n, x.k, x.alpha_sign < 0 ? 1 : 0, x.a, x.lda, x.b, x.ldb, x.cin, x.ldc, x.d,
                           x.ldd);
    g.batch = x.batch;
    g.sA = x.stride_a;
    g.sB = x.stride_b;
    g.sC = x.stride_c;
    g.sD = x.stride_d;
    gs.push_back(g);
  }
  BI_CUDA_TRY(init_attributes());
  finalize_descs(gs.data(), count);
  GemmDesc* dd = nullptr;
  if (count > kGemmInline) {
    dd = static_cast<GemmDesc*>(workspace);
    BI_CUDA_TRY(cudaMemcpyAsync(dd, gs.data(), gs.size() * sizeof(GemmDesc), cudaMemcpyHostToDevice,
                                static_cast<cudaStream_t>(stream)));
  }
  BI_CUDA_TRY(launch_gemm(gs.data(), dd, count, static_cast<cudaStream_t>(stream)));
  return 0;
}

extern "C" int64_t bi_inv_workspace_bytes(int count, int64_t n) {
  if (count < 0 || n < 0) return -1;
  return a256(inv_group_scratch_bytes((int)n, count));
}

extern "C" int bi_inv_batched(int count, int64_t n, const double* in, int64_t ld_in, int64_t stride_in,
                              double* out, int64_t ld_out, int64_t stride_out, int* info, void* workspace,
                              int64_t workspace_bytes, void* stream) {
  BI_REQUIRE(count >= 0 && n >= 0, "negative dimension");
  if (count == 0 || n == 0) return 0;
  BI_REQUIRE(n <= INT32_MAX / 2, "block order too large");
  BI_REQUIRE(in && out && info && workspace, "null argument");
  BI_REQUIRE(ld_in >= n && ld_out >= n, "leading dimension too small");
  BI_REQUIRE(workspace_bytes >= bi_inv_workspace_bytes(count, n), "workspace too small");
  BI_CUDA_TRY(init_attributes());
  InvGroup g{};
  g.n = (int)n;
  g.count = count;
  g.src_base = in;
  g.src_stride = stride_in;
  g.ld_src = ld_in;
  g.dst_base = out;
  g.dst_stride = stride_out;
  g.ld_dst = ld_out;
  inv_group_layout(g, workspace);
  g.info = info;
  BI_CUDA_TRY(launch_inv_group(g, static_cast<cudaStream_t>(stream)));
  return 0;
}

extern "C" int bi_inv_batched_ptrs(int count, int64_t n, const double* const* in, const int64_t* ld_in,
                                   double* const* out, const int64_t* ld_out, int* info, void* workspace,
                                   int64_t workspace_bytes, void* stream) {
  BI_REQUIRE(count >= 0 && n >= 0, "negative dimension");
  if (count == 0 || n == 0) return 0;
  BI_REQUIRE(n <= INT32_MAX / 2, "block order too large");
  BI_REQUIRE(in && ld_in && out && ld_out && info && workspace, "null argument");
  BI_REQUIRE(workspace_bytes >= bi_inv_workspace_bytes(count, n), "workspace too small");
  BI_CUDA_TRY(init_attributes());
  InvGroup g{};
  g.n = (int)n;
  g.count = count;
  g.src_ptrs = in;
  g.src_lds = ld_in;
  g.dst_ptrs = out;
  g.dst_lds = ld_out;
  inv_group_layout(g, workspace);
  g.info = info;
  std::vector<const double*> hs(count);
  std::vector<double*> hd(count);
  std::vector<int64_t> hsl(count), hdl(count);
  if (n > kInvMaxDirect) {  // the recursion addresses the blocks from the host: mirror the tables
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    BI_CUDA_TRY(cudaMemcpyAsync(hs.data(), in, count * sizeof(void*), cudaMemcpyDeviceToHost, st));
    BI_CUDA_TRY(cudaMemcpyAsync(hd.data(), out, count * sizeof(void*), cudaMemcpyDeviceToHost, st));
    BI_CUDA_TRY(cudaMemcpyAsync(hsl.data(), ld_in, count * 8, cudaMemcpyDeviceToHost, st));
    BI_CUDA_TRY(cudaMemcpyAsync(hdl.data(), ld_out, count * 8, cudaMemcpyDeviceToHost, st));
    BI_CUDA_TRY(cudaStreamSynchronize(st));
    g.h_src_ptrs = hs.data();
    g.h_src_lds = hsl.data();
    g.h_dst_ptrs = hd.data();
    g.h_dst_lds = hdl.data();
  }
  BI_CUDA_TRY(launch_inv_group(g, static_cast<cudaStream_t>(stream)));
  return 0;
}

// ---------------------------------------------------------------------------
// Single-level Schur paths (schur.py:114-164, 219-259)
// workspace: [Pinv p*p][Qinv q*q][X q*p][Y p*q][S max(p,q)^2][info 8 ints][K3 scratch]
// ---------------------------------------------------------------------------
extern "C" int64_t bi_schur2x2_workspace_bytes(int64_t n, int64_t p) {
  if (p < 1 || p >= n) return -1;
  const int64_t q = n - p, mx = std::max(p, q);
  return a256(p * p * 8) + a256(q * q * 8) + a256(q * p * 8) + a256(p * q * 8) + a256(mx * mx * 8) + 256 +
         a256(inv_group_scratch_bytes((int)mx, 1));
}

extern "C" int bi_schur2x2(int pivot, int64_t n, int64_t p, const double* m, int64_t ldm, double* out,
                           int64_t ldo, void* workspace, int64_t workspace_bytes, int* fail_block, void* stream) {
  BI_REQUIRE(pivot == 'A' || pivot == 'D' || pivot == 'X' || pivot == 'B' || pivot == 'C' || pivot == 'Y',
             "pivot must be 'A', 'D', 'X', 'B', 'C' or 'Y'");
  BI_REQUIRE(p >= 1 && p < n, "split outside 1..n-1");
  BI_REQUIRE(m && out && workspace, "null argument");
  BI_REQUIRE(ldm >= n && ldo >= n, "leading dimension too small");
  BI_REQUIRE(workspace_bytes >= bi_schur2x2_workspace_bytes(n, p), "workspace too small");
  BI_CUDA_TRY(init_attributes());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t q = n - p, mx = std::max(p, q);
  char* w = static_cast<char*>(workspace);
  double* Pinv = reinterpret_cast<double*>(w);
  w += a256(p * p * 8);
  double* Qinv = reinterpret_cast<double*>(w);
  w += a256(q * q * 8);
  double* X = reinterpret_cast<double*>(w);  // q x p
  w += a256(q * p * 8);
  double* Y = reinterpret_cast<double*>(w);  // p x q
  w += a256(p * q * 8);
  double* S = reinterpret_cast<double*>(w);  // Schur complement, ld = its order
  w += a256(mx * mx * 8);
  int* info = reinterpret_cast<int*>(w);
  w += 256;
  void* scratch = w;
  BI_CUDA_TRY(cudaMemsetAsync(info, 0, 8 * sizeof(int), s));
  const double* A = m;
  const double* B = m + p;
  const double* C = m + p * ldm;
  const double* D = m + p * ldm + p;
  double* o00 = out;
  double* o01 = out + p;
  double* o10 = out + p * ldo;
  double* o11 = out + p * ldo + p;
  // info slots: 0 = A, 1 = D, 2 = SchurA, 3 = SchurD, 4 = B, 5 = C, 6 = SchurB, 7 = SchurC
  char labels[8] = {'A', 'D', 'a', 'd', 'B', 'C', 'b', 'c'};
  int order[4] = {0, 1, 2, 3};
  // A singular pivot block ends the formula at once (one sync after its
  // inversion), so invert_with_fallback's failed attempts cost one block
  // inversion instead of the whole formula (cfg3's via_a: ~2 ms, not ~17).
  auto early_singular = [&](std::initializer_list<int> slots) -> int {
    int h[8];
    if (cudaMemcpyAsync(h, info, sizeof(h), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return -1;
    for (int slot : slots)
      if (h[slot] != 0) {
        if (fail_block) *fail_block = labels[slot];
        set_error(std::string("singular pivot block ") + labels[slot]);
        return 1;
      }
    return 0;
  };
#define BI_EARLY(...)                                          \
  do {                                                         \
    const int r_ = early_singular({__VA_ARGS__});              \
    BI_REQUIRE(r_ >= 0, "bi_schur2x2: CUDA error reading info"); \
    if (r_) return 1;                                          \
  } while (0)
  // counter-diagonal layout (schur.py:92-101): rows split at p, columns at q = n - p
  const double* cA = m;                 // p x q
  const double* cB = m + q;             // p x p
  const double* cC = m + p * ldm;       // q x q
  const double* cD = m + p * ldm + q;   // q x p
  double* oTL = out;                    // q x p
  double* oTR = out + p;                // q x q
  double* oBL = out + q * ldo;          // p x p
  double* oBR = out + q * ldo + p;      // p x q
  if (pivot == 'B') {
    // schur.py:167-190, S_B = C - D B^-1 A
    BI_CUDA_TRY(inv1(p, cB, ldm, Pinv, p, scratch, info + 4, s));
    BI_EARLY(4);
    BI_CUDA_TRY(gemm1(p, q, p, 1, Pinv, p, cA, ldm, nullptr, 0, Y, q, s));     // Y = -B^-1 A
    BI_CUDA_TRY(gemm1(q, p, p, 0, cD, ldm, Pinv, p, nullptr, 0, X, p, s));     // X = D B^-1
    BI_CUDA_TRY(gemm1(q, q, p, 0, cD, ldm, Y, q, cC, ldm, S, q, s));           // S_B = C + D Y
    BI_CUDA_TRY(inv1(q, S, q, oTR, ldo, scratch, info + 6, s));                // out[:q, p:] = S_B^-1
    BI_CUDA_TRY(gemm1(p, q, q, 0, Y, q, oTR, ldo, nullptr, 0, oBR, ldo, s));   // out[q:, p:] = Y S_B^-1
    BI_CUDA_TRY(gemm1(p, p, q, 1, oBR, ldo, X, p, Pinv, p, oBL, ldo, s));      // out[q:, :p] = B^-1 - . X
    BI_CUDA_TRY(gemm1(q, p, q, 1, oTR, ldo, X, p, nullptr, 0, oTL, ldo, s));   // out[:q, :p] = -S_B^-1 X
    order[0] = 4;
    order[1] = 6;
    order[2] = 4;
    order[3] = 6;
  } else if (pivot == 'C') {
    // schur.py:193-216, S_C = B - A C^-1 D
    BI_CUDA_TRY(inv1(q, cC, ldm, Qinv, q, scratch, info + 5, s));
    BI_EARLY(5);
    BI_CUDA_TRY(gemm1(q, p, q, 1, Qinv, q, cD, ldm, nullptr, 0, X, p, s));     // X = -C^-1 D
    BI_CUDA_TRY(gemm1(p, q, q, 0, cA, ldm, Qinv, q, nullptr, 0, Y, q, s));     // Y = A C^-1
    BI_CUDA_TRY(gemm1(p, p, q, 0, cA, ldm, X, p, cB, ldm, S, p, s));           // S_C = B + A X
    BI_CUDA_TRY(inv1(p, S, p, oBL, ldo, scratch, info + 7, s));                // out[q:, :p] = S_C^-1
    BI_CUDA_TRY(gemm1(q, p, p, 0, X, p, oBL, ldo, nullptr, 0, oTL, ldo, s));   // out[:q, :p] = X S_C^-1
    BI_CUDA_TRY(gemm1(q, q, p, 1, oTL, ldo, Y, q, Qinv, q, oTR, ldo, s));      // out[:q, p:] = C^-1 - . Y
    BI_CUDA_TRY(gemm1(p, q, p, 1, oBL, ldo, Y, q, nullptr, 0, oBR, ldo, s));   // out[q:, p:] = -S_C^-1 Y
    order[0] = 5;
    order[1] = 7;
    order[2] = 5;
    order[3] = 7;
  } else if (pivot == 'Y') {
    // schur.py:262-297 (combined counter-diagonal form)
    BI_CUDA_TRY(inv1(p, cB, ldm, Pinv, p, scratch, info + 4, s));
    BI_CUDA_TRY(inv1(q, cC, ldm, Qinv, q, scratch, info + 5, s));
    BI_EARLY(4, 5);
    BI_CUDA_TRY(gemm1(p, q, p, 1, Pinv, p, cA, ldm, nullptr, 0, Y, q, s));     // Y = -B^-1 A
    BI_CUDA_TRY(gemm1(q, p, q, 1, Qinv, q, cD, ldm, nullptr, 0, X, p, s));     // X = -C^-1 D
    BI_CUDA_TRY(gemm1(q, q, p, 0, cD, ldm, Y, q, cC, ldm, S, q, s));           // S_B = C + D Y
    BI_CUDA_TRY(inv1(q, S, q, oTR, ldo, scratch, info + 6, s));                // out[:q, p:] = S_B^-1
    BI_CUDA_TRY(gemm1(p, p, q, 0, cA, ldm, X, p, cB, ldm, S, p, s));           // S_C = B + A X
    BI_CUDA_TRY(inv1(p, S, p, oBL, ldo, scratch, info + 7, s));                // out[q:, :p] = S_C^-1
    BI_CUDA_TRY(gemm1(q, p, p, 0, X, p, oBL, ldo, nullptr, 0, oTL, ldo, s));   // out[:q, :p] = X S_C^-1
    BI_CUDA_TRY(gemm1(p, q, q, 0, Y, q, oTR, ldo, nullptr, 0, oBR, ldo, s));   // out[q:, p:] = Y S_B^-1
    order[0] = 4;
    order[1] = 5;
    order[2] = 6;
    order[3] = 7;
  } else if (pivot == 'A') {
    // schur.py:114-139
    BI_CUDA_TRY(inv1(p, A, ldm, Pinv, p, scratch, info + 0, s));
    BI_EARLY(0);
    BI_CUDA_TRY(gemm1(p, q, p, 1, Pinv, p, B, ldm, nullptr, 0, Y, q, s));      // Y = -A^-1 B
    BI_CUDA_TRY(gemm1(q, p, p, 0, C, ldm, Pinv, p, nullptr, 0, X, p, s));      // X = C A^-1
    BI_CUDA_TRY(gemm1(q, q, p, 0, C, ldm, Y, q, D, ldm, S, q, s));             // S_A = D + C Y
    BI_CUDA_TRY(inv1(q, S, q, o11, ldo, scratch, info + 2, s));                // out11 = S_A^-1
    BI_CUDA_TRY(gemm1(p, q, q, 0, Y, q, o11, ldo, nullptr, 0, o01, ldo, s));   // out01 = Y S_A^-1
    BI_CUDA_TRY(gemm1(p, p, q, 1, o01, ldo, X, p, Pinv, p, o00, ldo, s));      // out00 = A^-1 - out01 X
    BI_CUDA_TRY(gemm1(q, p, q, 1, o11, ldo, X, p, nullptr, 0, o10, ldo, s));   // out10 = -S_A^-1 X
    order[1] = 2;
    order[2] = 1;
  } else if (pivot == 'D') {
    // schur.py:142-164
    BI_CUDA_TRY(inv1(q, D, ldm, Qinv, q, scratch, info + 1, s));
    BI_EARLY(1);
    BI_CUDA_TRY(gemm1(q, p, q, 1, Qinv, q, C, ldm, nullptr, 0, X, p, s));      // X = -D^-1 C
    BI_CUDA_TRY(gemm1(p, q, q, 0, B, ldm, Qinv, q, nullptr, 0, Y, q, s));      // Y = B D^-1
    BI_CUDA_TRY(gemm1(p, p, q, 0, B, ldm, X, p, A, ldm, S, p, s));             // S_D = A + B X
    BI_CUDA_TRY(inv1(p, S, p, o00, ldo, scratch, info + 3, s));                // out00 = S_D^-1
    BI_CUDA_TRY(gemm1(q, p, p, 0, X, p, o00, ldo, nullptr, 0, o10, ldo, s));   // out10 = X S_D^-1
    BI_CUDA_TRY(gemm1(q, q, p, 1, o10, ldo, Y, q, Qinv, q, o11, ldo, s));      // out11 = D^-1 - out10 Y
    BI_CUDA_TRY(gemm1(p, q, p, 1, o00, ldo, Y, q, nullptr, 0, o01, ldo, s));   // out01 = -S_D^-1 Y
    order[0] = 1;
    order[1] = 3;
    order[2] = 0;
    order[3] = 2;
  } else {
    // schur.py:219-259 (Eq. 7); S_D first, then S_A
    BI_CUDA_TRY(inv1(p, A, ldm, Pinv, p, scratch, info + 0, s));
    BI_CUDA_TRY(inv1(q, D, ldm, Qinv, q, scratch, info + 1, s));
    BI_EARLY(0, 1);
    BI_CUDA_TRY(gemm1(p, q, p, 1, Pinv, p, B, ldm, nullptr, 0, Y, q, s));      // Y = -A^-1 B
    BI_CUDA_TRY(gemm1(q, p, q, 1, Qinv, q, C, ldm, nullptr, 0, X, p, s));      // X = -D^-1 C
    BI_CUDA_TRY(gemm1(p, p, q, 0, B, ldm, X, p, A, ldm, S, p, s));             // S_D = A + B X
    BI_CUDA_TRY(inv1(p, S, p, o00, ldo, scratch, info + 3, s));                // out00 = S_D^-1
    BI_CUDA_TRY(gemm1(q, q, p, 0, C, ldm, Y, q, D, ldm, S, q, s));             // S_A = D + C Y
    BI_CUDA_TRY(inv1(q, S, q, o11, ldo, scratch, info + 2, s));                // out11 = S_A^-1
    BI_CUDA_TRY(gemm1(p, q, q, 0, Y, q, o11, ldo, nullptr, 0, o01, ldo, s));   // out01 = Y S_A^-1
    BI_CUDA_TRY(gemm1(q, p, p, 0, X, p, o00, ldo, nullptr, 0, o10, ldo, s));   // out10 = X S_D^-1
    order[2] = 3;
    order[3] = 2;
  }
#undef BI_EARLY
  int h[8];
  BI_CUDA_TRY(cudaMemcpyAsync(h, info, sizeof(h), cudaMemcpyDeviceToHost, s));
  BI_CUDA_TRY(cudaStreamSynchronize(s));
  if (fail_block) *fail_block = 0;
  for (int i = 0; i < 4; ++i) {
    const int slot = order[i];
    if (h[slot] != 0) {
      if (fail_block) *fail_block = labels[slot];
      set_error(std::string("singular pivot block ") + labels[slot]);
      return 1;
    }
  }
  return 0;
}

// ---------------------------------------------------------------------------
// invertor_inplace_by_a (recursive.py:273-333) with K3 leaves
// ---------------------------------------------------------------------------
namespace {
struct InplaceCtx {
  double* tmp;       // >= (n/2+1)^2 doubles
  void* scratch;     // K3 scratch for order <= leaf
  int* info;         // leaf info slots
  int nleaf = 0, max_leaf = 0;
  std::vector<std::string> paths;
  int64_t leaf;
  cudaStream_t s;
};

cudaError_t inplace_rec(InplaceCtx& c, double* x, int64_t ldx, int64_t n, const std::string& path) {
  cudaError_t e;
  if (n <= c.leaf) {
    if (c.nleaf >= c.max_leaf) return cudaErrorInvalidValue;
    c.paths.push_back(path);
    return inv1(n, x, ldx, x, ldx, c.scratch, c.info + c.nleaf++, c.s);
  }
  const int64_t p = n / 2, q = n - p;
  double* a = x;
  double* b = x + p;
  double* cc = x + p * ldx;
  double* d = x + p * ldx + p;
  if ((e = inplace_rec(c, a, ldx, p, path + "A")) != cudaSuccess) return e;
  // b <- -A^-1 B
  if ((e = gemm1(p, q, p, 1, a, ldx, b, ldx, nullptr, 0, c.tmp, q, c.s)) != cudaSuccess) return e;
  if ((e = cudaMemcpy2DAsync(b, ldx * 8, c.tmp, q * 8, q * 8, p, cudaMemcpyDeviceToDevice, c.s)) != cudaSuccess)
    return e;
  // d <- D + C b  (S_A)
  if ((e = gemm1(q, q, p, 0, cc, ldx, b, ldx, d, ldx, d, ldx, c.s)) != cudaSuccess) return e;
  // c <- -C A^-1
  if ((e = gemm1(q, p, p, 1, cc, ldx, a, ldx, nullptr, 0, c.tmp, p, c.s)) != cudaSuccess) return e;
  if ((e = cudaMemcpy2DAsync(cc, ldx * 8, c.tmp, p * 8, p * 8, q, cudaMemcpyDeviceToDevice, c.s)) != cudaSuccess)
    return e;
  if ((e = inplace_rec(c, d, ldx, q, path + "S")) != cudaSuccess) return e;
  // c <- S_A^-1 c
  if ((e = gemm1(q, p, q, 0, d, ldx, cc, ldx, nullptr, 0, c.tmp, p, c.s)) != cudaSuccess) return e;
  if ((e = cudaMemcpy2DAsync(cc, ldx * 8, c.tmp, p * 8, p * 8, q, cudaMemcpyDeviceToDevice, c.s)) != cudaSuccess)
    return e;
  // a <- a + b c
  if ((e = gemm1(p, p, q, 0, b, ldx, cc, ldx, a, ldx, a, ldx, c.s)) != cudaSuccess) return e;
  // b <- b d
  if ((e = gemm1(p, q, q, 0, b, ldx, d, ldx, nullptr, 0, c.tmp, q, c.s)) != cudaSuccess) return e;
  return cudaMemcpy2DAsync(b, ldx * 8, c.tmp, q * 8, q * 8, p, cudaMemcpyDeviceToDevice, c.s);
}

int64_t inplace_leaf_slots(int64_t n, int64_t leaf) {
  if (n <= leaf) return 1;
  return inplace_leaf_slots(n / 2, leaf) + inplace_leaf_slots(n - n / 2, leaf);
}
}  // namespace

extern "C" int64_t bi_inplace_by_a_workspace_bytes(int64_t n, int64_t leaf_order) {
  if (n < 1 || leaf_order < 1) return -1;
  const int64_t h = n - n / 2;
  const int64_t slots = inplace_leaf_slots(n, leaf_order);
  const int64_t leaf = std::min(n, leaf_order);
  return a256(h * h * 8) + a256(slots * 4) + a256(inv_group_scratch_bytes((int)leaf, 1));
}

extern "C" int bi_inplace_by_a(int64_t n, double* x, int64_t ldx, int64_t leaf_order, void* workspace,
                               int64_t workspace_bytes, char* fail_path, void* stream) {
  BI_REQUIRE(n >= 1 && x && workspace, "bad argument");
  BI_REQUIRE(ldx >= n, "leading dimension too small");
  BI_REQUIRE(leaf_order >= 1 && leaf_order <= 8192, "leaf order outside 1..8192");
  BI_REQUIRE(workspace_bytes >= bi_inplace_by_a_workspace_bytes(n, leaf_order), "workspace too small");
  BI_CUDA_TRY(init_attributes());
  InplaceCtx c;
  const int64_t h = n - n / 2;
  char* w = static_cast<char*>(workspace);
  c.tmp = reinterpret_cast<double*>(w);
  w += a256(h * h * 8);
  c.max_leaf = (int)inplace_leaf_slots(n, leaf_order);
  c.info = reinterpret_cast<int*>(w);
  w += a256((int64_t)c.max_leaf * 4);
  c.scratch = w;
  c.leaf = leaf_order;
  c.s = static_cast<cudaStream_t>(stream);
  BI_CUDA_TRY(inplace_rec(c, x, ldx, n, ""));
  std::vector<int> info(c.nleaf);
  BI_CUDA_TRY(cudaMemcpyAsync(info.data(), c.info, info.size() * 4, cudaMemcpyDeviceToHost, c.s));
  BI_CUDA_TRY(cudaStreamSynchronize(c.s));
  if (fail_path) fail_path[0] = 0;
  for (int i = 0; i < c.nleaf; ++i) {
    if (info[i] != 0) {
      if (fail_path) {
        std::strncpy(fail_path, c.paths[i].c_str(), 63);
        fail_path[63] = 0;
      }
      set_error("singular pivot block on path " + c.paths[i]);
      return 1;
    }
  }
  return 0;
}

extern "C" int64_t bi_residual_workspace_bytes(int64_t n, int batch) {
  if (n < 1 || batch < 0) return -1;
  const int64_t w = std::min(n, residual_panel_width(n));
  return a256(n * round_up(w, 4) * 8);
}

extern "C" int bi_residual(int64_t n, int batch, const double* a, int64_t lda, int64_t stride_a, const double* x,
                           int64_t ldx, int64_t stride_x, double* out, void* workspace, int64_t workspace_bytes,
                           void* stream) {
  BI_REQUIRE(n >= 1 && batch >= 1 && a && x && out && workspace, "bad argument");
  BI_REQUIRE(lda >= n && ldx >= n, "leading dimension too small");
  BI_REQUIRE(workspace_bytes >= bi_residual_workspace_bytes(n, batch), "workspace too small");
  BI_CUDA_TRY(init_attributes());
  BI_CUDA_TRY(launch_residual(n, batch, a, lda, stride_a, x, ldx, stride_x, out, static_cast<double*>(workspace),
                              static_cast<cudaStream_t>(stream)));
  return 0;
}
