// Per-phase cycle breakdown of the K3 panel kernel (clock64 probes compiled
// in with BI_PANEL_PROBE): batched inversion of `count` blocks of order n,
// prints the last panel launch's per-phase cycles for warps 0 and 7.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//     tools/microbench/panel_probe.cu paper_2305_11103_b200/csrc/bi_gemm.cu \
//     paper_2305_11103_b200/csrc/bi_gemm_tma.cu -o tools/microbench/panel_probe
#define BI_PANEL_PROBE
#include "../../paper_2305_11103_b200/csrc/bi_inv.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 512, count = argc > 2 ? atoi(argv[2]) : 8;
  std::vector<double> h((size_t)count * n * n);
  unsigned s = 1;
  for (size_t i = 0; i < h.size(); ++i) {
    s = s * 1664525u + 1013904223u;
    h[i] = ((s >> 8) * (1.0 / 16777216.0) - 0.5) / 16.0;
  }
  for (int b = 0; b < count; ++b)
    for (int i = 0; i < n; ++i) h[(size_t)b * n * n + (size_t)i * n + i] += 2.0;
  double *src, *dst;
  void* scratch;
  int* info;
  cudaMalloc(&src, h.size() * 8);
  cudaMalloc(&dst, h.size() * 8);
  cudaMalloc(&info, count * 4);
  cudaMemcpy(src, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  bi::InvGroup g{};
  g.n = n;
  g.count = count;
  g.src_base = src;
  g.src_stride = (int64_t)n * n;
  g.ld_src = n;
  g.dst_base = dst;
  g.dst_stride = (int64_t)n * n;
  g.ld_dst = n;
  g.info = info;
  cudaMalloc(&scratch, bi::inv_group_scratch_bytes(n, count));
  bi::inv_group_layout(g, scratch);
  for (int rep = 0; rep < 3; ++rep) {
    cudaError_t e = bi::launch_inv_group(g, 0);
    if (e != cudaSuccess) {
      printf("launch failed: %s\n", cudaGetErrorString(e));
      return 1;
    }
  }
  cudaDeviceSynchronize();
  long long p[2][16];
  cudaMemcpyFromSymbol(p, bi::g_panel_probe, sizeof(p));
  const char* names[] = {"prologue", "publish", "barrier", "xwarp argmax", "bookkeep+prow",
                         "f + column c+1", "next candidate", "other FMAs", "epilogue"};
  const int cols = 32;
  for (int w = 0; w < 2; ++w) {
    long long tot = 0;
    for (int i = 0; i < 9; ++i) tot += p[w][i];
    printf("warp %d: total %lld cycles\n", w ? 7 : 0, tot);
    for (int i = 0; i < 9; ++i)
      printf("  %-16s %8lld cyc  %7.1f /col\n", names[i], p[w][i], (i >= 1 && i <= 7) ? (double)p[w][i] / cols : 0.0);
  }
  return 0;
}
