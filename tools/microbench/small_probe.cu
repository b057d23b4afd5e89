// Per-phase cycle breakdown of the fused small-block K3 kernel (clock64
// probes compiled in with BI_SMALL_PROBE): batched inversion of `count`
// blocks of order n; prints CTA 0 and CTA 1 (cluster ranks 0 and 1 of block 0).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//     tools/microbench/small_probe.cu paper_2305_11103_b200/csrc/bi_gemm.cu \
//     paper_2305_11103_b200/csrc/bi_gemm_tma.cu -o tools/microbench/small_probe -lcuda
#define BI_SMALL_PROBE
#define BI_PANEL_PROBE
#include "../../paper_2305_11103_b200/csrc/bi_inv.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 256, count = argc > 2 ? atoi(argv[2]) : 64;
  std::vector<double> h((size_t)count * n * n);
  unsigned s = 1;
  for (size_t i = 0; i < h.size(); ++i) {
    s = s * 1664525u + 1013904223u;
    h[i] = ((s >> 8) * (1.0 / 16777216.0) - 0.5) / 16.0;
  }
  for (int b = 0; b < count; ++b)
    for (int i = 0; i < n; ++i) h[(size_t)b * n * n + (size_t)i * n + i] += 4.0;
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
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) bi::launch_inv_group(g, 0);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int rep = 0; rep < reps; ++rep) {
    cudaError_t e = bi::launch_inv_group(g, 0);
    if (e != cudaSuccess) {
      printf("launch failed: %s\n", cudaGetErrorString(e));
      return 1;
    }
  }
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long p[2][8];
  cudaMemcpyFromSymbol(p, bi::g_small_probe, sizeof(p));
  const char* names[] = {"load+max", "panels", "inner updates", "outer gathers", "outer updates", "store",
                         "cluster syncs", "-"};
  printf("n=%d count=%d: %.3f ms per call (%s)\n", n, count, ms / reps, cudaGetErrorString(cudaGetLastError()));
  for (int c = 0; c < 2; ++c) {
    long long tot = 0;
    for (int i = 0; i < 7; ++i) tot += p[c][i];
    printf("CTA %d: total %lld cycles\n", c, tot);
    for (int i = 0; i < 7; ++i) printf("  %-16s %8lld cyc\n", names[i], p[c][i]);
  }
  long long pp[2][16];
  cudaMemcpyFromSymbol(pp, bi::g_panel_probe, sizeof(pp));
  const char* pn[] = {"prologue", "A/publish", "barrier", "B/xwarp", "verdict/bookkeep", "f+col", "next cand",
                      "other FMAs", "epilogue"};
  for (int w = 0; w < 2; ++w) {
    printf("last panel, thread %d:", w ? 224 : 0);
    for (int i = 0; i < 9; ++i) printf(" %s=%lld", pn[i], pp[w][i]);
    printf("\n");
  }
  return 0;
}
