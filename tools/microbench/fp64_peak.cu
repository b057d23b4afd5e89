// Microbenchmark: FP64 DMMA (mma.sync m8n8k4 f64) and DFMA issue rates on sm_100a.
// Used once to pick the GEMM inner-loop instruction; numbers recorded in profiles/.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double acc[NACC][2];
  for (int i = 0; i < NACC; ++i) { acc[i][0] = 0.0; acc[i][1] = 0.0; }
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double acc[NACC];
  for (int i = 0; i < NACC; ++i) acc[i] = i;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clock %d kHz smem/block optin %zu\n", p.name, p.multiProcessorCount, clk, p.sharedMemPerBlockOptin);
  double* out; cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int ctas_per_sm = 1; ctas_per_sm <= 2; ++ctas_per_sm) {
      int iters = 4000;
      dim3 grid(sms * ctas_per_sm), block(32 * warps);
      dmma_loop<16><<<grid, block>>>(out, 10);
      cudaEventRecord(e0);
      dmma_loop<16><<<grid, block>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 16 * (double)iters * warps * grid.x;
      printf("DMMA m8n8k4: warps/cta %2d ctas/sm %d : %.2f TFLOP/s (%.3f ms)\n", warps, ctas_per_sm, flops / ms / 1e9, ms);
    }
  }
  for (int warps = 4; warps <= 32; warps *= 2) {
    int iters = 4000;
    dim3 grid(sms * 2), block(32 * warps);
    dfma_loop<16><<<grid, block>>>(out, 10);
    cudaEventRecord(e0);
    dfma_loop<16><<<grid, block>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * (double)iters * 32 * warps * grid.x;
    printf("DFMA: warps/cta %2d ctas/sm 2 : %.2f TFLOP/s (%.3f ms)\n", warps, flops / ms / 1e9, ms);
  }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
