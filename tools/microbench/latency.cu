// Dependent-chain latencies (cycles per op) of the primitives on the K3
// column-step critical path.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>

constexpr int N = 1024;

__global__ void k_redux(unsigned* out, long long* cyc) {
  unsigned v = threadIdx.x * 2654435761u;
  __syncwarp();
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) v = __reduce_max_sync(0xffffffffu, v ^ i) + threadIdx.x;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl(unsigned* out, long long* cyc) {
  unsigned v = threadIdx.x * 2654435761u;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1 + (i & 15)) + 1;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// one butterfly round of a (64-bit key, row) argmax
__global__ void k_shfl_argmax(unsigned* out, long long* cyc) {
  unsigned long long key = (unsigned long long)(threadIdx.x * 2654435761u) << 20;
  int row = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < N / 8; ++i) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, o);
      const int orow = __shfl_xor_sync(0xffffffffu, row, o);
      if (ok > key || (ok == key && orow < row)) { key = ok; row = orow; }
    }
    key ^= i;
  }
  long long t1 = clock64();
  out[threadIdx.x] = (unsigned)key + row;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) * 8 / 5;  // per round x N
}
__global__ void k_bar(unsigned* out, long long* cyc) {
  __shared__ unsigned s[256];
  unsigned v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) {
    s[threadIdx.x] = v;
    __syncthreads();
    v = s[(threadIdx.x + 32) & 255] + 1;
  }
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dfma(double* out, long long* cyc) {
  double v = threadIdx.x * 1e-3;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) v = fma(v, 0.999, 1e-7);
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_drcp(double* out, long long* cyc) {
  double v = 1.5 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) v = 1.0 / v + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds(unsigned* out, long long* cyc) {
  __shared__ unsigned s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  unsigned v = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) v = s[v];
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  unsigned* o;
  double* od;
  long long* c;
  cudaMalloc(&o, 4096);
  cudaMalloc(&od, 8192);
  cudaMalloc(&c, 8);
  long long h;
  auto rep = [&](const char* name, int threads, auto launch) {
    for (int w = 0; w < 2; ++w) launch(threads);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-28s %7.1f cycles/op (block %d)\n", name, (double)h / N, threads);
  };
  rep("redux.sync.max.u32", 32, [&](int t) { k_redux<<<1, t>>>(o, c); });
  rep("redux.sync.max.u32 8 warps", 256, [&](int t) { k_redux<<<1, t>>>(o, c); });
  rep("shfl.bfly.b32", 32, [&](int t) { k_shfl<<<1, t>>>(o, c); });
  rep("argmax round (u64 key,row)", 32, [&](int t) { k_shfl_argmax<<<1, t>>>(o, c); });
  rep("argmax round 8 warps", 256, [&](int t) { k_shfl_argmax<<<1, t>>>(o, c); });
  rep("bar.sync + sts/lds 8 warps", 256, [&](int t) { k_bar<<<1, t>>>(o, c); });
  rep("dfma", 32, [&](int t) { k_dfma<<<1, t>>>(od, c); });
  rep("1.0/x (f64 div)", 32, [&](int t) { k_drcp<<<1, t>>>(od, c); });
  rep("lds.32 pointer chase", 32, [&](int t) { k_lds<<<1, t>>>(o, c); });
  return 0;
}
