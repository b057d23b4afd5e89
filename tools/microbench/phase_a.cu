// Phase A of the verified fast panel (bi_inv.cu): one warp runs the 32
// unpivoted GJ column steps on the panel's 32 pivot rows (row per lane,
// register rotation).  Variants differ only in how pivot row c reaches the
// other lanes; the FMAs are the same, so every variant must be bitwise equal.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/microbench/phase_a.cu -o /tmp/phase_a
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>

constexpr int NB = 32;

__device__ __forceinline__ double fast_rcp(double p) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(p));
  const double e = fma(-p, r, 1.0);
  r = fma(r, fma(e, e, e), r);
  return fma(r, fma(-p, r, 1.0), r);
}

__device__ __forceinline__ void st_pred_v2(unsigned addr, double x, double y, bool p) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n @q st.shared.v2.f64 [%0], {%1, %2};\n}\n" ::"r"(addr), "d"(x),
      "d"(y), "r"((unsigned)p)
      : "memory");
}
__device__ __forceinline__ void st_pred_f64(unsigned addr, double x, bool p) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.shared.f64 [%0], %1;\n}\n" ::"r"(addr), "d"(x),
               "r"((unsigned)p)
               : "memory");
}

template <int V>
__global__ void phase_a(const double* in, double* out, long long* cyc, int reps) {
  __shared__ __align__(16) double s_fpr[NB][NB + 2];
  const int lane = threadIdx.x & 31;
  const double* src = in + (size_t)blockIdx.x * NB * NB;
  double P[NB];
  long long total = 0;
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
    for (int k = 0; k < NB; ++k) P[k] = src[lane * NB + k];
    double rc_own = fast_rcp(P[0]);
    __syncwarp();
    const long long t0 = clock64();
    for (int c = 0; c < NB; ++c) {
      double prr[NB];
      double inv;
      if constexpr (V == 0) {  // as bi_inv.cu: divergent store, two syncwarps
        if (lane == c) {
          double2* dst = reinterpret_cast<double2*>(s_fpr[c]);
#pragma unroll
          for (int k = 0; k < NB / 2; ++k) dst[k] = make_double2(P[2 * k], P[2 * k + 1]);
          s_fpr[c][NB] = rc_own;
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < NB / 2; ++k) {
          const double2 v = reinterpret_cast<const double2*>(s_fpr[c])[k];
          prr[2 * k] = v.x;
          prr[2 * k + 1] = v.y;
        }
        inv = s_fpr[c][NB];
      } else if constexpr (V == 1 || V >= 3) {  // shuffles
#pragma unroll
        for (int k = 0; k < NB; ++k) prr[k] = __shfl_sync(0xffffffffu, P[k], c);
        inv = __shfl_sync(0xffffffffu, rc_own, c);
      } else {  // predicated stores, one syncwarp (one slot per step: no WAR)
        const unsigned base = (unsigned)__cvta_generic_to_shared(s_fpr[c]);
        const bool me = lane == c;
#pragma unroll
        for (int k = 0; k < NB / 2; ++k) st_pred_v2(base + 16 * k, P[2 * k], P[2 * k + 1], me);
        st_pred_f64(base + 8 * NB, rc_own, me);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < NB / 2; ++k) {
          const double2 w = *reinterpret_cast<const double2*>(&s_fpr[c][2 * k]);
          prr[2 * k] = w.x;
          prr[2 * k + 1] = w.y;
        }
        inv = s_fpr[c][NB];
      }
      const double fi = lane == c ? 1.0 - inv : P[0] * inv;
      const double ti = lane == c ? inv : -fi;
      P[0] = fma(-fi, prr[1], P[1]);
      if constexpr (V == 3) rc_own = P[0];  // timing only: no reciprocal
      else rc_own = fast_rcp(P[0]);
      if constexpr (V != 4) {
#pragma unroll
        for (int k = 1; k < NB - 1; ++k) P[k] = fma(-fi, prr[k + 1], P[k + 1]);
      }
      P[NB - 1] = ti;
      if constexpr (V == 0) __syncwarp();
    }
    const long long t1 = clock64();
    total += t1 - t0;
  }
#pragma unroll
  for (int k = 0; k < NB; ++k) out[(size_t)blockIdx.x * NB * NB + lane * NB + k] = P[k];
  if (lane == 0) cyc[blockIdx.x] = total / reps;
}

__global__ void chains(long long* cyc) {
  double v = threadIdx.x * 1e-3 + 1.5, w = 1.25;
  long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < 1024; ++i) v = fma(v, 0.999, 1e-3);
  long long t1 = clock64();
#pragma unroll 8
  for (int i = 0; i < 1024; ++i) w = fast_rcp(w) + 1.0;
  long long t2 = clock64();
  double x = 1.5;
#pragma unroll 8
  for (int i = 0; i < 1024; ++i) x = fast_rcp(fma(-(x * 0.5), 0.25, 1.7));
  long long t3 = clock64();
  double y = v;
#pragma unroll 8
  for (int i = 0; i < 1024; ++i) y = __shfl_sync(0xffffffffu, y, (threadIdx.x + 1) & 31) + 1.0;
  long long t4 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
  }
  if (v + w + x + y == 12345.0) cyc[5] = 1;
}

// V5: the CTA-wide (256 threads) fixed-column phase A of bi_inv.cu
__global__ void phase_a_2d(const double* in, double* out, long long* cyc, int reps) {
  __shared__ double s_col[2][NB], s_row[2][NB], s_inv[2];
  __shared__ double s_fpr[NB][NB + 2];
  const int t = threadIdx.x, pr_ = t >> 3, g4 = (t & 7) * 4;
  const double* src = in + (size_t)blockIdx.x * NB * NB;
  double w[4];
  long long total = 0;
  int bad = 0;
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
    for (int m = 0; m < 4; ++m) w[m] = src[pr_ * NB + g4 + m];
    if (t == 0) s_inv[0] = fast_rcp(src[0]);
    __syncthreads();
    const long long t0 = clock64();
    for (int c = 0; c < NB; ++c) {
      const int buf = c & 1;
      if ((c >> 2) == (t & 7)) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
          if (g4 + m == c) s_col[buf][pr_] = w[m];
      }
      if (pr_ == c) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          s_row[buf][g4 + m] = w[m];
          s_fpr[c][(g4 + m - c) & (NB - 1)] = w[m];
        }
      }
      __syncthreads();
      const double inv = s_inv[buf];
      const double x = s_col[buf][pr_];
      if (pr_ > c && x > s_row[buf][c]) bad = 1;
      const double fi = pr_ == c ? 1.0 - inv : x * inv;
      const double ti = pr_ == c ? inv : -fi;
#pragma unroll
      for (int m = 0; m < 4; ++m) w[m] = g4 + m == c ? ti : fma(-fi, s_row[buf][g4 + m], w[m]);
      if (pr_ == c + 1) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
          if (g4 + m == c + 1) s_inv[buf ^ 1] = fast_rcp(w[m]);
      }
    }
    const long long t1 = clock64();
    total += t1 - t0;
    __syncthreads();
  }
  // final rows in rotated order after 32 steps = identity: lane r, col k
  double* o = out + (size_t)blockIdx.x * NB * NB;
#pragma unroll
  for (int m = 0; m < 4; ++m) o[pr_ * NB + g4 + m] = w[m];
  if (t == 0) cyc[blockIdx.x] = total / reps + bad;
}

int main() {
  const int blocks = 64, reps = 20;
  std::vector<double> h((size_t)blocks * NB * NB);
  unsigned s = 7;
  for (size_t i = 0; i < h.size(); ++i) {
    s = s * 1664525u + 1013904223u;
    h[i] = ((s >> 8) * (1.0 / 16777216.0) - 0.5) / 16.0;
  }
  for (int b = 0; b < blocks; ++b)
    for (int i = 0; i < NB; ++i) h[(size_t)b * NB * NB + i * NB + i] += 4.0;
  double *din, *dout;
  long long* dc;
  cudaMalloc(&din, h.size() * 8);
  cudaMalloc(&dout, h.size() * 8);
  cudaMalloc(&dc, blocks * 8);
  cudaMemcpy(din, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  std::vector<double> ref(h.size()), got(h.size());
  std::vector<long long> c(blocks);
  auto run = [&](auto kern, const char* name, std::vector<double>& o) {
    kern<<<blocks, kern == (decltype(kern))phase_a_2d ? 256 : 32>>>(din, dout, dc, reps);
    cudaDeviceSynchronize();
    cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(c.data(), dc, blocks * 8, cudaMemcpyDeviceToHost);
    long long mx = 0, sum = 0;
    for (auto v : c) {
      mx = v > mx ? v : mx;
      sum += v;
    }
    printf("%-28s %6lld cyc / 32 steps (max %lld) = %.1f cyc/step\n", name, sum / blocks, mx,
           (double)sum / blocks / 32);
  };
  run(phase_a<0>, "V0 smem divergent (current)", ref);
  run(phase_a<1>, "V1 shfl", got);
  printf("  V1 bitwise %s\n", memcmp(ref.data(), got.data(), ref.size() * 8) ? "DIFFER" : "equal");
  run(phase_a<2>, "V2 smem predicated", got);
  printf("  V2 bitwise %s\n", memcmp(ref.data(), got.data(), ref.size() * 8) ? "DIFFER" : "equal");
  run(phase_a_2d, "V5 CTA-wide 2D (256 thr)", got);
  printf("  V5 bitwise %s\n", memcmp(ref.data(), got.data(), ref.size() * 8) ? "DIFFER" : "equal");
  run(phase_a<3>, "V3 shfl, no rcp (timing)", got);
  run(phase_a<4>, "V4 shfl, no row FMAs (timing)", got);
  chains<<<1, 32>>>(dc);
  cudaDeviceSynchronize();
  long long cc[4];
  cudaMemcpy(cc, dc, sizeof(cc), cudaMemcpyDeviceToHost);
  printf("latency: DFMA %.1f  fast_rcp %.1f  DMUL+DFMA+rcp %.1f  shfl64 %.1f cyc\n", cc[0] / 1024.0, cc[1] / 1024.0,
         cc[2] / 1024.0, cc[3] / 1024.0);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
