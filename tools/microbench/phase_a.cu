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

// V6: lockstep column loop of the single-CTA panel (256 threads, one row each):
// owner publishes row c, one barrier, every row updates.  MODE bit 1: skip rcp,
// bit 2: skip the 30 row FMAs, bit 4: skip the objection check.
template <int MODE>
__global__ void lockstep(const double* in, double* out, long long* cyc, int reps) {
  __shared__ __align__(16) double s_lrow[2][NB + 2];
  const int t = threadIdx.x;
  const double* src = in + (size_t)blockIdx.x * 256 * NB;
  double P[NB];
  long long total = 0;
  int objection = 0;
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
    for (int k = 0; k < NB; ++k) P[k] = src[t * NB + k];
    double rc = 1.0 / P[0];
    __syncthreads();
    const long long t0 = clock64();
    for (int c = 0; c < NB; ++c) {
      const int buf = c & 1;
      if (MODE & 32) {  // predicated stores, no branch
        const unsigned base = (unsigned)__cvta_generic_to_shared(s_lrow[buf]);
        const bool me = t == c;
#pragma unroll
        for (int k = 0; k < NB / 2; ++k) st_pred_v2(base + 16 * k, P[2 * k], P[2 * k + 1], me);
        st_pred_f64(base + 8 * NB, rc, me);
      } else if (t == c && !(MODE & 16)) {
        double2* dst = reinterpret_cast<double2*>(s_lrow[buf]);
#pragma unroll
        for (int k = 0; k < NB / 2; ++k) dst[k] = make_double2(P[2 * k], P[2 * k + 1]);
        s_lrow[buf][NB] = rc;
      }
      __syncthreads();
      double prr[NB];
      if (MODE & 8) {
        const double v0 = s_lrow[buf][c & 7];
#pragma unroll
        for (int k = 0; k < NB; ++k) prr[k] = v0 + k;
      } else {
#pragma unroll
        for (int k = 0; k < NB / 2; ++k) {
          const double2 v = reinterpret_cast<const double2*>(s_lrow[buf])[k];
          prr[2 * k] = v.x;
          prr[2 * k + 1] = v.y;
        }
      }
      const double inv = s_lrow[buf][NB];
      if (!(MODE & 4)) {
        if (t > c && fabs(P[0]) > fabs(prr[0])) objection = 1;
      }
      const bool isp = t == c;
      const double fi = isp ? 1.0 - inv : P[0] * inv;
      const double ti = isp ? inv : -fi;
      P[0] = fma(-fi, prr[1], P[1]);
      if (!(MODE & 1)) rc = fast_rcp(P[0]);
      else rc = P[0];
      if (!(MODE & 2)) {
#pragma unroll
        for (int k = 1; k < NB - 1; ++k) P[k] = fma(-fi, prr[k + 1], P[k + 1]);
      }
      P[NB - 1] = ti;
    }
    const long long t1 = clock64();
    total += t1 - t0;
  }
#pragma unroll
  for (int k = 0; k < NB; ++k) out[(size_t)blockIdx.x * 256 * NB + t * NB + k] = P[k];
  if (t == 0) cyc[blockIdx.x] = total / reps + objection;
}

// V7: lockstep with 8 x 4 blocks per thread (256 threads: i = t / 8 row block,
// j = t % 8 column block): per step the column-c owners publish their 8
// values, the row-c owners their 4, one barrier, every thread reads 8 + 4 + 1.
template <int STATIC>
__global__ void __launch_bounds__(256, 1) lockstep2d(const double* in, double* out, long long* cyc, int reps) {
  __shared__ __align__(16) double s_col[2][256], s_row[2][NB + 2];
  const int t = threadIdx.x, bi = t >> 3, bj = t & 7;
  const double* src = in + (size_t)blockIdx.x * 256 * NB;
  double w[8][4];
  long long total = 0;
  int objection = 0;
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) w[a][b] = src[(bi * 8 + a) * NB + bj * 4 + b];
    if (t == 0) s_row[0][NB] = 1.0 / w[0][0];
    __syncthreads();
    const long long t0 = clock64();
#pragma unroll 1
    for (int c = 0; c < NB; ++c) {
      const int buf = c & 1;
      // publish column c (owners: bj == c / 4) and row c (owners: bi == c / 8)
      if (bj == (c >> 2)) {
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          double v = w[a][0];
          if (!STATIC) {
#pragma unroll
            for (int b = 1; b < 4; ++b) v = (c & 3) == b ? w[a][b] : v;
          }
          s_col[buf][bi * 8 + a] = v;
        }
      }
      if (bi == (c >> 3)) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          double v = w[0][b];
          if (!STATIC) {
#pragma unroll
            for (int a = 1; a < 8; ++a) v = (c & 7) == a ? w[a][b] : v;
          }
          s_row[buf][bj * 4 + b] = v;
        }
      }
      __syncthreads();
      const double inv = s_row[buf][NB];
      double x[8], pr[4];
#pragma unroll
      for (int a = 0; a < 8; ++a) x[a] = s_col[buf][bi * 8 + a];
#pragma unroll
      for (int b = 0; b < 4; ++b) pr[b] = s_row[buf][bj * 4 + b];
      const double pc = s_row[buf][c];
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const int r = bi * 8 + a;
        if (r > c && fabs(x[a]) > fabs(pc)) objection = 1;
        const bool isp = r == c;
        const double fi = isp ? 1.0 - inv : x[a] * inv;
        const double ti = isp ? inv : -fi;
#pragma unroll
        for (int b = 0; b < 4; ++b) w[a][b] = (!STATIC && bj * 4 + b == c) ? ti : fma(-fi, pr[b], w[a][b]);
      }
      // the next pivot's reciprocal
      if (bi == ((c + 1) >> 3) && bj == ((c + 1) >> 2) && c + 1 < NB) {
        double v = w[0][0];
        if (!STATIC) {
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
              if (bi * 8 + a == c + 1 && bj * 4 + b == c + 1) v = w[a][b];
        }
        s_row[buf ^ 1][NB] = fast_rcp(v);
      }
    }
    const long long t1 = clock64();
    total += t1 - t0;
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) out[(size_t)blockIdx.x * 256 * NB + (bi * 8 + a) * NB + bj * 4 + b] = w[a][b];
  if (t == 0) cyc[blockIdx.x] = total / reps + objection;
}

// V8: lockstep with TWO threads per row (512 threads, lanes 2i / 2i+1 = row
// halves): register rotation over the 32 columns split 16 / 16, the boundary
// value and the multiplier exchanged by one shuffle each; the owner pair
// publishes 8 + 8 values, readers load only their half.
constexpr int H = NB / 2;
__global__ void __launch_bounds__(512, 1) lockstep2(const double* in, double* out, long long* cyc, int reps) {
  __shared__ __align__(16) double s_lrow[2][NB + 2];
  const int t = threadIdx.x, row = t >> 1, h = t & 1;
  const double* src = in + (size_t)blockIdx.x * 256 * NB;
  double P[H];
  long long total = 0;
  int objection = 0;
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
    for (int k = 0; k < H; ++k) P[k] = src[row * NB + h * H + k];
    double rc = h == 0 ? fast_rcp(P[0]) : 0.0;
    __syncthreads();
    const long long t0 = clock64();
    for (int c = 0; c < NB; ++c) {
      const int buf = c & 1;
      if (row == c) {  // the owner pair publishes its halves (rotated row: P of h=0 = cols c.., h=1 = rest)
        double2* dst = reinterpret_cast<double2*>(s_lrow[buf] + h * H);
#pragma unroll
        for (int k = 0; k < H / 2; ++k) dst[k] = make_double2(P[2 * k], P[2 * k + 1]);
        if (h == 0) s_lrow[buf][NB] = rc;
      }
      __syncthreads();
      // reader: needs prr[k + 1] for its registers k: h = 0 -> pr[1 .. 16], h = 1 -> pr[17 .. 31] (+ none)
      double prr[H + 1];
#pragma unroll
      for (int k = 0; k < H / 2; ++k) {
        const double2 v = reinterpret_cast<const double2*>(s_lrow[buf] + h * H)[k];
        prr[2 * k] = v.x;
        prr[2 * k + 1] = v.y;
      }
      prr[H] = h == 0 ? s_lrow[buf][H] : 0.0;
      const double inv = s_lrow[buf][NB];
      // multiplier from the h = 0 thread (it holds the current column), boundary from h = 1
      const double x = __shfl_sync(0xffffffffu, P[0], (threadIdx.x & 31) & ~1);
      const double nb0 = __shfl_down_sync(0xffffffffu, P[0], 1);  // h=0 receives h=1's old P[0]
      if (h == 0 && row > c && fabs(x) > fabs(prr[0])) objection = 1;
      const bool isp = row == c;
      const double fi = isp ? 1.0 - inv : x * inv;
      const double ti = isp ? inv : -fi;
      if (h == 0) {
        P[0] = fma(-fi, prr[1], P[1]);
        rc = fast_rcp(P[0]);
#pragma unroll
        for (int k = 1; k < H - 1; ++k) P[k] = fma(-fi, prr[k + 1], P[k + 1]);
        P[H - 1] = fma(-fi, prr[H], nb0);
      } else {
#pragma unroll
        for (int k = 0; k < H - 1; ++k) P[k] = fma(-fi, prr[k + 1], P[k + 1]);
        P[H - 1] = ti;
      }
    }
    const long long t1 = clock64();
    total += t1 - t0;
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < H; ++k) out[(size_t)blockIdx.x * 256 * NB + row * NB + h * H + k] = P[k];
  if (t == 0) cyc[blockIdx.x] = total / reps + objection;
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
  {
    const int lb = 64;
    std::vector<double> h2((size_t)lb * 256 * NB);
    for (size_t i = 0; i < h2.size(); ++i) h2[i] = ((i * 2654435761u) % 1000) / 16000.0;
    for (int b = 0; b < lb; ++b)
      for (int i = 0; i < NB; ++i) h2[(size_t)b * 256 * NB + i * NB + i] += 4.0;
    double *d2, *o2;
    cudaMalloc(&d2, h2.size() * 8);
    cudaMalloc(&o2, h2.size() * 8);
    cudaMemcpy(d2, h2.data(), h2.size() * 8, cudaMemcpyHostToDevice);
    long long* c2;
    cudaMalloc(&c2, lb * 8);
    auto runl = [&](auto kern, const char* name) {
      kern<<<lb, 256>>>(d2, o2, c2, reps);
      cudaDeviceSynchronize();
      std::vector<long long> cc(lb);
      cudaMemcpy(cc.data(), c2, lb * 8, cudaMemcpyDeviceToHost);
      long long sum = 0;
      for (auto v : cc) sum += v;
      printf("%-34s %6lld cyc / 32 steps = %.1f cyc/step\n", name, sum / lb, (double)sum / lb / 32);
    };
    runl(lockstep<0>, "V6 lockstep 256 thr (full)");
    runl(lockstep<1>, "V6 lockstep, no rcp");
    runl(lockstep<2>, "V6 lockstep, no row FMAs");
    runl(lockstep<4>, "V6 lockstep, no objection check");
    runl(lockstep<7>, "V6 lockstep, barrier+bcast only");
    runl(lockstep<15>, "V6 barrier + 1-value bcast only");
    runl(lockstep<23>, "V6 barrier + bcast, no owner STS");
    runl(lockstep<32>, "V6 lockstep full, predicated STS");
    runl(lockstep<39>, "V6 barrier+bcast, predicated STS");
    runl(lockstep2d<0>, "V7 lockstep 8x4 blocks");
    {
      lockstep2<<<lb, 512>>>(d2, o2, c2, reps);
      cudaDeviceSynchronize();
      std::vector<long long> cc(lb);
      cudaMemcpy(cc.data(), c2, lb * 8, cudaMemcpyDeviceToHost);
      long long sum = 0;
      for (auto v : cc) sum += v;
      printf("%-34s %6lld cyc / 32 steps = %.1f cyc/step\n", "V8 lockstep 2 thr/row (512 thr)", sum / lb, (double)sum / lb / 32);
      std::vector<double> a6(h2.size()), a8(h2.size());
      lockstep<0><<<lb, 256>>>(d2, o2, c2, 1);
      cudaMemcpy(a6.data(), o2, a6.size() * 8, cudaMemcpyDeviceToHost);
      lockstep2<<<lb, 512>>>(d2, o2, c2, 1);
      cudaMemcpy(a8.data(), o2, a8.size() * 8, cudaMemcpyDeviceToHost);
      printf("  V8 vs V6 bitwise %s (%s)\n", memcmp(a6.data(), a8.data(), a6.size() * 8) ? "DIFFER" : "equal",
             cudaGetErrorString(cudaGetLastError()));
    }
    runl(lockstep2d<1>, "V7 static publish (timing only)");
    {  // bitwise: V6 full vs V7
      std::vector<double> a6(h2.size()), a7(h2.size());
      lockstep<0><<<lb, 256>>>(d2, o2, c2, 1);
      cudaMemcpy(a6.data(), o2, a6.size() * 8, cudaMemcpyDeviceToHost);
      lockstep2d<0><<<lb, 256>>>(d2, o2, c2, 1);
      cudaMemcpy(a7.data(), o2, a7.size() * 8, cudaMemcpyDeviceToHost);
      printf("  V7 vs V6 bitwise %s\n", memcmp(a6.data(), a7.data(), a6.size() * 8) ? "DIFFER" : "equal");
    }
  }
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
