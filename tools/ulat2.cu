// ulat2.cu -- what an independent instruction costs inside the Gibbs sweep's
// dependent fp64 chain (one warp; cycles per sweep).  DESIGN.md §7 (cfg1).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ulat2.cu -o /tmp/ulat2 && /tmp/ulat2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int N = 4096;

template <int MODE, int K>
__global__ void k(double* out, long long* cyc, double y) {
  double x = 0.3;
  double s[5] = {0, 0, 0, 0, 0};
  float f[5] = {0, 0, 0, 0, 0};
  uint32_t u[5] = {1, 2, 3, 4, 5};
  __syncwarp();
  const long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) {
    x = __dmul_rn(__fma_rn(y, -0.5, 1.0), 0.7);
    y = __dmul_rn(__fma_rn(x, -0.5, 1.0), 0.3);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (MODE == 0) s[j] = __dadd_rn(s[j], 1e-9);              // independent fp64
      if (MODE == 1) s[j] = __dadd_rn(s[j], j & 1 ? y : x);     // stats-like fp64
      if (MODE == 2) f[j] = __fmaf_rn(f[j], 0.999f, 1e-7f);     // independent fp32
      if (MODE == 3) u[j] = (u[j] ^ 0x9E3779B9u) + j;           // integer ALU
    }
  }
  const long long t1 = clock64();
  double acc = x + y;
  for (int j = 0; j < 5; ++j) acc += s[j] + f[j] + u[j];
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// The latency kernel's batch body: 32 sweeps unrolled with the 5 statistics;
// U selects how the uniforms arrive: 0 constants (no loads), 1 LDS.128 per
// sweep at use, 2 one sweep of lookahead, 3 all 32 loaded before the batch,
// 4 a ring 4 sweeps ahead.  REC: lane 0 also stores each (X, Y) to a shared row.
template <int U, bool REC>
__global__ void kb(double* out, long long* cyc, double y) {
  __shared__ double2 su[40], sxy[32];
  const uint32_t lane = threadIdx.x & 31;
  su[lane] = make_double2(0.7 + lane * 1e-3, 0.3 + lane * 1e-3);
  if (lane < 8) su[32 + lane] = make_double2(0.6, 0.4);
  sxy[lane] = make_double2(0.0, 0.0);
  __syncwarp();
  double x = 0.3, S1X = 0, S2X = 0, S1Y = 0, S2Y = 0, SXY = 0;
  const long long t0 = clock64();
  asm volatile("" : "+d"(x), "+d"(y));
  for (int i = 0; i < N / 32; ++i) {
    double2 ur[32], ring[4];
    double2 un = su[0];
    if (U == 3) {
#pragma unroll
      for (int j = 0; j < 32; ++j) ur[j] = su[j];
    }
    if (U == 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) ring[j] = su[j];
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      double2 uj = make_double2(0.7, 0.3);
      if (U == 1) uj = su[j];
      if (U == 2) { uj = un; if (j + 1 < 32) un = su[j + 1]; }
      if (U == 3) uj = ur[j];
      if (U == 4) { uj = ring[j & 3]; ring[j & 3] = su[j + 4]; }
      x = __dmul_rn(__fma_rn(y, -0.5, 1.0), uj.x);
      y = __dmul_rn(__fma_rn(x, -0.5, 1.0), uj.y);
      S1X = __dadd_rn(S1X, x); S2X = __fma_rn(x, x, S2X);
      S1Y = __dadd_rn(S1Y, y); S2Y = __fma_rn(y, y, S2Y);
      SXY = __fma_rn(x, y, SXY);
      if (REC && lane == 0) sxy[j] = make_double2(x, y);
    }
    __syncwarp();
  }
  asm volatile("" : "+d"(x), "+d"(y), "+d"(S1X), "+d"(S2X), "+d"(S1Y), "+d"(S2Y), "+d"(SXY));
  const long long t1 = clock64();
  out[threadIdx.x] = x + y + S1X + S2X + S1Y + S2Y + SXY + sxy[lane].x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int U, bool REC>
void runb(const char* name, double* out, long long* cyc) {
  long long c = 0;
  for (int rep = 0; rep < 3; ++rep) {
    kb<U, REC><<<1, 32>>>(out, cyc, 0.5);
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  }
  printf("%-44s %7.2f cycles/sweep\n", name, (double)c / N);
}

// The latency kernel's warp_batch (gibbs.cu), verbatim arithmetic: scaled
// state, constant -2^-64, 32 uniforms loaded up front.  C selects the
// constant's form: 0 the kernel's, 1 an immediate-friendly -0.5 (timing only).
template <int C>
__global__ void kw(double* out, long long* cyc, double y0) {
  __shared__ double2 su[32], sxy[32];
  const uint32_t lane = threadIdx.x & 31;
  su[lane] = make_double2(0.7e19 + lane * 1e15, 0.3e19 + lane * 1e15);
  sxy[lane] = make_double2(0.0, 0.0);
  __syncwarp();
  const double kc = C == 1 ? -0.5 : -5.42101086242752217004e-20;
  double X = 0.3e19, Y = y0 * 1e19, S1X = 0, S2X = 0, S1Y = 0, S2Y = 0, SXY = 0;
  const bool rec = lane == 0;
  const long long t0 = clock64();
  asm volatile("" : "+d"(X), "+d"(Y));
  for (int i = 0; i < N / 32; ++i) {
    double2 ur[32], ring[4];
    if (C < 2) {
#pragma unroll
      for (int j = 0; j < 32; ++j) ur[j] = su[j];
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) ring[j] = su[j];
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      double2 uj;
      if (C < 2) {
        uj = ur[j];
      } else {
        uj = ring[j & 3];
        if (j + 4 < 32) ring[j & 3] = su[j + 4];
      }
      X = __dmul_rn(__fma_rn(Y, kc, 1.0), uj.x);
      Y = __dmul_rn(__fma_rn(X, kc, 1.0), uj.y);
      S1X = __dadd_rn(S1X, X); S2X = __fma_rn(X, X, S2X);
      S1Y = __dadd_rn(S1Y, Y); S2Y = __fma_rn(Y, Y, S2Y);
      SXY = __fma_rn(X, Y, SXY);
      if (rec) sxy[j] = make_double2(X, Y);
    }
    __syncwarp();
  }
  asm volatile("" : "+d"(X), "+d"(Y), "+d"(S1X), "+d"(S2X), "+d"(S1Y), "+d"(S2Y), "+d"(SXY));
  const long long t1 = clock64();
  out[threadIdx.x] = X + Y + S1X + S2X + S1Y + S2Y + SXY + sxy[lane].x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int C>
void runw(const char* name, double* out, long long* cyc, int threads) {
  long long c = 0;
  for (int rep = 0; rep < 3; ++rep) {
    kw<C><<<1, threads>>>(out, cyc, 0.5);
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  }
  printf("%-44s %7.2f cycles/sweep (%d threads)\n", name, (double)c / N, threads);
}

template <int MODE, int K>
void run(const char* name, double* out, long long* cyc) {
  long long c = 0;
  for (int rep = 0; rep < 3; ++rep) {
    k<MODE, K><<<1, 32>>>(out, cyc, 0.5);
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  }
  printf("%-28s K=%d  %7.2f cycles/sweep\n", name, K, (double)c / N);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  run<0, 0>("chain only", out, cyc);
  run<0, 1>("+ independent DADD", out, cyc);
  run<0, 2>("+ independent DADD", out, cyc);
  run<0, 3>("+ independent DADD", out, cyc);
  run<0, 5>("+ independent DADD", out, cyc);
  run<1, 1>("+ DADD of x/y", out, cyc);
  run<1, 3>("+ DADD of x/y", out, cyc);
  run<1, 5>("+ DADD of x/y", out, cyc);
  run<2, 5>("+ independent FFMA", out, cyc);
  run<3, 5>("+ independent LOP3/IADD", out, cyc);
  runb<0, false>("batch x32 + stats: u constant", out, cyc);
  runb<1, false>("batch x32 + stats: LDS at use", out, cyc);
  runb<2, false>("batch x32 + stats: LDS 1 ahead", out, cyc);
  runb<3, false>("batch x32 + stats: 32 LDS up front", out, cyc);
  runb<4, false>("batch x32 + stats: LDS ring 4 ahead", out, cyc);
  runb<3, true>("batch x32 + stats: 32 LDS up front + STS", out, cyc);
  runb<4, true>("batch x32 + stats: ring 4 + STS", out, cyc);
  runw<0>("kernel warp_batch", out, cyc, 32);
  runw<0>("kernel warp_batch", out, cyc, 128);
  runw<1>("kernel warp_batch, constant -0.5", out, cyc, 32);
  runw<2>("kernel warp_batch, ring 4", out, cyc, 32);
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
