// ulat.cu -- dependent-chain LATENCY microbenchmarks on B200 (one warp,
// clock64 around N dependent ops): the constants of the Gibbs latency
// roofline (cfg1).  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/ulat.cu -o /tmp/ulat && /tmp/ulat
// Caveat: the loops are fully unrolled over N = 4096 steps, so the multi-op
// modes (stats, lagged stats, LDS ring, records) run from a code footprint far
// beyond the instruction cache and overstate their cost; tools/ulat2.cu
// measures the same bodies 32-unrolled as the kernels run them.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void k_lat(double* out, long long* cyc, double seed, int mode) {
  double x = seed + threadIdx.x * 1e-9, y = 0.5;
  uint32_t u = (uint32_t)threadIdx.x + 12345u;
  __syncwarp();
  const long long t0 = clock64();
  if (mode == 0) {                         // DFMA chain
    for (int i = 0; i < N; ++i) x = __fma_rn(x, 0.999999, 1e-7);
  } else if (mode == 1) {                  // DMUL chain
    for (int i = 0; i < N; ++i) x = __dmul_rn(x, 1.0000001);
  } else if (mode == 2) {                  // DADD chain
    for (int i = 0; i < N; ++i) x = __dadd_rn(x, 1e-9);
  } else if (mode == 3) {                  // Gibbs sweep: fma, mul, fma, mul (dependent)
    for (int i = 0; i < N; ++i) {
      x = __dmul_rn(__fma_rn(y, -0.5, 1.0), 0.7);
      y = __dmul_rn(__fma_rn(x, -0.5, 1.0), 0.3);
    }
  } else if (mode == 6) {                  // Gibbs sweep + the 5 running statistics
    double s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0;
    for (int i = 0; i < N; ++i) {
      x = __dmul_rn(__fma_rn(y, -0.5, 1.0), 0.7);
      y = __dmul_rn(__fma_rn(x, -0.5, 1.0), 0.3);
      s1 = __dadd_rn(s1, x); s2 = __fma_rn(x, x, s2); s3 = __dadd_rn(s3, y);
      s4 = __fma_rn(y, y, s4); s5 = __fma_rn(x, y, s5);
    }
    x += s1 + s2 + s3 + s4 + s5;
  } else if (mode == 8) {                  // sweep + stats lagged one step (software pipelined)
    double s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, px = 0, py = 0;
    for (int i = 0; i < N; ++i) {
      x = __dmul_rn(__fma_rn(y, -0.5, 1.0), 0.7);
      s1 = __dadd_rn(s1, px); s2 = __fma_rn(px, px, s2); s5 = __fma_rn(px, py, s5);
      y = __dmul_rn(__fma_rn(x, -0.5, 1.0), 0.3);
      s3 = __dadd_rn(s3, py); s4 = __fma_rn(py, py, s4);
      px = x; py = y;
    }
    x += s1 + s2 + s3 + s4 + s5;
  } else if (mode == 9) {                  // 8 independent DFMA chains: per-warp fp64 issue rate
    double a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3, a4 = x + 4, a5 = x + 5, a6 = x + 6, a7 = x + 7;
    for (int i = 0; i < N / 8; ++i) {
      a0 = __fma_rn(a0, 0.999, 1e-7); a1 = __fma_rn(a1, 0.999, 1e-7);
      a2 = __fma_rn(a2, 0.999, 1e-7); a3 = __fma_rn(a3, 0.999, 1e-7);
      a4 = __fma_rn(a4, 0.999, 1e-7); a5 = __fma_rn(a5, 0.999, 1e-7);
      a6 = __fma_rn(a6, 0.999, 1e-7); a7 = __fma_rn(a7, 0.999, 1e-7);
    }
    x = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  } else if (mode == 10) {                 // 8 independent FFMA chains (fp32 reference)
    float a0 = x, a1 = x + 1, a2 = x + 2, a3 = x + 3, a4 = x + 4, a5 = x + 5, a6 = x + 6, a7 = x + 7;
    for (int i = 0; i < N / 8; ++i) {
      a0 = __fmaf_rn(a0, 0.999f, 1e-7f); a1 = __fmaf_rn(a1, 0.999f, 1e-7f);
      a2 = __fmaf_rn(a2, 0.999f, 1e-7f); a3 = __fmaf_rn(a3, 0.999f, 1e-7f);
      a4 = __fmaf_rn(a4, 0.999f, 1e-7f); a5 = __fmaf_rn(a5, 0.999f, 1e-7f);
      a6 = __fmaf_rn(a6, 0.999f, 1e-7f); a7 = __fmaf_rn(a7, 0.999f, 1e-7f);
    }
    x = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  } else if (mode == 11 || mode == 12) {  // sweep, u from LDS (lookahead 4), state recorded per step
    __shared__ double2 su2[36], sxy2[32];
    su2[threadIdx.x & 31] = make_double2(0.7 + threadIdx.x * 1e-3, 0.3);
    if ((threadIdx.x & 31) < 4) su2[32 + (threadIdx.x & 31)] = make_double2(0.6, 0.4);
    __syncwarp();
    const uint32_t lane = threadIdx.x & 31;
    double mx = 0, my = 0;
    for (int i = 0; i < N / 32; ++i) {
      double2 ring[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) ring[j] = su2[j];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const double2 uj = ring[j % 4];
        ring[j % 4] = su2[j + 4];
        x = __dmul_rn(__fma_rn(y, -0.5, 1.0), uj.x);
        y = __dmul_rn(__fma_rn(x, -0.5, 1.0), uj.y);
        if (mode == 11) { if (lane == 0) sxy2[j] = make_double2(x, y); }
        else if (lane == (uint32_t)j) { mx = x; my = y; }
      }
    }
    x += sxy2[lane].x + mx + my;
  } else if (mode == 7) {                  // Gibbs sweep with u from shared memory (LDS.128)
    __shared__ double2 su[64];
    su[threadIdx.x] = make_double2(0.7 + threadIdx.x * 1e-3, 0.3);
    su[threadIdx.x + 32] = make_double2(0.6, 0.4 + threadIdx.x * 1e-3);
    __syncwarp();
    for (int i = 0; i < N; ++i) {
      const double2 u = su[i & 63];
      x = __dmul_rn(__fma_rn(y, -0.5, 1.0), u.x);
      y = __dmul_rn(__fma_rn(x, -0.5, 1.0), u.y);
    }
  } else if (mode == 4) {                  // SHFL of a double (2 x 32-bit), dependent
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (int)(i & 31)) + 1e-9;
  } else if (mode == 5) {                  // IMAD.WIDE + LOP3 (Philox half-round) chain
    for (int i = 0; i < N; ++i) {
      const uint64_t p = (uint64_t)0xD2511F53u * u;
      u = (uint32_t)(p >> 32) ^ (uint32_t)p ^ 0x9E3779B9u;
    }
    x += u;
  }
  const long long t1 = clock64();
  out[threadIdx.x & 31] = x + y;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main(int argc, char** argv) {
  const int nthreads = argc > 1 ? atoi(argv[1]) : 32;   // 32: one warp; 256: 2 warps/SMSP
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * sizeof(double));
  cudaMalloc(&cyc, sizeof(long long));
  const char* names[] = {"DFMA", "DMUL", "DADD", "gibbs sweep (4 fp64)", "SHFL f64 + DADD",
                         "IMAD.WIDE+LOP3", "sweep + 5 stats", "sweep, u from LDS.128",
                         "sweep + lagged stats", "DFMA x8 indep (per op)", "FFMA x8 indep (per op)",
                         "sweep, LDS ring4, STS/step", "sweep, LDS ring4, lane select"};
  for (int m = 0; m < 13; ++m) {
    if (m == 7 && nthreads > 32) continue;
    long long c = 0;
    for (int rep = 0; rep < 3; ++rep) {
      k_lat<<<1, nthreads>>>(out, cyc, 0.3, m);
      cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    }
    printf("%-22s %7.2f cycles per dependent op/step\n", names[m], (double)c / N);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
