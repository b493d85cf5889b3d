// ubench3.cu -- a Philox-like mix on B200: two 32x32->64 products whose both
// halves are used (as in a Philox round) plus fp64 FMAs (the Gibbs sweep's
// ratio is 16 products : 9 fp64), with the products as IMAD.WIDE or as
// IMAD.HI + a low IMAD kept unfused by an opaque operand.  Iterations per
// clock per SM.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ubench3.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ILP 6
constexpr int kIters = 2048;

template <bool SPLIT, int ND>
__global__ void k(uint32_t* out, double* outd, uint32_t seed, uint32_t zero) {
  uint32_t x[ILP], y[ILP], z[ILP], w[ILP];
  double d[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    x[i] = seed + threadIdx.x * 7 + i; y[i] = x[i] ^ 0x55; z[i] = x[i] + 3; w[i] = x[i] * 5;
    d[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      uint32_t h0, l0, h1, l1;
      if (SPLIT) {
        h0 = __umulhi(x[i], 0xD2511F53u); l0 = (x[i] ^ zero) * 0xD2511F53u;
        h1 = __umulhi(z[i], 0xCD9E8D57u); l1 = (z[i] ^ zero) * 0xCD9E8D57u;
      } else {
        const uint64_t p0 = (uint64_t)0xD2511F53u * x[i], p1 = (uint64_t)0xCD9E8D57u * z[i];
        h0 = (uint32_t)(p0 >> 32); l0 = (uint32_t)p0; h1 = (uint32_t)(p1 >> 32); l1 = (uint32_t)p1;
      }
      const uint32_t nx = h1 ^ y[i] ^ (0x9E3779B9u + it), nz = h0 ^ w[i] ^ 0xBB67AE85u;
      y[i] = l1; w[i] = l0; x[i] = nx; z[i] = nz;
#pragma unroll
      for (int k2 = 0; k2 < ND; ++k2) d[i] = __fma_rn(d[i], 0.999999, 1e-7);
    }
  }
  uint32_t s = 0; double t = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) { s ^= x[i] ^ y[i] ^ z[i] ^ w[i]; t += d[i]; }
  if (s == 0x12345678) out[0] = s;
  if (t == 1234.5) outd[0] = t;
}

template <bool SPLIT, int ND>
void run(const char* name, uint32_t* u, double* dd, int sms, int clk_khz) {
  const int grid = sms * 8, block = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<SPLIT, ND><<<grid, block>>>(u, dd, 1, 0);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) k<SPLIT, ND><<<grid, block>>>(u, dd, 1, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 3;
  const double iters = (double)grid * block * kIters * ILP;
  printf("%-28s %8.3f ms  %7.2f iterations/clk/SM (2 products + %d dfma each)\n", name, ms,
         iters / (ms * 1e-3) / sms / (clk_khz * 1e3), ND);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  uint32_t* u; double* dd;
  cudaMalloc(&u, 64); cudaMalloc(&dd, 64);
  run<false, 0>("wide, 0 dfma", u, dd, sms, clk);
  run<true, 0>("hi+lo, 0 dfma", u, dd, sms, clk);
  run<false, 1>("wide, 1 dfma", u, dd, sms, clk);
  run<true, 1>("hi+lo, 1 dfma", u, dd, sms, clk);
  run<false, 2>("wide, 2 dfma", u, dd, sms, clk);
  run<true, 2>("hi+lo, 2 dfma", u, dd, sms, clk);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
