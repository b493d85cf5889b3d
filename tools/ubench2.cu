// ubench2.cu -- which pipe do IMAD.HI and IMAD (low half) use on B200, and do
// they overlap with fp64?  Throughput per SM per clock of independent mixes
// (8-way ILP, 8 CTAs x 256 threads per SM).  DESIGN.md §7 (K5).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ubench2.cu -o /tmp/ubench2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ILP 8
constexpr int kIters = 2048;

// NH IMAD.HI, NL IMAD (lo), NW IMAD.WIDE, ND DFMA per ILP slot per iteration
template <int NH, int NL, int NW, int ND>
__global__ void k_mix(uint32_t* out, double* outd, uint32_t seed) {
  uint32_t a[ILP], b[ILP], c[ILP];
  double d[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) {
    a[i] = seed + threadIdx.x * 7 + i; b[i] = a[i] ^ 0x55; c[i] = a[i] + 3;
    d[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
#pragma unroll
      for (int k = 0; k < NH; ++k) a[i] = __umulhi(a[i], 0xD2511F53u) ^ (uint32_t)k;
#pragma unroll
      for (int k = 0; k < NL; ++k) b[i] = b[i] * 0xCD9E8D57u + (uint32_t)k;
#pragma unroll
      for (int k = 0; k < NW; ++k) {
        const uint64_t p = (uint64_t)0xD2511F53u * c[i];
        c[i] = (uint32_t)(p >> 32) ^ (uint32_t)p;
      }
#pragma unroll
      for (int k = 0; k < ND; ++k) d[i] = __fma_rn(d[i], 0.999999, 1e-7);
    }
  }
  uint32_t s = 0;
  double t = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) { s ^= a[i] ^ b[i] ^ c[i]; t += d[i]; }
  if (s == 0x12345678) out[0] = s;
  if (t == 1234.5) outd[0] = t;
}

template <int NH, int NL, int NW, int ND>
void run(const char* name, uint32_t* u, double* dd, int sms, int clk_khz) {
  const int grid = sms * 8, block = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_mix<NH, NL, NW, ND><<<grid, block>>>(u, dd, 1);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) k_mix<NH, NL, NW, ND><<<grid, block>>>(u, dd, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 3;
  const double iters = (double)grid * block * kIters * ILP;     // thread-iterations
  const double per_clk = iters / (ms * 1e-3) / sms / (clk_khz * 1e3);
  printf("%-34s %7.3f ms  %6.2f iterations/clk/SM  (hi %d lo %d wide %d dfma %d)\n", name, ms,
         per_clk, NH, NL, NW, ND);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t* u; double* d;
  cudaMalloc(&u, 64); cudaMalloc(&d, 64);
  run<0, 0, 0, 1>("dfma", u, d, sms, clk);
  run<1, 0, 0, 0>("imad.hi", u, d, sms, clk);
  run<0, 1, 0, 0>("imad.lo", u, d, sms, clk);
  run<0, 0, 1, 0>("imad.wide", u, d, sms, clk);
  run<1, 0, 0, 2>("imad.hi + 2 dfma", u, d, sms, clk);
  run<0, 1, 0, 2>("imad.lo + 2 dfma", u, d, sms, clk);
  run<0, 0, 1, 2>("imad.wide + 2 dfma", u, d, sms, clk);
  run<1, 1, 0, 0>("imad.hi + imad.lo", u, d, sms, clk);
  run<1, 1, 0, 2>("imad.hi + imad.lo + 2 dfma", u, d, sms, clk);
  run<1, 0, 1, 0>("imad.hi + imad.wide", u, d, sms, clk);
  run<1, 0, 0, 1>("imad.hi + 1 dfma", u, d, sms, clk);
  run<1, 0, 0, 4>("imad.hi + 4 dfma", u, d, sms, clk);
  run<2, 0, 0, 2>("2 imad.hi + 2 dfma", u, d, sms, clk);
  run<2, 2, 0, 4>("2 (hi + lo) + 4 dfma", u, d, sms, clk);
  run<0, 0, 2, 4>("2 wide + 4 dfma", u, d, sms, clk);
  run<0, 0, 1, 4>("1 wide + 4 dfma", u, d, sms, clk);
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
