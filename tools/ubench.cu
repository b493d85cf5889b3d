// ubench.cu -- throughput microbenchmarks for the instruction mix of the brng
// kernels on B200.  Standalone: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a tools/ubench.cu -o ubench && ./ubench
// Prints, per op: thread-ops per clock per SM at the measured SM clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ILP 8
constexpr int kIters = 4096;

__global__ void k_imad_wide(uint32_t* out, uint32_t seed) {
  uint32_t a[ILP], b[ILP];
  for (int i = 0; i < ILP; ++i) { a[i] = seed + threadIdx.x * 7 + i; b[i] = a[i] ^ 0x55; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      uint64_t p = (uint64_t)0xD2511F53u * a[i];
      a[i] = (uint32_t)(p >> 32) ^ b[i];
      b[i] = (uint32_t)p;
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < ILP; ++i) s ^= a[i] ^ b[i];
  if (s == 0x12345678) out[0] = s;
}

__global__ void k_imad_hilo(uint32_t* out, uint32_t seed) {
  uint32_t a[ILP], b[ILP];
  for (int i = 0; i < ILP; ++i) { a[i] = seed + threadIdx.x * 7 + i; b[i] = a[i] ^ 0x55; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      uint32_t hi, lo;
      asm volatile("mul.hi.u32 %0, %1, 0xD2511F53;" : "=r"(hi) : "r"(a[i]));
      asm volatile("mul.lo.u32 %0, %1, 0xD2511F53;" : "=r"(lo) : "r"(a[i]));
      a[i] = hi ^ b[i];
      b[i] = lo;
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < ILP; ++i) s ^= a[i] ^ b[i];
  if (s == 0x12345678) out[0] = s;
}

__global__ void k_lop3(uint32_t* out, uint32_t seed) {
  uint32_t a[ILP], b[ILP];
  for (int i = 0; i < ILP; ++i) { a[i] = seed + threadIdx.x * 7 + i; b[i] = a[i] ^ 0x55; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      a[i] = a[i] ^ b[i] ^ (0x9E3779B9u + it);
      b[i] = b[i] ^ a[i] ^ 0xBB67AE85u;
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < ILP; ++i) s ^= a[i] ^ b[i];
  if (s == 0x12345678) out[0] = s;
}

__global__ void k_dfma(double* out, double seed) {
  double a[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = seed + threadIdx.x + i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], 0.999999, 1e-9);
  }
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}

__global__ void k_i2f64(double* out, uint32_t seed) {
  uint32_t a[ILP];
  double acc[ILP];
  for (int i = 0; i < ILP; ++i) { a[i] = seed + threadIdx.x * 7 + i; acc[i] = 0; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      acc[i] = (double)(a[i] + it);
    }
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] ^= (uint32_t)__double2loint(acc[i]);
  }
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 1.2345) out[0] = s;
}

__global__ void k_atoms(uint32_t* out, uint32_t seed) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  uint32_t x = seed + threadIdx.x * 2654435761u;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      x = x * 1664525u + 1013904223u;
      atomicAdd(&h[x >> 24], 1u);
    }
  }
  __syncthreads();
  if (h[threadIdx.x] == 0x12345678) out[0] = 1;
}


// mixes: does fp64 / LOP3 / I2F share a pipe with IMAD.WIDE?
template <int ND, int NL>
__global__ void k_mix(uint32_t* out, uint32_t seed) {
  uint32_t a[ILP], b[ILP];
  double d[ILP];
  for (int i = 0; i < ILP; ++i) { a[i] = seed + threadIdx.x * 7 + i; b[i] = a[i] ^ 0x55; d[i] = a[i]; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      uint64_t p = (uint64_t)0xD2511F53u * a[i];
      a[i] = (uint32_t)(p >> 32);
      b[i] = (uint32_t)p ^ b[i];
#pragma unroll
      for (int j = 0; j < NL; ++j) b[i] = b[i] ^ a[i] ^ (0x9E3779B9u * (j + 1));
#pragma unroll
      for (int j = 0; j < ND; ++j) d[i] = fma(d[i], 0.999999, 1e-9);
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < ILP; ++i) s ^= a[i] ^ b[i] ^ (uint32_t)__double2loint(d[i]);
  if (s == 0x12345678) out[0] = s;
}

__global__ void k_i2f64u64(double* out, uint32_t seed) {
  uint64_t a[ILP];
  double acc[ILP];
  for (int i = 0; i < ILP; ++i) { a[i] = seed + threadIdx.x * 7 + i; acc[i] = 0; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = (double)((a[i] + it) >> 11);
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] ^= (uint64_t)__double2loint(acc[i]);
  }
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 1.2345) out[0] = s;
}


__global__ void k_imad_hi(uint32_t* out, uint32_t seed) {
  uint32_t a[ILP], b[ILP];
  for (int i = 0; i < ILP; ++i) { a[i] = seed + threadIdx.x * 7 + i; b[i] = a[i] ^ 0x55; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = __umulhi(a[i], 0xD2511F53u) ^ b[i];
  }
  uint32_t s = 0;
  for (int i = 0; i < ILP; ++i) s ^= a[i];
  if (s == 0x12345678) out[0] = s;
}
__global__ void k_imad_lo(uint32_t* out, uint32_t seed) {
  uint32_t a[ILP], b[ILP];
  for (int i = 0; i < ILP; ++i) { a[i] = seed + threadIdx.x * 7 + i; b[i] = a[i] ^ 0x55; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = (a[i] * 0xD2511F53u) ^ b[i];
  }
  uint32_t s = 0;
  for (int i = 0; i < ILP; ++i) s ^= a[i];
  if (s == 0x12345678) out[0] = s;
}
// hi via IMAD.HI and lo via IMAD on a register copy the compiler cannot merge
__global__ void k_imad_split(uint32_t* out, uint32_t seed, uint32_t zero) {
  uint32_t a[ILP], b[ILP];
  for (int i = 0; i < ILP; ++i) { a[i] = seed + threadIdx.x * 7 + i; b[i] = a[i] ^ 0x55; }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      const uint32_t hi = __umulhi(a[i], 0xD2511F53u);
      const uint32_t lo = (a[i] ^ zero) * 0xD2511F53u;
      a[i] = hi ^ b[i];
      b[i] = lo;
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < ILP; ++i) s ^= a[i] ^ b[i];
  if (s == 0x12345678) out[0] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 3;
}

int main() {
  int sms, clk_khz;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  uint32_t* u; double* d;
  cudaMalloc(&u, 64); cudaMalloc(&d, 64);
  const int grid = sms * 8, block = 256;
  const double threads = (double)grid * block;
  auto report = [&](const char* name, float ms, double ops_per_iter) {
    const double ops = threads * kIters * ops_per_iter;
    const double per_s = ops / (ms * 1e-3);
    printf("%-14s %8.3f ms  %10.1f Gop/s  %6.1f ops/clk/SM @%d MHz\n", name, ms, per_s / 1e9,
           per_s / sms / (clk_khz * 1e3), clk_khz / 1000);
  };
  report("imad.wide", timeit([&] { k_imad_wide<<<grid, block>>>(u, 1); }), ILP);
  report("imad.hi+lo", timeit([&] { k_imad_hilo<<<grid, block>>>(u, 1); }), ILP);
  report("lop3 x2", timeit([&] { k_lop3<<<grid, block>>>(u, 1); }), 2 * ILP);
  report("dfma", timeit([&] { k_dfma<<<grid, block>>>(d, 1.0); }), ILP);
  report("i2f.f64", timeit([&] { k_i2f64<<<grid, block>>>(d, 1); }), ILP);
  report("atoms", timeit([&] { k_atoms<<<grid, block>>>(u, 1); }), ILP);
  report("i2f.f64.u64", timeit([&] { k_i2f64u64<<<grid, block>>>(d, 1); }), ILP);
  report("wide+0d+0l", timeit([&] { k_mix<0, 0><<<grid, block>>>(u, 1); }), ILP);
  report("wide+2d (wide)", timeit([&] { k_mix<2, 0><<<grid, block>>>(u, 1); }), ILP);
  report("wide+4d (wide)", timeit([&] { k_mix<4, 0><<<grid, block>>>(u, 1); }), ILP);
  report("wide+4l (wide)", timeit([&] { k_mix<0, 4><<<grid, block>>>(u, 1); }), ILP);
  report("wide+2d+4l", timeit([&] { k_mix<2, 4><<<grid, block>>>(u, 1); }), ILP);
  report("imad.hi", timeit([&] { k_imad_hi<<<grid, block>>>(u, 1); }), ILP);
  report("imad.lo", timeit([&] { k_imad_lo<<<grid, block>>>(u, 1); }), ILP);
  report("imad split", timeit([&] { k_imad_split<<<grid, block>>>(u, 1, 0); }), ILP);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
