// gibbs_lab.cu -- design experiments for the Gibbs sweep loop (K5) on B200.
// Standalone; times variants of the per-sweep loop on 2^24 chains x 256
// sweeps and checks they produce identical final states.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gibbs_lab.cu -o tools/gibbs_lab
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;

struct Args {
  uint32_t rk0[10], rk1[10];
  uint64_t n_chains;
  uint32_t n_sweeps;
  double* fx;
  unsigned* hist_out;
};

__device__ __forceinline__ uint4 rnd(uint4 c, uint32_t k0, uint32_t k1) {
  const uint64_t p0 = (uint64_t)M0 * c.x, p1 = (uint64_t)M1 * c.z;
  return make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ k0, (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ k1,
                    (uint32_t)p0);
}

template <int U53>
__device__ __forceinline__ double u53(uint32_t lo, uint32_t hi) {
  if (U53 == 0) {   // one I2F.F64.U64
    const uint64_t m = (((uint64_t)hi << 32) | lo) >> 11;
    return __dmul_rn(__ull2double_rn(m), 0x1p-53);
  } else if (U53 == 1) {  // two I2F.F64.U32
    return fma((double)(lo >> 11), 0x1p-53, (double)hi * 0x1p-32);
  } else {          // integer bit assembly, no conversion
    const uint32_t mhi = 0x3FF00000u | (hi >> 12);
    const uint32_t mlo = __funnelshift_r(lo, hi, 12);
    const double a = __dsub_rn(__hiloint2double(mhi, mlo), 1.0);
    const double b = __hiloint2double((lo & 0x800u) ? 0x3CA00000u : 0u, 0u);
    return __dadd_rn(a, b);
  }
}

__device__ __forceinline__ uint32_t bin256(double x) {
  return ((uint32_t)__double2hiint(__dadd_rz(x, 1.0)) >> 12) & 255u;
}

// C chains per thread interleaved; HIST: 0 none, 1 per-CTA smem atomics
template <int C, int U53, int HIST, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) lab(Args a) {
  __shared__ unsigned hist[256];
  for (int i = threadIdx.x; i < 256; i += THREADS) hist[i] = 0;
  __syncthreads();
  const uint64_t base_c = ((uint64_t)blockIdx.x * THREADS + threadIdx.x) * C;
  double x[C], y[C], s1[C], s2[C];
  uint32_t r1x[C], r1y[C], c3k1[C];
  uint64_t p0r2[C];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    const uint64_t stream = base_c + k;
    const uint64_t p1 = (uint64_t)M1 * (uint32_t)stream;
    r1x[k] = (uint32_t)(p1 >> 32) ^ a.rk0[0];
    r1y[k] = (uint32_t)p1;
    c3k1[k] = (uint32_t)(stream >> 32) ^ a.rk1[0];
    p0r2[k] = (uint64_t)M0 * r1x[k];
    x[k] = 0.5; y[k] = 0.5; s1[k] = 0; s2[k] = 0;
  }
  uint64_t p0 = 0;
#pragma unroll 2
  for (uint32_t s = 0; s < a.n_sweeps; ++s) {
#pragma unroll
    for (int k = 0; k < C; ++k) {
      uint4 c = make_uint4(r1x[k], r1y[k], (uint32_t)(p0 >> 32) ^ c3k1[k], (uint32_t)p0);
      {
        const uint64_t p1 = (uint64_t)M1 * c.z;
        c = make_uint4((uint32_t)(p1 >> 32) ^ c.y ^ a.rk0[1], (uint32_t)p1,
                       (uint32_t)(p0r2[k] >> 32) ^ c.w ^ a.rk1[1], (uint32_t)p0r2[k]);
      }
#pragma unroll
      for (int r = 2; r < 10; ++r) c = rnd(c, a.rk0[r], a.rk1[r]);
      x[k] = __dmul_rn(__dsub_rn(1.0, y[k]), u53<U53>(c.x, c.y));
      y[k] = __dmul_rn(__dsub_rn(1.0, x[k]), u53<U53>(c.z, c.w));
      s1[k] = __dadd_rn(s1[k], x[k]);
      s2[k] = fma(x[k], x[k], s2[k]);
      if (HIST) atomicAdd(&hist[bin256(x[k])], 1u);
    }
    p0 += M0;
  }
#pragma unroll
  for (int k = 0; k < C; ++k) a.fx[base_c + k] = x[k] + 1e-300 * (s1[k] + s2[k]);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += THREADS) atomicAdd(&a.hist_out[i], hist[i]);
}

template <int C, int U53, int HIST, int THREADS, int MINB>
void run(const char* name, Args a, std::vector<double>& ref) {
  const unsigned grid = (unsigned)(a.n_chains / (THREADS * C));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lab<C, U53, HIST, THREADS, MINB>, THREADS, 0);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, lab<C, U53, HIST, THREADS, MINB>);
  cudaMemset(a.hist_out, 0, 1024);
  lab<C, U53, HIST, THREADS, MINB><<<grid, THREADS>>>(a);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  lab<C, U53, HIST, THREADS, MINB><<<grid, THREADS>>>(a);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  std::vector<double> fx(a.n_chains);
  cudaMemcpy(fx.data(), a.fx, 8 * a.n_chains, cudaMemcpyDeviceToHost);
  bool same = true;
  if (ref.empty()) ref = fx; else for (size_t i = 0; i < fx.size(); ++i) same &= (fx[i] == ref[i]);
  const double sweeps = (double)a.n_chains * a.n_sweeps;
  printf("%-34s regs=%3d occ=%2d CTA/SM  %8.3f ms  %7.1f Gsweeps/s  %s\n", name, fa.numRegs, occ,
         ms, sweeps / ms / 1e6, same ? "same" : "DIFFERENT");
}

int main() {
  Args a;
  for (int r = 0; r < 10; ++r) { a.rk0[r] = 42u + r * W0; a.rk1[r] = 0u + r * W1; }
  a.n_chains = 1ull << 24;
  a.n_sweeps = 256;
  cudaMalloc(&a.fx, 8 * a.n_chains);
  cudaMalloc(&a.hist_out, 1024);
  std::vector<double> ref;
  run<1, 0, 1, 256, 4>("C1 i2f64 hist 256x4", a, ref);
  run<1, 0, 0, 256, 4>("C1 i2f64 nohist 256x4", a, ref);
  run<1, 1, 1, 256, 4>("C1 2xi2f32 hist 256x4", a, ref);
  run<1, 2, 1, 256, 4>("C1 bits hist 256x4", a, ref);
  run<1, 0, 1, 256, 3>("C1 i2f64 hist 256x3", a, ref);
  run<1, 0, 1, 128, 8>("C1 i2f64 hist 128x8", a, ref);
  run<1, 0, 1, 256, 5>("C1 i2f64 hist 256x5", a, ref);
  run<1, 0, 1, 256, 6>("C1 i2f64 hist 256x6", a, ref);
  run<2, 0, 1, 256, 2>("C2 i2f64 hist 256x2", a, ref);
  run<2, 0, 1, 256, 3>("C2 i2f64 hist 256x3", a, ref);
  run<2, 2, 1, 256, 3>("C2 bits hist 256x3", a, ref);
  run<4, 0, 1, 128, 2>("C4 i2f64 hist 128x2", a, ref);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
