// curand_xcheck.cu -- test-only: Philox4x32-10 blocks from cuRAND's device
// generator, an implementation independent of brng's (SURVEY.md §4 tier 2:
// "cuRAND-device cross-check of K1 raw words").  curand_init(seed,
// subsequence = stream, offset = 4 * pos) positions the generator at word 0
// of block `pos` of that stream; curand4 returns the block's four words.
#include <cstdint>
#include <curand_kernel.h>

__global__ void k_curand_blocks(uint64_t seed, uint64_t stream, uint64_t base, uint64_t n,
                                uint32_t* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  curandStatePhilox4_32_10_t st;
  curand_init(seed, stream, 4 * (base + i), &st);
  const uint4 w = curand4(&st);
  out[4 * i + 0] = w.x;
  out[4 * i + 1] = w.y;
  out[4 * i + 2] = w.z;
  out[4 * i + 3] = w.w;
}

extern "C" int curand_blocks(uint64_t seed, uint64_t stream, uint64_t base, uint64_t n,
                             uint32_t* out, void* s) {
  k_curand_blocks<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)s>>>(seed, stream, base,
                                                                          n, out);
  return (int)cudaGetLastError();
}
