// philox.cuh -- device primitives of the brng hot path (sm_100a).
//
// Philox4x32-10 block function (the paper's "core engine" producing uniform
// integers, PAPER.md P:L45 / P:L52; contract R-01, R-02) and the exact
// word -> standard-uniform conversions ("standard uniform U[0,1)";
// R-04).  Written for the GPU from the published algorithm; shares nothing
// with oracle/.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace brng {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

// One round: (c0,c1,c2,c3) -> (hi(M1 c2)^c1^k0, lo(M1 c2), hi(M0 c0)^c3^k1, lo(M0 c0)).
// Each 32x32->64 product is one IMAD.WIDE.U32; each 3-way xor one LOP3.
__device__ __forceinline__ uint4 philox_round(uint4 c, uint32_t k0, uint32_t k1) {
  const uint64_t p0 = (uint64_t)kPhiloxM0 * c.x;
  const uint64_t p1 = (uint64_t)kPhiloxM1 * c.z;
  uint4 r;
  r.x = (uint32_t)(p1 >> 32) ^ c.y ^ k0;
  r.y = (uint32_t)p1;
  r.z = (uint32_t)(p0 >> 32) ^ c.w ^ k1;
  r.w = (uint32_t)p0;
  return r;
}

// Philox4x32-10.  The round keys k + r*W are kernel-uniform (the seed is a
// kernel argument), so they live in uniform registers and cost nothing per
// thread.
__device__ __forceinline__ uint4 philox10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    c = philox_round(c, k0 + (uint32_t)r * kPhiloxW0, k1 + (uint32_t)r * kPhiloxW1);
  }
  return c;
}

// Block `pos` of stream `stream` (R-02 counter layout).
__device__ __forceinline__ uint4 philox_block(uint64_t pos, uint64_t stream, uint32_t k0,
                                              uint32_t k1) {
  return philox10(make_uint4((uint32_t)pos, (uint32_t)(pos >> 32), (uint32_t)stream,
                             (uint32_t)(stream >> 32)),
                  k0, k1);
}

// ---- conversions (all exact) ----------------------------------------------
// u24(w) = (w >> 8) * 2^-24, binary32.
__device__ __forceinline__ float u24(uint32_t w) {
  return __uint2float_rn(w >> 8) * 0x1p-24f;
}
// u53(lo, hi) = ((hi*2^32 + lo) >> 11) * 2^-53, binary64.  Computed as
// hi*2^-32 + (lo>>11)*2^-53: both terms exact and the sum exact (53 bits),
// avoiding the slow 64-bit integer -> double conversion.
__device__ __forceinline__ double u53(uint32_t lo, uint32_t hi) {
  return fma((double)(lo >> 11), 0x1p-53, (double)hi * 0x1p-32);
}
// u32d(w) = w * 2^-32, binary64.
__device__ __forceinline__ double u32d(uint32_t w) { return (double)w * 0x1p-32; }

// ---- warp helpers -----------------------------------------------------------
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp-aggregated add of per-thread invalid-sample counts into *err.
__device__ __forceinline__ void flush_errors(unsigned long long* err, uint32_t local) {
  const uint32_t any = __ballot_sync(0xffffffffu, local != 0);
  if (any == 0) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(err, (unsigned long long)local);
}

}  // namespace brng
