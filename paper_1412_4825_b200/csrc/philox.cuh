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

#include "../../include/brng_device.cuh"

namespace brng {

// The primitives are the public device API's (include/brng_device.cuh), so
// the bulk kernels and user kernels calling brng_dev:: getters produce the
// same values.
using brng_dev::kPhiloxM0;
using brng_dev::kPhiloxM1;
using brng_dev::kPhiloxW0;
using brng_dev::kPhiloxW1;
using brng_dev::philox10;
using brng_dev::philox_block;
using brng_dev::philox_round;
using brng_dev::u24;
using brng_dev::u32d;
using brng_dev::u53;

// Round keys k + r W (mod 2^32) of the 10 rounds, and the round-1 terms that
// depend only on the launch's stream, computed on the host and passed in a
// __grid_constant__ kernel argument: the LOP3s of every round read them from
// the constant bank (no per-block key schedule, no registers), and round 1
// needs one multiply instead of two.  Round 1 of counter (pos_lo, pos_hi,
// s_lo, s_hi): x = hi(M1 s_lo) ^ pos_hi ^ k0, y = lo(M1 s_lo),
// z = hi(M0 pos_lo) ^ s_hi ^ k1, w = lo(M0 pos_lo).
// Bit-identical to philox_block(pos, stream, k0, k1).
struct RoundKeys {
  uint32_t k0[10], k1[10];
  uint32_t r1x, r1y, r1z;   // hi(M1 s_lo) ^ k0, lo(M1 s_lo), s_hi ^ k1
};
inline RoundKeys make_round_keys(uint32_t k0, uint32_t k1, uint64_t stream) {
  RoundKeys rk;
  for (int r = 0; r < 10; ++r) {
    rk.k0[r] = k0 + (uint32_t)r * kPhiloxW0;
    rk.k1[r] = k1 + (uint32_t)r * kPhiloxW1;
  }
  const uint64_t p1 = (uint64_t)kPhiloxM1 * (uint32_t)stream;
  rk.r1x = (uint32_t)(p1 >> 32) ^ k0;
  rk.r1y = (uint32_t)p1;
  rk.r1z = (uint32_t)(stream >> 32) ^ k1;
  return rk;
}
// Block `pos` of the stream rk was made for.
__device__ __forceinline__ uint4 philox_block_rk(uint64_t pos, const RoundKeys& rk) {
  const uint64_t p0 = (uint64_t)kPhiloxM0 * (uint32_t)pos;
  uint4 c;
  c.x = rk.r1x ^ (uint32_t)(pos >> 32);
  c.y = rk.r1y;
  c.z = (uint32_t)(p0 >> 32) ^ rk.r1z;
  c.w = (uint32_t)p0;
#pragma unroll
  for (int r = 1; r < 10; ++r) c = philox_round(c, rk.k0[r], rk.k1[r]);
  return c;
}

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
