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

// Round keys k + r W (mod 2^32) of the 10 rounds, computed on the host and
// passed in a __grid_constant__ kernel argument: the LOP3s of every round then
// read them straight from the constant bank (no per-block key schedule, no
// registers).  Bit-identical to philox_block(pos, stream, k0, k1).
struct RoundKeys {
  uint32_t k0[10], k1[10];
};
inline RoundKeys make_round_keys(uint32_t k0, uint32_t k1) {
  RoundKeys rk;
  for (int r = 0; r < 10; ++r) {
    rk.k0[r] = k0 + (uint32_t)r * kPhiloxW0;
    rk.k1[r] = k1 + (uint32_t)r * kPhiloxW1;
  }
  return rk;
}
__device__ __forceinline__ uint4 philox_block_rk(uint64_t pos, uint64_t stream,
                                                 const RoundKeys& rk) {
  uint4 c = make_uint4((uint32_t)pos, (uint32_t)(pos >> 32), (uint32_t)stream,
                       (uint32_t)(stream >> 32));
#pragma unroll
  for (int r = 0; r < 10; ++r) c = philox_round(c, rk.k0[r], rk.k1[r]);
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
