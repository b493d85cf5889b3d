// gibbs.cu -- K5/K6/K7: many independent Gibbs chains on the triangle
// (Eq. 1, Fig. 1):
//     x ~ U(0, 1-y);  y ~ U(0, 1-x)      from (x0, y0) = (0.5, 0.5)
// Chain c uses Philox stream stream_id + c and sweep s uses block cursor + s
// (R-15, R-16).  Per chain: mean/var of x and y and cov(x,y) over sweeps
// >= burn_in (R-18); the 256-bin histogram of x goes to a per-CTA shared
// histogram (R-19).  Per-CTA partials are reduced in a fixed order by a
// second small kernel, so totals are deterministic for a given launch shape.
//
// B200 design (measured, tools/ubench.cu + tools/gibbs_lab.cu): the sweep is
// bound by the FMA-heavy pipe, which executes both the 32x32->64 IMAD.WIDE of
// Philox (4 cycles/warp) and every fp64 op (2 cycles/warp).  So:
//   * the parts of Philox that are constant along a chain are hoisted
//     (17 IMAD.WIDE per block instead of 20; the round-1 product is advanced
//     with a 64-bit add), and when all chains of a launch share the high
//     stream word, round 2's M1 product is computed once per sweep for all of
//     them (uniform datapath): 16 per-chain products;
//   * the chain state is kept SCALED by 2^64: X = x 2^64 = fl(fl(1-y) u53 2^64)
//     where u53 2^64 is the Philox word pair with its low 11 bits cleared,
//     converted exactly by one I2F.F64.U64 (XU pipe), and 1-x =
//     fma(X, -2^-64, 1).  Power-of-two scaling commutes with IEEE rounding
//     away from under/overflow (values here are 0 or >= 2^-106 unscaled), so
//     every x, y, sum and fma is bit-identical to the oracle's unscaled
//     arithmetic while saving the two u53 scalings and their shifts;
//   * the histogram bin floor(256 x) = floor(X 2^-56) is read from the bits
//     of X with integer ops (ALU pipe), not fp64;
//   * each thread runs three chains interleaved (ILP) with the round keys in
//     the kernel-parameter constant bank.
// Only IEEE sub/mul/fma are used, with explicit _rn intrinsics so nvcc cannot
// contract them: samples, final states, per-chain statistics and histogram are
// bit-identical to the CPU oracle's.
#include "brng_internal.h"
#include "philox.cuh"

namespace brng {
namespace {

constexpr int kThreads = 256;
#ifndef BRNG_GIBBS_CPT
#define BRNG_GIBBS_CPT 3
#endif
#ifndef BRNG_GIBBS_MINB
#define BRNG_GIBBS_MINB 2
#endif
#ifndef BRNG_GIBBS_UNROLL
#define BRNG_GIBBS_UNROLL 2
#endif
constexpr int kCPT = BRNG_GIBBS_CPT;                      // chains per thread
constexpr int kUnroll = BRNG_GIBBS_UNROLL;                // sweeps per loop iteration
#ifndef BRNG_GIBBS_SMALL_UNROLL
#define BRNG_GIBBS_SMALL_UNROLL 2
#endif
constexpr int kSmallUnroll = BRNG_GIBBS_SMALL_UNROLL;     // small (1 chain/thread) launches
constexpr int kHdr = 16;
constexpr int kTot = kHdr + 256;
constexpr double kScale = 18446744073709551616.0;          // 2^64 (state scale)
constexpr double kInvScale = 5.42101086242752217004e-20;   // 2^-64
constexpr double kInvScale2 = kInvScale * kInvScale;       // 2^-128

struct GibbsArgs {
  uint64_t n_chains, base, stream_id;
  uint32_t n_sweeps, burn_in;   // n_sweeps < 2^23 (host-checked; u32 histogram)
  uint32_t rounds;              // grid-stride rounds (kCPT chains per thread each)
  uint32_t tail_rounds;         // then rounds of one chain per thread (bulk kernel)
  uint32_t rk0[10], rk1[10];    // Philox round keys k + r*W (kernel constants)
  uint32_t c3k1_u;              // UHI launches: hi32(stream) ^ k1, the same for every chain
  const double* x0;
  const double* y0;
  double* out_x;
  double* out_y;
  double* chain_stats;
  double* final_xy;
  double* partials;             // [gridDim.x][kTot]
  unsigned long long* err;
};

// u53(lo, hi) * 2^64 = m * 2^11 with m = (hi:lo) >> 11: clearing the low 11
// bits of the 64-bit word gives a value with <= 53 significant bits, so one
// I2F.F64.U64 converts it exactly (one LOP3, no shifts).
__device__ __forceinline__ double u53_scaled(uint32_t lo, uint32_t hi) {
  return __ull2double_rn(((uint64_t)hi << 32) | (lo & 0xFFFFF800u));
}

// floor(256 x) = floor(X 2^-56) for X = x 2^64 in [0, 2^64): X's integer
// part, exact, by one F2I.U64.F64.TRUNC on the XU pipe; its bits 63..56 are
// the bin (X = 0 and tiny X give 0; a dead chain's NaN converts to 0 and
// counts into the sink).  Shared address of the counter: base | 4 bin, base
// 1024-aligned (a live chain's histogram, or the sink of a dead chain): the
// high word shifted by 22 is 4 bin + 2 stray low bits, cleared by the LOP3
// that ORs the base in.  Round 1 read the bin from the exponent and mantissa
// bits with five ALU operations to stay off the FMA pipe; the conversion is
// the same value with three instructions fewer per chain-sweep and the XU
// pipe has the room: cfg5 181.96 -> 177.17 ms, identical histograms
// (profiles/r02_gibbs_bin.txt).
__device__ __forceinline__ uint32_t bin_addr_scaled(double X, uint32_t base) {
  const uint32_t h64 = (uint32_t)(__double2ull_rz(X) >> 32);
  uint32_t b;
  asm("shr.b32 %0, %1, 22;" : "=r"(b) : "r"(h64));
  return (b & 0x3FCu) | base;
}

// Histogram increment at a 32-bit shared-window address (no return value).
__device__ __forceinline__ void hist_inc(uint32_t saddr) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(saddr) : "memory");
}

// Philox parts constant along a chain segment (stream fixed, high counter
// word fixed), pre-combined with their round keys so that ptxas keeps them in
// registers instead of re-deriving them each sweep:
//   round 1: x = r1x (constant), y = r1y (constant), z = hi(M0 pos_lo) ^ c3k1
//   round 2: x = hi(M1 z) ^ d2, y = lo(M1 z), z = lo(M0 pos_lo) ^ a2, w = b2
// with a2 = hi(M0 r1x) ^ k1', b2 = lo(M0 r1x), d2 = r1y ^ k0'.  Per sweep only
// M0 * pos_lo changes; it is advanced by +M0 (a 64-bit add, no multiply).
struct ChainKey {
  uint32_t c3k1, a2, b2, d2;
};

__device__ __forceinline__ ChainKey chain_key(uint64_t stream, uint32_t pos_hi,
                                              const GibbsArgs& a) {
  ChainKey ck;
  const uint64_t p1 = (uint64_t)kPhiloxM1 * (uint32_t)stream;
  const uint32_t r1x = (uint32_t)(p1 >> 32) ^ pos_hi ^ a.rk0[0];
  const uint32_t r1y = (uint32_t)p1;
  ck.c3k1 = (uint32_t)(stream >> 32) ^ a.rk1[0];
  const uint64_t p0r2 = (uint64_t)kPhiloxM0 * r1x;
  ck.a2 = (uint32_t)(p0r2 >> 32) ^ a.rk1[1];
  ck.b2 = (uint32_t)p0r2;
  ck.d2 = r1y ^ a.rk0[1];
  return ck;
}

// Round keys of rounds 2..9.  With BRNG_GIBBS_KEYREG they are pinned in
// registers (an opaque asm barrier stops ptxas from re-loading them from the
// constant bank every sweep).
#ifndef BRNG_GIBBS_KEYREG
#define BRNG_GIBBS_KEYREG 1
#endif
struct RoundKeys {
  uint32_t k0[8], k1[8];
};
__device__ __forceinline__ RoundKeys load_keys(const GibbsArgs& a) {
  RoundKeys rk;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    rk.k0[r] = a.rk0[r + 2];
    rk.k1[r] = a.rk1[r + 2];
#if BRNG_GIBBS_KEYREG
    asm volatile("" : "+r"(rk.k0[r]), "+r"(rk.k1[r]));
#endif
  }
  return rk;
}

__device__ __forceinline__ uint4 chain_block(const ChainKey& ck, uint64_t p0, const RoundKeys& rk) {
  // rounds 1 and 2 (round 1 is free: its products are chain constants or p0)
  const uint32_t z1 = (uint32_t)(p0 >> 32) ^ ck.c3k1;
  const uint64_t p1 = (uint64_t)kPhiloxM1 * z1;
  uint4 c;
  c.x = (uint32_t)(p1 >> 32) ^ ck.d2;
  c.y = (uint32_t)p1;
  c.z = (uint32_t)p0 ^ ck.a2;
  c.w = ck.b2;
#pragma unroll
  for (int r = 0; r < 8; ++r) c = philox_round(c, rk.k0[r], rk.k1[r]);
  return c;
}

// UHI (every chain of the launch has the same high stream word): round 2's
// M1 product depends only on the sweep, so it is computed once per sweep for
// all chains (uniform datapath) and passed in: 16 per-chain products per
// sweep instead of 17.
__device__ __forceinline__ uint4 chain_block_u(const ChainKey& ck, uint64_t p0, uint64_t p1,
                                               const RoundKeys& rk) {
  uint4 c;
  c.x = (uint32_t)(p1 >> 32) ^ ck.d2;
  c.y = (uint32_t)p1;
  c.z = (uint32_t)p0 ^ ck.a2;
  c.w = ck.b2;
#pragma unroll
  for (int r = 0; r < 8; ++r) c = philox_round(c, rk.k0[r], rk.k1[r]);
  return c;
}

// Per-chain state, scaled: X = x 2^64, Y = y 2^64, S1* = s1 2^64,
// S2*, SXY = s2 2^128.
struct Chain {
  double X, Y, S1X, S2X, S1Y, S2Y, SXY;
  uint64_t c;
  bool live;     // a real chain with a valid start (stores, histogram)
};

// Sweeps [s_begin, s_end) of the thread's kCPT chains.
template <bool STORE, bool STATS, int CPT, int UNROLL, bool UHI>
__device__ __forceinline__ void sweeps(const GibbsArgs& a, const RoundKeys& rk, uint32_t s_begin,
                                       uint32_t s_end, Chain (&ch)[CPT], uint32_t hist_base) {
  uint32_t s = s_begin;
  // -2^-64 multiplied by a 1.0 read from memory: the same constant, but one
  // ptxas keeps in a register instead of rematerialising it with two
  // IMAD.MOVs (FMA pipe) in every unrolled iteration: cfg5 183.5 -> 181.95 ms,
  // identical output (profiles/r02_gibbs_pin.txt)
  const double ninv = -kInvScale * __ldg(&brng_dev::tab::kExp2[0]);
  while (s < s_end) {
    const uint64_t pos = a.base + s;
    const uint32_t pos_lo = (uint32_t)pos;
    const uint64_t room = 0x100000000ull - pos_lo;     // sweeps before lo(pos) wraps
    const uint32_t e = ((uint64_t)(s_end - s) < room) ? s_end : (uint32_t)(s + room);
    ChainKey ck[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k)
      ck[k] = chain_key(a.stream_id + ch[k].c, (uint32_t)(pos >> 32), a);
    uint64_t p0 = (uint64_t)kPhiloxM0 * pos_lo;
#pragma unroll UNROLL
    for (; s < e; ++s) {
      const uint64_t p1u = UHI ? (uint64_t)kPhiloxM1 * ((uint32_t)(p0 >> 32) ^ a.c3k1_u) : 0;
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        Chain& q = ch[k];
        const uint4 w = UHI ? chain_block_u(ck[k], p0, p1u, rk) : chain_block(ck[k], p0, rk);
        // x = fl(fl(1-y) u53)  <=>  X = fl(fl(1-y) u53 2^64),  1-y = fma(Y, -2^-64, 1)
        q.X = __dmul_rn(__fma_rn(q.Y, ninv, 1.0), u53_scaled(w.x, w.y));
        q.Y = __dmul_rn(__fma_rn(q.X, ninv, 1.0), u53_scaled(w.z, w.w));
        if (STORE && q.live) {
          if (a.out_x) a.out_x[(uint64_t)s * a.n_chains + q.c] = __dmul_rn(q.X, kInvScale);
          if (a.out_y) a.out_y[(uint64_t)s * a.n_chains + q.c] = __dmul_rn(q.Y, kInvScale);
        }
        if (STATS) {
          q.S1X = __dadd_rn(q.S1X, q.X); q.S2X = __fma_rn(q.X, q.X, q.S2X);
          q.S1Y = __dadd_rn(q.S1Y, q.Y); q.S2Y = __fma_rn(q.Y, q.Y, q.S2Y);
          q.SXY = __fma_rn(q.X, q.Y, q.SXY);
          // a dead chain (invalid start / padding) counts into the sink
          // histogram hist[256..511], never read
          hist_inc(bin_addr_scaled(q.X, q.live ? hist_base : hist_base + 1024u));
        }
      }
      p0 += kPhiloxM0;
    }
  }
}

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// One round of a CTA: each thread runs CPT chains, chain k of thread t being
// c0 + k * THREADS + t; then their statistics, the fixed-order round sums and
// the histogram drain.
template <bool STORE, int CPT, int THREADS, bool UHI, int KB>
__device__ __forceinline__ void gibbs_round(const GibbsArgs& a, const RoundKeys& rk, uint64_t c0,
                                            uint32_t* hist, double (*red)[8], double (&bins)[KB],
                                            uint32_t& nbad, uint32_t hist_base) {
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  const double n = (double)(a.n_sweeps - a.burn_in);
  const double nm1 = __dsub_rn(n, 1.0);
  Chain ch[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    Chain& q = ch[k];
    q.c = c0 + (uint64_t)k * THREADS + threadIdx.x;
    const bool real = q.c < a.n_chains;
    const double x = (real && a.x0) ? a.x0[q.c] : 0.5;
    const double y = (real && a.y0) ? a.y0[q.c] : 0.5;
    const bool valid = (y >= 0.0) && (y <= 1.0);
    q.live = real && valid;
    nbad += (real && !valid);
    q.X = __dmul_rn(x, kScale);
    q.Y = __dmul_rn(valid ? y : qnan, kScale);
    q.S1X = q.S2X = q.S1Y = q.S2Y = q.SXY = 0.0;
  }
  // one chain per thread (latency-bound small launches, the bulk tail):
  // unroll deeper so the Philox blocks of several sweeps overlap the serial
  // x/y update chain
  constexpr int U = CPT == 1 ? kSmallUnroll : kUnroll;
  sweeps<STORE, false, CPT, U, UHI>(a, rk, 0, a.burn_in, ch, hist_base);
  sweeps<STORE, true, CPT, U, UHI>(a, rk, a.burn_in, a.n_sweeps, ch, hist_base);

  double t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const Chain& q = ch[k];
    if (q.c >= a.n_chains) continue;
    const double s1x = __dmul_rn(q.S1X, kInvScale), s1y = __dmul_rn(q.S1Y, kInvScale);
    const double s2x = __dmul_rn(q.S2X, kInvScale2), s2y = __dmul_rn(q.S2Y, kInvScale2);
    const double sxy = __dmul_rn(q.SXY, kInvScale2);
    const double mx = __ddiv_rn(s1x, n), my = __ddiv_rn(s1y, n);
    const double vx = __ddiv_rn(__dsub_rn(s2x, __dmul_rn(s1x, mx)), nm1);
    const double vy = __ddiv_rn(__dsub_rn(s2y, __dmul_rn(s1y, my)), nm1);
    const double cxy = __ddiv_rn(__dsub_rn(sxy, __dmul_rn(s1x, my)), nm1);
    const double fx = __dmul_rn(q.X, kInvScale), fy = __dmul_rn(q.Y, kInvScale);
    if (a.chain_stats) {
      a.chain_stats[0 * a.n_chains + q.c] = mx;
      a.chain_stats[1 * a.n_chains + q.c] = vx;
      a.chain_stats[2 * a.n_chains + q.c] = my;
      a.chain_stats[3 * a.n_chains + q.c] = vy;
      a.chain_stats[4 * a.n_chains + q.c] = cxy;
    }
    if (a.final_xy) { a.final_xy[q.c] = fx; a.final_xy[a.n_chains + q.c] = fy; }
    if (STORE && !q.live) {             // invalid start: NaN samples (oracle semantics)
      for (uint32_t s = 0; s < a.n_sweeps; ++s) {
        if (a.out_x) a.out_x[(uint64_t)s * a.n_chains + q.c] = qnan;
        if (a.out_y) a.out_y[(uint64_t)s * a.n_chains + q.c] = qnan;
      }
    }
    t[0] += mx; t[1] += vx; t[2] += mx * mx; t[3] += my; t[4] += vy; t[5] += my * my;
    t[6] += cxy; t[7] += mx * my;
  }
  // fixed-order reduction of this round's chain-level sums (warp tree, then
  // lane 0 accumulates across rounds in order)
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double v = warp_sum(t[j]);
    if (lane == 0) red[wid][j] += v;
  }
  // drain the u32 shared histogram every round: a round holds at most
  // THREADS * CPT = 768 chains and the C ABI refuses n_sweeps >= 2^22, so a
  // bin holds < 768 * 2^22 < 2^32 counts by construction
  __syncthreads();
#pragma unroll
  for (int j = 0; j < KB; ++j) {
    bins[j] += (double)hist[threadIdx.x + j * THREADS];
    hist[threadIdx.x + j * THREADS] = 0;
  }
  __syncthreads();
}

// THREADS threads x CPT chains per thread.  The bulk configuration is
// <.., kCPT, kThreads> (kCPT = 3 chains per thread for ILP); small chain counts
// (cfg1: 1024 chains) use one chain per thread in 64-thread CTAs to spread
// the latency-bound chains over more SMs.
// Bulk launches are one full resident wave: a.rounds rounds of CPT chains per
// thread, then a.tail_rounds rounds of ONE chain per thread for the chains
// left over.  The tail is what keeps the wave full when the chain count is
// not a multiple of a wave (strong scaling: 2^24 / 8 GPUs = 9.2 waves): a
// one-chain round costs about a third of a three-chain round, so the last
// partial wave costs its size rounded up to a third, not a whole round.
template <bool STORE, int CPT, int THREADS, bool UHI>
__global__ void __launch_bounds__(THREADS, (THREADS == kThreads ? BRNG_GIBBS_MINB : 1))
gibbs_kernel(GibbsArgs a) {
  constexpr int kW = THREADS / 32;
  constexpr int kBinsPerThread = 256 / THREADS;
  __shared__ __align__(1024) uint32_t hist[512];   // [256..511]: sink for dead chains
  __shared__ double red[kW][8];
  const uint32_t hist_base = (uint32_t)__cvta_generic_to_shared(hist);
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int b = threadIdx.x; b < 512; b += THREADS) hist[b] = 0;
  if (lane < 8) red[wid][lane] = 0.0;
  double bins[kBinsPerThread];                 // bins threadIdx.x + j*THREADS, accumulated
#pragma unroll
  for (int j = 0; j < kBinsPerThread; ++j) bins[j] = 0.0;
  uint32_t nbad = 0;
  const RoundKeys rk = load_keys(a);
  __syncthreads();

  const uint64_t per_round = (uint64_t)gridDim.x * THREADS * CPT;
  for (uint32_t rnd = 0; rnd < a.rounds; ++rnd)
    gibbs_round<STORE, CPT, THREADS, UHI>(
        a, rk, (uint64_t)rnd * per_round + (uint64_t)blockIdx.x * CPT * THREADS, hist, red, bins,
        nbad, hist_base);
  if (CPT > 1) {
    const uint64_t tail0 = (uint64_t)a.rounds * per_round;
    const uint64_t per_tail = (uint64_t)gridDim.x * THREADS;
    for (uint32_t rnd = 0; rnd < a.tail_rounds; ++rnd)
      gibbs_round<STORE, 1, THREADS, UHI>(
          a, rk, tail0 + (uint64_t)rnd * per_tail + (uint64_t)blockIdx.x * THREADS, hist, red,
          bins, nbad, hist_base);
  }

  double* part = a.partials + (uint64_t)blockIdx.x * kTot;
  if (threadIdx.x < 8) {
    double v = 0.0;
    for (int w = 0; w < kW; ++w) v += red[w][threadIdx.x];
    part[threadIdx.x] = v;
  }
#pragma unroll
  for (int j = 0; j < kBinsPerThread; ++j) part[kHdr + threadIdx.x + j * THREADS] = bins[j];
  flush_errors(a.err, nbad);
}

// K7: totals[j] = sum over CTAs of partials[cta][j] in a fixed order: one
// warp per column j, lane l sums rows l, l+32, ... in increasing order, then
// a fixed xor-shuffle tree (deterministic for a launch shape; ~3 us instead
// of the ~22 us of one thread walking all rows with dependent L2 loads).
// accumulate != 0: add to totals (a host-staged call processed in chunks).
constexpr int kRedThreads = 256;
// K7 as a programmatic dependent launch (its launch overlaps the Gibbs
// kernel's tail instead of following it).
#ifndef BRNG_K7_PDL
#define BRNG_K7_PDL 1
#endif
__global__ void __launch_bounds__(kRedThreads) reduce_partials_kernel(const double* partials,
                                                                     uint32_t n_parts,
                                                                     double* totals,
                                                                     double n_chains,
                                                                     double n_samples,
                                                                     int accumulate) {
#if BRNG_K7_PDL
  // launched as a programmatic dependent of the Gibbs kernel: wait here until
  // that grid has completed and its partials are visible
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t j = blockIdx.x * (kRedThreads / 32) + (threadIdx.x >> 5);
  if (j >= (uint32_t)kTot) return;
  double v = 0.0;
  if (j < 8 || j >= kHdr)
    for (uint32_t p = lane; p < n_parts; p += 32) v += partials[(uint64_t)p * kTot + j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane != 0) return;
  if (j == 8) v = n_chains;
  if (j == 9) v = n_samples;
  totals[j] = accumulate ? totals[j] + v : v;
}

constexpr int kSmallThreads = 64;
constexpr int kSmallCPT = 1;

// ---- latency mode (small chain counts, e.g. cfg1) -------------------------
// With few chains a thread-per-chain launch leaves the GPU nearly empty and
// each thread walks its 1000+ sweeps serially.  Here the sweep loop of a chain
// runs with nothing else in its instruction stream:
//  * a CHAIN warp runs kCPW = 4 chains (8 lanes each, redundantly computing
//    the same chain): the dependent update x = (1-y) u, y = (1-x) u' and the
//    five running statistics, 32 sweeps per batch, the uniforms read from a
//    shared row 4 sweeps ahead of use; the first lane of each chain records
//    every sweep's state in a shared row.  Several chains per warp share one
//    instruction stream, so cfg1's 1024 chains need 256 chain warps, fewer
//    than the 592 SM sub-partitions.
//  * its HELPER warp computes the Philox blocks of the next batch (one sweep
//    per lane, every chain of the warp) and, for the previous batch, the
//    histogram and the sample stores.
// The pair meets at one named barrier per batch (double-buffered rows).
// Warp w runs on sub-partition w % 4: chain warps 0, 1 and helpers 2, 3 never
// share one, so Philox's IMAD.WIDEs stay off the chain's FMA-heavy pipe.
// Measured (tools/lat_probe.py, tools/ulat2.cu): the one-warp-
// per-chain kernel with Philox in the chain's own stream took 44 us for cfg1;
// this one ~21 us, the chain itself ~42 cycles/sweep against the 32-cycle
// dependency floor.  Same operations in the same order as the oracle:
// bit-identical samples and statistics (tests compare all launch shapes
// chain by chain).
#ifndef BRNG_LAT_RING
#define BRNG_LAT_RING 4
#endif
#ifndef BRNG_LAT_PAIRS
#define BRNG_LAT_PAIRS 2
#endif
#ifndef BRNG_LAT_CPW
#define BRNG_LAT_CPW 4
#endif
constexpr int kRing = BRNG_LAT_RING;             // uniform lookahead (sweeps)
constexpr int kPairs = BRNG_LAT_PAIRS;           // chain warps per CTA
constexpr int kCPW = BRNG_LAT_CPW;               // chains per chain warp
constexpr int kLPC = 32 / kCPW;                  // lanes per chain
constexpr int kLatThreads = 2 * kPairs * 32;     // + one helper warp each
constexpr int kLatChains = kCPW * kPairs;        // chains per CTA per round

// All 10 rounds (no per-chain hoisting: 32 sweeps per lane-block here).
__device__ __forceinline__ uint4 gibbs_block(uint64_t pos, uint64_t stream, const GibbsArgs& a) {
  uint4 c = make_uint4((uint32_t)pos, (uint32_t)(pos >> 32), (uint32_t)stream,
                       (uint32_t)(stream >> 32));
#pragma unroll
  for (int r = 0; r < 10; ++r) c = philox_round(c, a.rk0[r], a.rk1[r]);
  return c;
}

__device__ __forceinline__ void pair_bar(uint32_t p) {
  asm volatile("bar.sync %0, 64;" ::"r"(p + 1) : "memory");
}

struct WarpChain {
  double X, Y, S1X, S2X, S1Y, S2Y, SXY;
};

// Serial update of one batch: sweeps s0 .. s0+nb-1 with uniforms u[j]; the
// recording lane stores sweep j's scaled (X, Y) in xy[j].  STATS: 1 all
// sweeps, 2 sweeps >= burn_in.  A full batch reads its uniforms kRing sweeps
// ahead through a register ring (ptxas then keeps the loads off the chain's
// path: 37 vs 54 cycles/sweep for all 32 loaded up front, tools/ulat2.cu).
// (Only the full, all-statistics batch is unrolled.)
template <int STATS, bool FULL>
__device__ __forceinline__ void warp_batch(WarpChain& q, const double2* u, double2* xy, bool rec,
                                           uint32_t nb, uint32_t s0, uint32_t burn_in) {
  if (FULL) {
    double2 ring[kRing];
#pragma unroll
    for (int j = 0; j < kRing; ++j) ring[j] = u[j];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double2 uj = ring[j % kRing];
      if (j + kRing < 32) ring[j % kRing] = u[j + kRing];
      q.X = __dmul_rn(__fma_rn(q.Y, -kInvScale, 1.0), uj.x);
      q.Y = __dmul_rn(__fma_rn(q.X, -kInvScale, 1.0), uj.y);
      q.S1X = __dadd_rn(q.S1X, q.X); q.S2X = __fma_rn(q.X, q.X, q.S2X);
      q.S1Y = __dadd_rn(q.S1Y, q.Y); q.S2Y = __fma_rn(q.Y, q.Y, q.S2Y);
      q.SXY = __fma_rn(q.X, q.Y, q.SXY);
      if (rec) xy[j] = make_double2(q.X, q.Y);
    }
  } else {
    for (int j = 0; j < (int)nb; ++j) {
      const double2 uj = u[j];
      q.X = __dmul_rn(__fma_rn(q.Y, -kInvScale, 1.0), uj.x);
      q.Y = __dmul_rn(__fma_rn(q.X, -kInvScale, 1.0), uj.y);
      if (STATS == 1 || s0 + (uint32_t)j >= burn_in) {
        q.S1X = __dadd_rn(q.S1X, q.X); q.S2X = __fma_rn(q.X, q.X, q.S2X);
        q.S1Y = __dadd_rn(q.S1Y, q.Y); q.S2Y = __fma_rn(q.Y, q.Y, q.S2Y);
        q.SXY = __fma_rn(q.X, q.Y, q.SXY);
      }
      if (rec) xy[j] = make_double2(q.X, q.Y);
    }
  }
}

template <bool STORE>
__global__ void __launch_bounds__(kLatThreads) gibbs_lat_kernel(GibbsArgs a) {
  __shared__ __align__(1024) uint32_t hist[512];   // [256..511]: sink for dead chains
  __shared__ double red[kLatChains][8];
  __shared__ double2 su[kPairs][2][kCPW][32];     // [pair][buffer][chain][sweep] uniforms
  __shared__ double2 sxy[kPairs][2][kCPW][32];    // [pair][buffer][chain][sweep] states
  const uint32_t hist_base = (uint32_t)__cvta_generic_to_shared(hist);
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // chain warps first: warp w runs on sub-partition w % 4, so with two pairs
  // the chain warps (0, 1) and their helpers (2, 3) never share one
  const bool helper = wid >= (uint32_t)kPairs;
  const uint32_t p = helper ? wid - kPairs : wid;
  for (int b = threadIdx.x; b < 512; b += kLatThreads) hist[b] = 0;
  if (threadIdx.x < kLatChains * 8) red[threadIdx.x >> 3][threadIdx.x & 7] = 0.0;
  uint32_t nbad = 0;
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  __syncthreads();
  const uint64_t n_pairs = (a.n_chains + kCPW - 1) / kCPW;   // chain groups
  const uint64_t stride = (uint64_t)gridDim.x * kPairs;
  for (uint64_t cp = (uint64_t)blockIdx.x * kPairs + p; cp < n_pairs; cp += stride) {
    const uint64_t c0 = (uint64_t)kCPW * cp;
    if (helper) {
      bool ex[kCPW], lv[kCPW];
      uint32_t hb[kCPW];
#pragma unroll
      for (int h = 0; h < kCPW; ++h) {
        ex[h] = c0 + h < a.n_chains;
        const double y0 = (ex[h] && a.y0) ? a.y0[c0 + h] : 0.5;
        lv[h] = ex[h] && (y0 >= 0.0) && (y0 <= 1.0);
        hb[h] = lv[h] ? hist_base : hist_base + 1024u;
      }
      auto fill = [&](uint32_t s0, uint32_t buf) {
#pragma unroll
        for (int h = 0; h < kCPW; ++h) {
          const uint4 w = gibbs_block(a.base + s0 + lane, a.stream_id + c0 + h, a);
          su[p][buf][h][lane] = make_double2(u53_scaled(w.x, w.y), u53_scaled(w.z, w.w));
        }
      };
      auto record = [&](uint32_t s0, uint32_t buf, uint32_t nb) {
        const uint32_t s = s0 + lane;
#pragma unroll
        for (int h = 0; h < kCPW; ++h) {
          if (!ex[h] || lane >= nb) continue;
          const double2 st = sxy[p][buf][h][lane];
          if (s >= a.burn_in) hist_inc(bin_addr_scaled(st.x, hb[h]));
          if (STORE) {
            const uint64_t o = (uint64_t)s * a.n_chains + c0 + h;
            if (a.out_x) a.out_x[o] = lv[h] ? __dmul_rn(st.x, kInvScale) : qnan;
            if (a.out_y) a.out_y[o] = lv[h] ? __dmul_rn(st.y, kInvScale) : qnan;
          }
        }
      };
      fill(0, 0);
      pair_bar(p);
      uint32_t bb = 0;
      for (uint32_t s0 = 0; s0 < a.n_sweeps; s0 += 32, bb ^= 1) {
        if (s0 + 32 < a.n_sweeps) fill(s0 + 32, bb ^ 1);
        if (s0 >= 32) record(s0 - 32, bb ^ 1, 32);
        pair_bar(p);
      }
      if (a.n_sweeps) {
        const uint32_t sl = (a.n_sweeps - 1) & ~31u;
        record(sl, (sl >> 5) & 1, a.n_sweeps - sl);
      }
    } else {
      const uint32_t h = lane / kLPC;
      const uint64_t c = c0 + h;
      const bool ex = c < a.n_chains;
      const bool rec = (lane % kLPC) == 0;
      const double x0 = (ex && a.x0) ? a.x0[c] : 0.5;
      const double y0 = (ex && a.y0) ? a.y0[c] : 0.5;
      const bool live = ex && (y0 >= 0.0) && (y0 <= 1.0);
      nbad += (rec && ex && !live);
      WarpChain q;
      q.X = __dmul_rn(x0, kScale);
      q.Y = __dmul_rn(live ? y0 : qnan, kScale);
      q.S1X = q.S2X = q.S1Y = q.S2Y = q.SXY = 0.0;
      pair_bar(p);                               // batch 0's uniforms are in
      uint32_t bb = 0;
      for (uint32_t s0 = 0; s0 < a.n_sweeps; s0 += 32, bb ^= 1) {
        const uint32_t nb = a.n_sweeps - s0 < 32u ? a.n_sweeps - s0 : 32u;
        const double2* u = su[p][bb][h];
        double2* xy = sxy[p][bb][h];
        if (nb == 32 && s0 >= a.burn_in)
          warp_batch<1, true>(q, u, xy, rec, nb, s0, a.burn_in);
        else
          warp_batch<2, false>(q, u, xy, rec, nb, s0, a.burn_in);
        pair_bar(p);
      }
      if (ex) {
        const double n = (double)(a.n_sweeps - a.burn_in);
        const double nm1 = __dsub_rn(n, 1.0);
        const double s1x = __dmul_rn(q.S1X, kInvScale), s1y = __dmul_rn(q.S1Y, kInvScale);
        const double s2x = __dmul_rn(q.S2X, kInvScale2), s2y = __dmul_rn(q.S2Y, kInvScale2);
        const double sxy_ = __dmul_rn(q.SXY, kInvScale2);
        const double mx = __ddiv_rn(s1x, n), my = __ddiv_rn(s1y, n);
        const double vx = __ddiv_rn(__dsub_rn(s2x, __dmul_rn(s1x, mx)), nm1);
        const double vy = __ddiv_rn(__dsub_rn(s2y, __dmul_rn(s1y, my)), nm1);
        const double cxy = __ddiv_rn(__dsub_rn(sxy_, __dmul_rn(s1x, my)), nm1);
        if (rec) {
          if (a.chain_stats) {
            a.chain_stats[0 * a.n_chains + c] = mx;
            a.chain_stats[1 * a.n_chains + c] = vx;
            a.chain_stats[2 * a.n_chains + c] = my;
            a.chain_stats[3 * a.n_chains + c] = vy;
            a.chain_stats[4 * a.n_chains + c] = cxy;
          }
          if (a.final_xy) {
            a.final_xy[c] = __dmul_rn(q.X, kInvScale);
            a.final_xy[a.n_chains + c] = __dmul_rn(q.Y, kInvScale);
          }
          double* r = red[kCPW * p + h];
          r[0] += mx; r[1] += vx; r[2] += mx * mx; r[3] += my;
          r[4] += vy; r[5] += my * my; r[6] += cxy; r[7] += mx * my;
        }
      }
    }
  }
  __syncthreads();
  double* part = a.partials + (uint64_t)blockIdx.x * kTot;
  if (threadIdx.x < 8) {
    double v = 0.0;
    for (int w = 0; w < kLatChains; ++w) v += red[w][threadIdx.x];
    part[threadIdx.x] = v;
  }
  for (int b = threadIdx.x; b < 256; b += kLatThreads) part[kHdr + b] = (double)hist[b];
  flush_errors(a.err, nbad);
}


template <typename K>
int occupancy(K kernel, int threads) {
  int v = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kernel, threads, 0) != cudaSuccess ||
      v <= 0)
    v = 1;
  return v;
}
int ctas_per_sm_bulk() {
  static int cached = occupancy(gibbs_kernel<false, kCPT, kThreads, true>, kThreads);
  return cached;
}
int ctas_per_sm_small() {
  static int cached = occupancy(gibbs_kernel<true, kSmallCPT, kSmallThreads, false>, kSmallThreads);
  return cached;
}
int ctas_per_sm_lat() {
  static int cached = occupancy(gibbs_lat_kernel<true>, kLatThreads);
  return cached;
}
// Latency mode (chain/helper warp pairs) for chain counts up to this many per SM:
// below it the chain/helper warp pairs finish sooner than a thread per chain
// (4736 chains: 58 vs 91 us, 9472: 102 vs 91 us; tools/lat_probe.py) (cfg1:
// 1024 chains).
#ifndef BRNG_GIBBS_LAT_PER_SM
#define BRNG_GIBBS_LAT_PER_SM 32
#endif

// Launch shape: `threads` x `cpt` chains per CTA per round, one resident wave
// of CTAs.  Small launches: each thread runs `rounds` rounds so chains divide
// evenly.  Bulk launches: the full wave runs floor(n / wave) three-chain
// rounds, and the remainder in one-chain tail rounds when that is cheaper
// (at most 2 of them, ~2/3 of a round) than one more padded three-chain round.
struct Shape {
  unsigned grid;
  uint32_t rounds, tail_rounds;
  bool small;
};
#ifndef BRNG_GIBBS_TAIL
#define BRNG_GIBBS_TAIL 1
#endif
inline Shape grid_shape(uint64_t n_chains, const Ctx& ctx) {
  Shape sh;
  sh.tail_rounds = 0;
  const uint64_t bulk_wave = (uint64_t)ctx.num_sms * ctas_per_sm_bulk() * kThreads * kCPT;
  sh.small = n_chains < bulk_wave / 2;
  const int threads = sh.small ? kSmallThreads : kThreads;
  const int cpt = sh.small ? kSmallCPT : kCPT;
  const uint64_t max_ctas =
      (uint64_t)ctx.num_sms * (sh.small ? ctas_per_sm_small() : ctas_per_sm_bulk());
  const uint64_t per_round_max = max_ctas * threads * cpt;
  if (!sh.small && BRNG_GIBBS_TAIL && kCPT > 1) {
    const uint64_t full = n_chains / per_round_max;
    const uint64_t rem = n_chains - full * per_round_max;
    const uint64_t per_tail = max_ctas * threads;
    const uint64_t tail = (rem + per_tail - 1) / per_tail;
    if (tail <= 2) {
      sh.grid = (unsigned)max_ctas;
      sh.rounds = (uint32_t)full;
      sh.tail_rounds = (uint32_t)tail;
      return sh;
    }
  }
  const uint64_t r = (n_chains + per_round_max - 1) / per_round_max;
  sh.rounds = (uint32_t)(r ? r : 1);
  const uint64_t per_cta = (uint64_t)sh.rounds * threads * cpt;
  const uint64_t g = (n_chains + per_cta - 1) / per_cta;
  sh.grid = (unsigned)(g ? g : 1);
  return sh;
}

}  // namespace

uint64_t gibbs_wave_chains(const Ctx& ctx) {
  return (uint64_t)ctx.num_sms * ctas_per_sm_bulk() * kThreads * kCPT;
}

// Enough for any launch shape (one resident wave), so chunked calls that
// launch different grids can share the handle's scratch.
size_t gibbs_partials_len(uint64_t /*n_chains*/, const Ctx& ctx) {
  int c = ctas_per_sm_bulk() > ctas_per_sm_small() ? ctas_per_sm_bulk() : ctas_per_sm_small();
  if (ctas_per_sm_lat() > c) c = ctas_per_sm_lat();
  return (size_t)ctx.num_sms * c * kTot;
}

cudaError_t launch_gibbs(uint64_t n_chains, uint64_t n_sweeps, const double* x0,
                         const double* y0, uint64_t burn_in, double* out_x, double* out_y,
                         double* chain_stats, double* final_xy, double* totals,
                         double* partials, uint64_t base, const Ctx& ctx, bool accumulate) {
  GibbsArgs a;
  const Shape sh = grid_shape(n_chains, ctx);
  const unsigned grid = sh.grid;
  const uint32_t rounds = sh.rounds;
  a.n_chains = n_chains; a.base = base; a.stream_id = ctx.stream_id;
  a.n_sweeps = (uint32_t)n_sweeps; a.burn_in = (uint32_t)burn_in; a.rounds = rounds;
  a.tail_rounds = sh.tail_rounds;
  for (int r = 0; r < 10; ++r) {
    a.rk0[r] = ctx.k0 + (uint32_t)r * kPhiloxW0;
    a.rk1[r] = ctx.k1 + (uint32_t)r * kPhiloxW1;
  }
  a.x0 = x0; a.y0 = y0; a.out_x = out_x; a.out_y = out_y; a.chain_stats = chain_stats;
  a.final_xy = final_xy; a.partials = partials; a.err = ctx.err;
  const bool store = out_x != nullptr || out_y != nullptr;
  // every chain's stream (stream_id + c) has the same high word?  (the padding
  // chains of the last round never store or count, so only real ones matter)
#ifndef BRNG_GIBBS_UHI
#define BRNG_GIBBS_UHI 1
#endif
  const bool uhi = BRNG_GIBBS_UHI &&
                   (ctx.stream_id >> 32) == ((ctx.stream_id + (n_chains - 1)) >> 32);
  a.c3k1_u = (uint32_t)(ctx.stream_id >> 32) ^ a.rk1[0];
  unsigned n_parts = grid;
  if (n_chains <= (uint64_t)ctx.num_sms * BRNG_GIBBS_LAT_PER_SM) {
    const uint64_t want = (n_chains + kLatChains - 1) / kLatChains;
    const uint64_t cap = (uint64_t)ctx.num_sms * ctas_per_sm_lat();
    n_parts = (unsigned)(want < cap ? (want ? want : 1) : cap);
    if (store)
      gibbs_lat_kernel<true><<<n_parts, kLatThreads, 0, ctx.stream>>>(a);
    else
      gibbs_lat_kernel<false><<<n_parts, kLatThreads, 0, ctx.stream>>>(a);
  } else if (sh.small) {
    if (store)
      gibbs_kernel<true, kSmallCPT, kSmallThreads, false><<<grid, kSmallThreads, 0, ctx.stream>>>(a);
    else
      gibbs_kernel<false, kSmallCPT, kSmallThreads, false><<<grid, kSmallThreads, 0, ctx.stream>>>(a);
  } else if (uhi) {
    if (store)
      gibbs_kernel<true, kCPT, kThreads, true><<<grid, kThreads, 0, ctx.stream>>>(a);
    else
      gibbs_kernel<false, kCPT, kThreads, true><<<grid, kThreads, 0, ctx.stream>>>(a);
  } else {
    if (store)
      gibbs_kernel<true, kCPT, kThreads, false><<<grid, kThreads, 0, ctx.stream>>>(a);
    else
      gibbs_kernel<false, kCPT, kThreads, false><<<grid, kThreads, 0, ctx.stream>>>(a);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || totals == nullptr) return e;
  const double n_samples = (double)n_chains * (double)(n_sweeps - burn_in);
  const int acc = accumulate ? 1 : 0;
#if BRNG_K7_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((kTot + kRedThreads / 32 - 1) / (kRedThreads / 32));
  cfg.blockDim = dim3(kRedThreads);
  cfg.stream = ctx.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, reduce_partials_kernel, (const double*)partials, n_parts, totals,
                            (double)n_chains, n_samples, acc);
#else
  reduce_partials_kernel<<<(kTot + kRedThreads / 32 - 1) / (kRedThreads / 32), kRedThreads, 0,
                           ctx.stream>>>(partials, n_parts, totals, (double)n_chains, n_samples,
                                         acc);
  return cudaGetLastError();
#endif
}

}  // namespace brng
