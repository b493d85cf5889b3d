// gibbs.cu -- K5/K6/K7: many independent Gibbs chains on the triangle
// (Eq. 1, Fig. 1):
//     x ~ U(0, 1-y);  y ~ U(0, 1-x)      from (x0, y0) = (0.5, 0.5)
// One chain per thread, (x, y) and the running sums in registers; chain c uses
// Philox stream stream_id + c and sweep s uses block cursor + s (R-15, R-16).
// Per chain: mean/var of x and y and cov(x,y) over sweeps >= burn_in (R-18);
// the 256-bin histogram of x goes to a per-CTA shared-memory histogram
// (R-19).  Per-CTA partials are reduced in a fixed order by a second small
// kernel, so totals are deterministic for a given launch shape.
//
// Only IEEE sub/mul/fma appear in the chain and the statistics, written with
// explicit round-to-nearest intrinsics so nvcc cannot contract them: the
// samples, final states, per-chain statistics and histogram are bit-identical
// to the CPU oracle's.
#include "brng_internal.h"
#include "philox.cuh"

namespace brng {
namespace {

constexpr int kThreads = 256;
constexpr int kHdr = 16;
constexpr int kTot = kHdr + 256;

struct GibbsArgs {
  uint64_t n_chains, n_sweeps, burn_in, base, stream_id;
  uint32_t k0, k1;
  uint32_t rounds;            // grid-stride rounds per thread
  const double* x0;
  const double* y0;
  double* out_x;
  double* out_y;
  double* chain_stats;
  double* final_xy;
  double* partials;           // [gridDim.x][kTot]
  unsigned long long* err;
};

// floor(256 x) for x in [0, 1): 2^52 + 256 x rounded toward zero keeps the
// integer part in the low mantissa bits (exact; no F2I conversion).
__device__ __forceinline__ uint32_t bin256(double x) {
  return (uint32_t)__double2loint(__fma_rz(x, 256.0, 0x1p52)) & 255u;
}

// Philox4x32-10 of block (pos_lo, pos_hi) of a chain's stream with the parts
// that are invariant along the chain hoisted by the caller:
//   r1y  = lo(M1 * stream_lo)                     (round 1, word 1)
//   r1x  = hi(M1 * stream_lo) ^ pos_hi ^ k0       (round 1, word 0)
//   p0r2 = M0 * r1x                               (round 2, first product)
//   c3k1 = stream_hi ^ k1
// Only pos_lo varies per sweep (and it is warp-uniform).
struct ChainKey {
  uint32_t r1x, r1y, c3k1;
  uint64_t p0r2;
};

__device__ __forceinline__ ChainKey chain_key(uint64_t stream, uint32_t pos_hi, uint32_t k0,
                                              uint32_t k1) {
  ChainKey ck;
  const uint64_t p1 = (uint64_t)kPhiloxM1 * (uint32_t)stream;
  ck.r1x = (uint32_t)(p1 >> 32) ^ pos_hi ^ k0;
  ck.r1y = (uint32_t)p1;
  ck.c3k1 = (uint32_t)(stream >> 32) ^ k1;
  ck.p0r2 = (uint64_t)kPhiloxM0 * ck.r1x;
  return ck;
}

__device__ __forceinline__ uint4 chain_block(const ChainKey& ck, uint32_t pos_lo, uint32_t k0,
                                             uint32_t k1) {
  // round 1
  const uint64_t p0 = (uint64_t)kPhiloxM0 * pos_lo;
  uint4 c;
  c.x = ck.r1x;
  c.y = ck.r1y;
  c.z = (uint32_t)(p0 >> 32) ^ ck.c3k1;
  c.w = (uint32_t)p0;
  // round 2 (first product hoisted)
  {
    const uint32_t kk0 = k0 + kPhiloxW0, kk1 = k1 + kPhiloxW1;
    const uint64_t p1 = (uint64_t)kPhiloxM1 * c.z;
    uint4 r;
    r.x = (uint32_t)(p1 >> 32) ^ c.y ^ kk0;
    r.y = (uint32_t)p1;
    r.z = (uint32_t)(ck.p0r2 >> 32) ^ c.w ^ kk1;
    r.w = (uint32_t)ck.p0r2;
    c = r;
  }
#pragma unroll
  for (int r = 2; r < 10; ++r)
    c = philox_round(c, k0 + (uint32_t)r * kPhiloxW0, k1 + (uint32_t)r * kPhiloxW1);
  return c;
}

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

__global__ void __launch_bounds__(kThreads, 4) gibbs_kernel(GibbsArgs a) {
  __shared__ uint32_t hist[256];
  __shared__ double red[kThreads / 32][8];
  __shared__ double tot_s[8][kThreads];        // per-thread chain-level sums
  hist[threadIdx.x] = 0;                       // kThreads == 256 bins
#pragma unroll
  for (int j = 0; j < 8; ++j) tot_s[j][threadIdx.x] = 0.0;
  double bins = 0.0;                           // this thread's bin, accumulated
  uint32_t nbad = 0;
  __syncthreads();

  const uint64_t total_threads = (uint64_t)gridDim.x * kThreads;
  for (uint32_t rnd = 0; rnd < a.rounds; ++rnd) {
    const uint64_t c = (uint64_t)rnd * total_threads + (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    if (c < a.n_chains) {
      double x = a.x0 ? a.x0[c] : 0.5;
      double y = a.y0 ? a.y0[c] : 0.5;
      const bool valid = (y >= 0.0) && (y <= 1.0);
      if (!valid) { x = __longlong_as_double(0x7ff8000000000000ll); y = x; ++nbad; }
      const uint64_t stream = a.stream_id + c;
      double s1x = 0.0, s2x = 0.0, s1y = 0.0, s2y = 0.0, sxy = 0.0;
      uint64_t s = 0;
      while (s < a.n_sweeps) {
        // segment of sweeps with a constant high counter word
        const uint64_t pos = a.base + s;
        const uint32_t pos_hi = (uint32_t)(pos >> 32);
        const uint64_t room = 0x100000000ull - (uint32_t)pos;
        const uint64_t seg_end = (a.n_sweeps - s < room) ? a.n_sweeps : s + room;
        const ChainKey ck = chain_key(stream, pos_hi, a.k0, a.k1);
        for (; s < seg_end; ++s) {
          const uint4 w = chain_block(ck, (uint32_t)(a.base + s), a.k0, a.k1);
          x = __dmul_rn(__dsub_rn(1.0, y), u53(w.x, w.y));   // x ~ U(0, 1-y)
          y = __dmul_rn(__dsub_rn(1.0, x), u53(w.z, w.w));   // y ~ U(0, 1-x)
          if (a.out_x) a.out_x[s * a.n_chains + c] = x;
          if (a.out_y) a.out_y[s * a.n_chains + c] = y;
          if (s >= a.burn_in) {
            s1x = __dadd_rn(s1x, x); s2x = fma(x, x, s2x);
            s1y = __dadd_rn(s1y, y); s2y = fma(y, y, s2y);
            sxy = fma(x, y, sxy);
            if (valid) atomicAdd(&hist[bin256(x)], 1u);
          }
        }
      }
      const double n = (double)(a.n_sweeps - a.burn_in);
      const double nm1 = __dsub_rn(n, 1.0);
      const double mx = __ddiv_rn(s1x, n), my = __ddiv_rn(s1y, n);
      const double vx = __ddiv_rn(__dsub_rn(s2x, __dmul_rn(s1x, mx)), nm1);
      const double vy = __ddiv_rn(__dsub_rn(s2y, __dmul_rn(s1y, my)), nm1);
      const double cxy = __ddiv_rn(__dsub_rn(sxy, __dmul_rn(s1x, my)), nm1);
      if (a.chain_stats) {
        a.chain_stats[0 * a.n_chains + c] = mx;
        a.chain_stats[1 * a.n_chains + c] = vx;
        a.chain_stats[2 * a.n_chains + c] = my;
        a.chain_stats[3 * a.n_chains + c] = vy;
        a.chain_stats[4 * a.n_chains + c] = cxy;
      }
      if (a.final_xy) { a.final_xy[c] = x; a.final_xy[a.n_chains + c] = y; }
      double* t = &tot_s[0][threadIdx.x];
      t[0 * kThreads] += mx; t[1 * kThreads] += vx; t[2 * kThreads] += mx * mx;
      t[3 * kThreads] += my; t[4 * kThreads] += vy; t[5 * kThreads] += my * my;
      t[6 * kThreads] += cxy; t[7 * kThreads] += mx * my;
    }
    // drain the u32 shared histogram every round (<= 256 * n_sweeps counts)
    __syncthreads();
    bins += (double)hist[threadIdx.x];
    hist[threadIdx.x] = 0;
    __syncthreads();
  }

  // fixed-order CTA reduction of the 8 chain-level sums
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double v = warp_sum(tot_s[j][threadIdx.x]);
    if (lane == 0) red[wid][j] = v;
  }
  __syncthreads();
  double* part = a.partials + (uint64_t)blockIdx.x * kTot;
  if (threadIdx.x < 8) {
    double v = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) v += red[w][threadIdx.x];
    part[threadIdx.x] = v;
  }
  part[kHdr + threadIdx.x] = bins;
  flush_errors(a.err, nbad);
}

// K7: totals[j] = sum over CTAs of partials[cta][j], CTA order fixed.
__global__ void __launch_bounds__(kTot) reduce_partials_kernel(const double* partials,
                                                              uint32_t n_parts, double* totals,
                                                              double n_chains, double n_samples) {
  const uint32_t j = threadIdx.x;
  double v = 0.0;
  if (j < 8 || j >= kHdr)
    for (uint32_t p = 0; p < n_parts; ++p) v += partials[(uint64_t)p * kTot + j];
  if (j == 8) v = n_chains;
  if (j == 9) v = n_samples;
  totals[j] = v;
}

int ctas_per_sm() {
  static int cached = 0;
  if (cached == 0) {
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, gibbs_kernel, kThreads, 0) !=
            cudaSuccess || v <= 0)
      v = 4;
    cached = v;
  }
  return cached;
}

// One resident wave of CTAs; each thread runs `rounds` chains so that the
// chains divide as evenly as possible over the wave.
inline void grid_shape(uint64_t n_chains, const Ctx& ctx, unsigned& grid, uint32_t& rounds) {
  const uint64_t max_ctas = (uint64_t)ctx.num_sms * ctas_per_sm();
  const uint64_t max_threads = max_ctas * kThreads;
  const uint64_t r = (n_chains + max_threads - 1) / max_threads;
  rounds = (uint32_t)(r ? r : 1);
  uint64_t g = (n_chains + (uint64_t)rounds * kThreads - 1) / ((uint64_t)rounds * kThreads);
  grid = (unsigned)(g ? g : 1);
}

}  // namespace

size_t gibbs_partials_len(uint64_t n_chains, const Ctx& ctx) {
  unsigned g; uint32_t r;
  grid_shape(n_chains, ctx, g, r);
  return (size_t)g * kTot;
}

cudaError_t launch_gibbs(uint64_t n_chains, uint64_t n_sweeps, const double* x0,
                         const double* y0, uint64_t burn_in, double* out_x, double* out_y,
                         double* chain_stats, double* final_xy, double* totals,
                         double* partials, uint64_t base, const Ctx& ctx) {
  GibbsArgs a;
  unsigned grid; uint32_t rounds;
  grid_shape(n_chains, ctx, grid, rounds);
  a.n_chains = n_chains; a.n_sweeps = n_sweeps; a.burn_in = burn_in; a.base = base;
  a.stream_id = ctx.stream_id; a.k0 = ctx.k0; a.k1 = ctx.k1; a.rounds = rounds;
  a.x0 = x0; a.y0 = y0; a.out_x = out_x; a.out_y = out_y; a.chain_stats = chain_stats;
  a.final_xy = final_xy; a.partials = partials; a.err = ctx.err;
  gibbs_kernel<<<grid, kThreads, 0, ctx.stream>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || totals == nullptr) return e;
  reduce_partials_kernel<<<1, kTot, 0, ctx.stream>>>(
      partials, grid, totals, (double)n_chains, (double)n_chains * (double)(n_sweeps - burn_in));
  return cudaGetLastError();
}

}  // namespace brng
