// gamma.cu -- K3 (per-sample-alpha Gamma) and K4 (Dirichlet rows) on sm_100a.
//
// Gamma is the paper's irreducible distribution built on the Gaussian and
// log-uniform buffers (code withheld).  The
// algorithm is Marsaglia-Tsang (contract R-08..R-11, include/brng.h):
//   d = alpha' - 1/3, c = 1/sqrt(9d); trial t of sample i uses Philox block
//   cursor + 256 i + t; accept iff ln U < z^2/2 + d - d v + d ln v, g = d v;
//   alpha < 1: g *= exp(ln(1-u)/alpha) from block cursor + 256 i.
// Dirichlet (P:L34 footnote): y_k ~ Gamma(alpha_k, 1), x_k = y_k / sum y.
//
// GPU design: every lane of a warp owns one sample at a time.  After each
// trial, __ballot_sync/__popc hand the finished lanes the next samples of the
// warp's queue (a contiguous chunk), so rejected lanes simply retry with the
// next trial counter while the rest of the warp keeps doing useful trials --
// no lane idles until the queue drains.  Per-sample counters keep every
// sample a pure function of (key, cursor, i), independent of this schedule.
// All arithmetic is binary64 (R-28).
#include "brng_internal.h"
#include "philox.cuh"

namespace brng {
namespace {

constexpr int kThreads = 256;
// Samples per warp queue (Gamma): a queue's tail (lanes idle while its last
// samples finish) happens once per chunk.  Warps take chunks from a device
// counter (BRNG_GAMMA_DYN, one resident wave of CTAs), so the kernel's tail is
// at most one chunk per warp: cfg3 0.877 ms with a static grid-stride
// assignment of 4096-sample chunks -> 0.840 (2048, dynamic), 0.846 (4096,
// dynamic), 0.837 (1024, dynamic); Dirichlet row groups likewise 4.48 -> 4.33.
#ifndef BRNG_GAMMA_CHUNK
#define BRNG_GAMMA_CHUNK 2048
#endif
constexpr uint64_t kChunk = BRNG_GAMMA_CHUNK;
#ifndef BRNG_GAMMA_SPEC
#define BRNG_GAMMA_SPEC 0     // speculative boosts for Gamma (cfg3: 36% boosted)
#endif
constexpr uint32_t kStride = 256;          // blocks per sample (R-11)
constexpr uint32_t kMaxTrial = 255;
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ll); }

// A chunk's array pointer, formed once per chunk and hidden from the
// optimiser, so a sample's address is one IMAD.WIDE.U32 (offset x size +
// pointer) instead of a re-derived 64-bit (chunk start + offset) sum, shift
// and add per access: Gamma cfg3 0.839-0.847 -> 0.825-0.828 ms, identical
// output (profiles/r02_opaque_ptr.txt; the Dirichlet queue gained from it only
// after its other round-2 changes, profiles/r02_dir_addr.txt).
template <typename T>
__device__ __forceinline__ T* chunk_ptr(T* p) {
  asm("mov.b64 %0, %0;" : "+l"(p));
  return p;
}


// One Marsaglia-Tsang trial (R-09) and the alpha<1 boost (R-10): the public
// device API's (include/brng_device.cuh): binary32 decision with a binary64
// recheck band, binary64 values.
using brng_dev::mt_boost;
using brng_dev::mt_trial;

// Lookup tables of the trial/boost math: read through the read-only path
// (GlobalTables).  Staging them in shared memory was measured slower
// (cfg3 0.929 -> 0.987 ms: random 16-B LDS bank conflicts).
using Tables = brng_dev::dm::GlobalTables;
// The same tables with the six constants that meet another constant operand
// in one DFMA (Horner's first steps of ln / cos / exp, the ln table index and
// the exp range reduction) held in registers for the whole kernel: left to
// itself ptxas re-loads one of each pair with LDC in every iteration.  The
// values are multiplied by 1.0 read from memory (2^0 of the exp table), so
// they are the same constants but not ones ptxas could rematerialise.
// Dirichlet (cfg4) 4.061 -> 3.965 ms, identical output (56 registers); the
// Gamma kernel, at 62 of its 64 registers, is slower with any subset, and
// table addresses or the rsqrt Newton constant in registers too (64
// registers) undo the gain
// (profiles/r02_regk.txt).
struct RegTables : brng_dev::dm::GlobalTables {
  double l7, r128, s7, c6, e6, il2;
  __device__ __forceinline__ RegTables() {
    namespace dm = brng_dev::dm;
    const double one = __ldg(&brng_dev::tab::kExp2[0]);
    l7 = dm::kC[dm::kL7] * one; r128 = dm::kC[dm::kRndM128] * one; s7 = dm::kC[dm::kS7] * one;
    c6 = dm::kC[dm::kC6] * one; e6 = dm::kC[dm::kE6] * one; il2 = dm::kC[dm::kInvLn2x64] * one;
  }
  __device__ __forceinline__ double k(int i) const {
    namespace dm = brng_dev::dm;
    return i == dm::kL7 ? l7 : i == dm::kRndM128 ? r128 : i == dm::kS7 ? s7 : i == dm::kC6 ? c6
         : i == dm::kE6 ? e6 : i == dm::kInvLn2x64 ? il2 : dm::kC[i];
  }
};

// alpha<1 boost work item, parked in a per-warp shared-memory queue so that
// boosts run as full warps instead of as a divergent branch (36% of cfg3's
// samples, 91% of cfg4's).
// 32 bytes with the sample's alpha and beta (BRNG_SLIM_QUEUE=1: 16 bytes,
// the drain re-reading them from global memory).  The slim item was chosen in
// round 1 to halve the queue's shared memory; at 4 CTAs/SM the full item
// costs 16 KB per CTA and saves the drain's two loads and their address
// arithmetic: cfg3 0.801 -> 0.789 ms, identical output (profiles/r02_queue_item.txt).
#ifndef BRNG_SLIM_QUEUE
#define BRNG_SLIM_QUEUE 0
#endif
struct BoostItem {
  double g;
#if !BRNG_SLIM_QUEUE
  double alpha, beta;
#endif
  uint32_t off_t;          // sample offset in the queue's range | trial << 24
  uint32_t pad;
};
constexpr int kBoostCap = 64;
// a queue's range of samples is < 2^24 (Gamma chunks of kChunk, Dirichlet
// row groups / rows: the host limits k < 2^24), so 32-bit offsets suffice
constexpr uint32_t kOffBits = 24;

// Warp-cooperative Gamma queue over the samples beg + [0, n), n < 2^24.
//   load(off, alpha, beta)  -- parameters of sample beg + off
//   sink(off, value, trial) -- value = g * beta (NaN when invalid / capped)
//   q                       -- this warp's BoostItem[kBoostCap] in shared memory
// Offsets are 32-bit (the callers' lambdas address arrays already shifted by
// beg): the per-iteration bookkeeping has no 64-bit index arithmetic.
// All 32 lanes must call it (ballots use the full mask).  Every sample's
// value is a pure function of its counters; the schedule (which lane, which
// iteration, queued or not) never changes it.
// SPEC (speculative boost): every sample's boost log-uniform ln(1-u) is
// computed with its first trial (a second, independent Philox chain in the
// same lane: ILP) and kept in a register, and an accepted alpha<1 sample is
// boosted in place -- no boost queue.  Pays when most samples are boosted
// (cfg4: 91%); a sample with alpha >= 1 wastes the block.
template <typename P, bool SPEC = false, typename Load, typename Sink, typename Tab>
__device__ __forceinline__ void mt_queue(uint64_t beg, uint32_t n, uint64_t base,
                                         const RoundKeys& rk, const Tab& tb, Load load,
                                         Sink sink, uint32_t& nbad, BoostItem* q) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const uint64_t base_c = base + (uint64_t)kStride * beg;   // block of sample beg
  uint32_t head = 32;
  uint32_t off = lane;
  // a 32-bit flag: as a bool ptxas kept it in a byte of a register and
  // re-extracted it with PRMTs every iteration (Gamma 0.806 -> 0.802 ms)
  uint32_t active = off < n ? 1u : 0u;
  // the parameters stay in their storage type until used: a binary32 alpha
  // converted at the load (the refill, at the end of an iteration) made the
  // warp wait there for the load (cfg4: 14% of the kernel's stall samples on
  // that F2F.F64.F32, ncu source view)
  P alpha_r = P(1), beta_r = P(1);
  double d = 0.0;
  uint32_t t = 1;
  uint32_t qn = 0;                                   // queued boosts (warp-uniform)
  // issue the parameter loads only; they are consumed after the next trial's
  // Philox block and Box-Muller normal
  // SPEC: the sample's counter base kept from its refill (Dirichlet 3.70 ->
  // 3.68 ms); the Gamma queue, at its register cap, recomputes it (keeping it
  // there was 3.5% slower; profiles/r02_recheck.txt)
  uint64_t pos_r = SPEC ? base_c + ((uint64_t)off << 8) : 0;
  auto setup = [&]() {
    load(off, alpha_r, beta_r);
    t = 1;
    if (SPEC) pos_r = base_c + ((uint64_t)off << 8);
  };
  // lanes [0, k) take the last k queue entries, boost and sink them
  auto drain = [&](uint32_t k) {
    __syncwarp();
    if (lane < k) {
      const BoostItem it = q[qn - k + lane];
      const uint32_t oo = it.off_t & ((1u << kOffBits) - 1);
#if BRNG_SLIM_QUEUE
      P qa, qb;
      load(oo, qa, qb);
#else
      const double qa = it.alpha, qb = it.beta;
#endif
      const uint4 wb = philox_block_rk(base_c + ((uint64_t)oo << 8), rk);
      const double L = brng_dev::mt_boost_log(wb, tb);
      const double gb = brng_dev::mt_boost_from_log(L, it.g, (double)qa, tb);
      sink(oo, gb * (double)qb, it.off_t >> kOffBits);
    }
    qn -= k;
    __syncwarp();
  };
  if (active) setup();
  while (__any_sync(kFull, active)) {
    bool done = false, boost = false;
    double g = 0.0;
    double alpha = 1.0;
    double Lb = 0.0;                                 // SPEC: boost ln(1-u) of the sample
    if (active) {
      const uint64_t pos = SPEC ? pos_r : base_c + ((uint64_t)off << 8);   // 256 blocks per sample
      const uint4 w = philox_block_rk(pos + t, rk);
      if (SPEC) {
        // every lane computes it from trial 1 on: no divergent region
        // (retrying lanes would idle through it anyway): cfg4 4.160 ->
        // 4.052 ms.  The boost block does not depend on t, so every trial
        // gets the same value (no select of the trial-1 value: 3.902 ->
        // 3.878 ms, profiles/r02_queue_decision.txt).
        Lb = brng_dev::mt_boost_log(philox_block_rk(pos, rk), tb);
      }
      alpha = (double)alpha_r;
      const double beta = (double)beta_r;
      const bool valid = isfinite(alpha) && isfinite(beta) && alpha > 0.0 && beta > 0.0;
      const bool acc = mt_trial(w, alpha, d, g, tb);
      if (SPEC) {
        // the decision as predicates (the same outcomes as the branch chain
        // below), one select for the boost and one for the stored value:
        // 3.878 -> 3.817-3.832 ms; the Gamma queue is slower this way
        // (0.817 -> 0.834 ms) and keeps the chain
        const uint32_t tn = t + 1u;
        const bool cap = !acc & (tn > kMaxTrial);
        const bool fail = !valid | cap;
        done = !valid | acc | cap;
        t = fail ? 0u : (acc ? t : tn);
        nbad += fail ? 1u : 0u;
        const bool bst = (!fail & acc) & (alpha < 1.0);
        const double gb = brng_dev::mt_boost_from_log(Lb, g, alpha, tb);
        const double gv = bst ? gb : g;
        if (done) sink(off, fail ? qnan() : gv * beta, t);
      } else {
        if (!valid) {
          done = true; t = 0; ++nbad;
        } else if (acc) {
          done = true;
        } else if (++t > kMaxTrial) {
          done = true; t = 0; ++nbad;
        }
        boost = done && t != 0 && alpha < 1.0;
        if (done && !boost) sink(off, t != 0 ? g * beta : qnan(), t);
      }
    }
    const uint32_t bm = SPEC ? 0u : __ballot_sync(kFull, boost);
    if (boost) {
      BoostItem it;
      it.g = g;
#if !BRNG_SLIM_QUEUE
      it.alpha = alpha; it.beta = (double)beta_r;
#endif
      it.off_t = off | (t << kOffBits);
      q[qn + __popc(bm & lt)] = it;
    }
    qn += __popc(bm);
    if (!SPEC && qn >= 32) drain(32);
    const uint32_t dm = __ballot_sync(kFull, done);
    if (done) {
      off = head + __popc(dm & lt);
      active = off < n;
      if (active) setup();
    }
    head += __popc(dm);
  }
  if (!SPEC && qn) drain(qn);
}

template <typename T>
struct GammaArgs {
  const T* alpha;
  const T* beta;
  T* out;
  uint8_t* trials;
  uint64_t n, base, stream;
  RoundKeys rk;
  unsigned long long* err;
  unsigned long long* work;
};

// Dynamic chunk / row-group assignment: a warp's lane 0 takes the next index
// from the handle's work counter (zeroed by a memset before each launch).
// The values never depend on which warp ran a chunk.
#ifndef BRNG_GAMMA_DYN
#define BRNG_GAMMA_DYN 1
#endif
#ifndef BRNG_GAMMA_MINB
#define BRNG_GAMMA_MINB 4
#endif
// TR: the call passed a trials array (a compile-time branch: without one the
// queue's sink has no per-sample null test and address arithmetic for it)
template <typename T, bool TR>
__global__ void __launch_bounds__(kThreads, BRNG_GAMMA_MINB) gamma_kernel(const __grid_constant__ GammaArgs<T> a) {
  __shared__ BoostItem qs[kThreads / 32][kBoostCap];
  const Tables tb{};
  BoostItem* q = qs[threadIdx.x >> 5];
  const uint64_t warp = ((uint64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint64_t n_warps = ((uint64_t)gridDim.x * kThreads) >> 5;
  uint32_t nbad = 0;
#if BRNG_GAMMA_DYN
  (void)warp; (void)n_warps;
  for (;;) {
    unsigned long long cidx = 0;
    if ((threadIdx.x & 31) == 0) cidx = atomicAdd(a.work, 1ull);
    cidx = __shfl_sync(kFull, cidx, 0);
    const uint64_t beg = (uint64_t)cidx * kChunk;
    if (beg >= a.n) break;
#else
  for (uint64_t beg = warp * kChunk; beg < a.n; beg += n_warps * kChunk) {
#endif
    const uint32_t n = (uint32_t)(beg + kChunk < a.n ? kChunk : a.n - beg);
    const T* al_c = chunk_ptr(a.alpha + beg);
    const T* be_c = chunk_ptr(a.beta + beg);
    T* out_c = chunk_ptr(a.out + beg);
    uint8_t* tr_c = TR ? chunk_ptr(a.trials + beg) : nullptr;
    mt_queue<T, BRNG_GAMMA_SPEC != 0>(
        beg, n, a.base, a.rk, tb,
        [&](uint32_t o, T& al, T& be) {
          al = __ldg(al_c + o);
          be = __ldg(be_c + o);
        },
        [&](uint32_t o, double v, uint32_t t) {
          out_c[o] = (T)v;
          if (TR) tr_c[o] = (uint8_t)t;
        },
        nbad, q);
  }
  flush_errors(a.err, nbad);
}

template <typename T>
struct DirArgs {
  const T* alpha;
  T* out;
  uint8_t* trials;
  uint64_t n_rows, k, base, stream;
  RoundKeys rk;
  unsigned long long* err;
  uint32_t rpw;          // rows per warp queue (smem kernel)
  unsigned long long* work;   // dynamic group counter (BRNG_GAMMA_DYN)
  double* scratch;            // two-pass binary32: [gridDim.x * 4][k] Gammas (or null)
};

constexpr int kDirThreads = 128;     // 4 warps / CTA, one row per warp
#ifndef BRNG_DIR_SPEC
#define BRNG_DIR_SPEC 1                  // speculative in-place boosts (mt_queue SPEC)
#endif
#ifndef BRNG_DIR_SMEM_K
#define BRNG_DIR_SMEM_K 2048
#endif
constexpr uint64_t kDirSmemK = BRNG_DIR_SMEM_K;
#ifndef BRNG_DIR_SMEM_K32
#define BRNG_DIR_SMEM_K32 1024     // binary32 rows up to this K use shared memory
#endif   // rows up to this K are staged in smem
#ifndef BRNG_DIR_TARGET
#define BRNG_DIR_TARGET 512
#endif
constexpr uint64_t kDirTarget = BRNG_DIR_TARGET;   // samples per warp queue (rows grouped)

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  return s;
}

// K <= kDirSmemK: Gammas of the row staged in shared memory (8 K bytes/warp),
// summed lane-strided then by a fixed xor-shuffle tree, normalised, stored
// coalesced.
template <typename T, bool TR>
__global__ void __launch_bounds__(kDirThreads) dirichlet_smem_kernel(const __grid_constant__ DirArgs<T> a) {
  extern __shared__ double gsm[];
  __shared__ BoostItem qs[kDirThreads / 32][kBoostCap];
  const RegTables tb{};
  BoostItem* q = qs[threadIdx.x >> 5];
  const uint32_t lane = threadIdx.x & 31;
  // a.rpw rows per warp queue: one continuous queue over the group's
  // rpw * k samples, so the lanes idle at a queue's tail once per group
  // instead of once per row (the rows' values do not depend on the grouping)
  double* g_grp = gsm + (uint64_t)(threadIdx.x >> 5) * a.rpw * a.k;
  const uint64_t warp = ((uint64_t)blockIdx.x * kDirThreads + threadIdx.x) >> 5;
  const uint64_t n_warps = ((uint64_t)gridDim.x * kDirThreads) >> 5;
  const uint64_t n_groups = (a.n_rows + a.rpw - 1) / a.rpw;
  uint32_t nbad = 0;
#if BRNG_GAMMA_DYN
  (void)warp; (void)n_warps;
  for (;;) {
    unsigned long long gidx = 0;
    if (lane == 0) gidx = atomicAdd(a.work, 1ull);
    const uint64_t grp = __shfl_sync(kFull, gidx, 0);
    if (grp >= n_groups) break;
#else
  for (uint64_t grp = warp; grp < n_groups; grp += n_warps) {
#endif
    const uint64_t row0 = grp * a.rpw;
    const uint64_t rows = a.n_rows - row0 < a.rpw ? a.n_rows - row0 : a.rpw;
    const uint64_t beg = row0 * a.k;
    // the chunk pointer behind an empty asm (one IMAD.WIDE per address, as in
    // the Gamma kernel) and the staging row as a 32-bit shared address
    // (no per-store generic-to-shared window arithmetic): 3.811 -> 3.737-3.743
    // ms together (profiles/r02_dir_addr.txt)
    const T* al_c = chunk_ptr(a.alpha + beg);
    uint8_t* tr_c = TR ? a.trials + beg : nullptr;
    const uint32_t g_sh = (uint32_t)__cvta_generic_to_shared(g_grp);
    mt_queue<T, BRNG_DIR_SPEC != 0>(
        beg, (uint32_t)(rows * a.k), a.base, a.rk, tb,
        [&](uint32_t o, T& al, T& be) {
          al = __ldg(al_c + o);
          be = T(1);
        },
        [&](uint32_t o, double v, uint32_t t) {
          asm volatile("st.shared.f64 [%0], %1;" ::"r"(g_sh + 8u * o), "d"(v) : "memory");
          if (TR) tr_c[o] = (uint8_t)t;
        },
        nbad, q);
    __syncwarp();
    for (uint64_t r = 0; r < rows; ++r) {
      const double* g_row = g_grp + r * a.k;
      double s = 0.0;
      for (uint64_t j = lane; j < a.k; j += 32) s += g_row[j];
      s = warp_sum(s);
      const double inv = 1.0 / s;
      for (uint64_t j = lane; j < a.k; j += 32) a.out[beg + r * a.k + j] = (T)(g_row[j] * inv);
    }
    __syncwarp();
  }
  flush_errors(a.err, nbad);
}

// Any K: two passes over the row.  binary64 output: the first pass stores the
// unnormalised Gammas in the output row itself, the second rescales them in
// place.  binary32 output: a Gamma may not be representable in binary32
// before the division (a row of tiny alphas), so the Gammas go to a
// handle-owned binary64 scratch row per warp.  Both sum the row in the
// shared-memory kernel's order (lane-strided, then the xor tree), so they
// give the same values as it.  Without scratch (above 2 GB, or inside a graph
// capture that would have to grow it) the second pass recomputes every Gamma
// from its counters; that path sums in queue order (a deterministic order,
// but not the shared-memory kernel's: values may differ in the last bit).
template <typename T>
__global__ void __launch_bounds__(kDirThreads) dirichlet_2pass_kernel(const __grid_constant__ DirArgs<T> a) {
  __shared__ BoostItem qs[kDirThreads / 32][kBoostCap];
  const Tables tb{};
  BoostItem* q = qs[threadIdx.x >> 5];
  const uint64_t warp = ((uint64_t)blockIdx.x * kDirThreads + threadIdx.x) >> 5;
  const uint64_t n_warps = ((uint64_t)gridDim.x * kDirThreads) >> 5;
  uint32_t nbad = 0, nbad2 = 0;
  // with scratch (one resident wave) warps take rows from the work counter;
  // otherwise a static grid-stride assignment
  auto fetch = [&]() -> uint64_t {
    unsigned long long r = 0;
    if ((threadIdx.x & 31) == 0) r = atomicAdd(a.work, 1ull);
    return __shfl_sync(kFull, r, 0);
  };
  for (uint64_t row = a.scratch ? fetch() : warp; row < a.n_rows;
       row = a.scratch ? fetch() : row + n_warps) {
    const uint64_t beg = row * a.k;
    const uint32_t kk = (uint32_t)a.k;                  // k < 2^24 (host-checked)
    const T* al_c = a.alpha + beg;
    uint8_t* tr_c = a.trials ? a.trials + beg : nullptr;
    auto load = [&](uint32_t o, T& al, T& be) {
      al = __ldg(al_c + o);
      be = T(1);
    };
    double s = 0.0;
    if (sizeof(T) == 4 && a.scratch) {
      // binary32 with scratch: the warp's own row of binary64 Gammas
      double* g_row = a.scratch + warp * a.k;
      mt_queue<T>(beg, kk, a.base, a.rk, tb, load,
               [&](uint32_t o, double v, uint32_t t) {
                 g_row[o] = v;
                 if (tr_c) tr_c[o] = (uint8_t)t;
               },
               nbad, q);
      __syncwarp();                           // the row's Gammas are visible to the warp
      const uint32_t lane = threadIdx.x & 31;
      // the shared-memory kernel's sum order: lane-strided, then the xor tree
      for (uint64_t j = lane; j < a.k; j += 32) s += g_row[j];
      s = warp_sum(s);
      const double inv = 1.0 / s;
      for (uint64_t j = lane; j < a.k; j += 32) a.out[beg + j] = (T)(g_row[j] * inv);
      __syncwarp();
    } else if constexpr (sizeof(T) == 8) {
      mt_queue<T>(beg, kk, a.base, a.rk, tb, load,
               [&](uint32_t o, double v, uint32_t t) {
                 a.out[beg + o] = (T)v;
                 if (tr_c) tr_c[o] = (uint8_t)t;
               },
               nbad, q);
      __syncwarp();                           // the row's stores are visible to the warp
      const uint32_t lane = threadIdx.x & 31;
      for (uint64_t j = lane; j < a.k; j += 32) s += (double)a.out[beg + j];
      s = warp_sum(s);
      const double inv = 1.0 / s;
      for (uint64_t j = lane; j < a.k; j += 32) a.out[beg + j] = (T)((double)a.out[beg + j] * inv);
    } else {
      mt_queue<T>(beg, kk, a.base, a.rk, tb, load,
               [&](uint32_t, double v, uint32_t) { s += v; }, nbad, q);
      s = warp_sum(s);
      const double inv = 1.0 / s;
      mt_queue<T>(beg, kk, a.base, a.rk, tb, load,
               [&](uint32_t o, double v, uint32_t t) {
                 a.out[beg + o] = (T)(v * inv);
                 if (tr_c) tr_c[o] = (uint8_t)t;
               },
               nbad2, q);
    }
  }
  flush_errors(a.err, nbad);
}

template <typename T>
cudaError_t gamma_typed(const T* alpha, const T* beta, T* out, uint8_t* trials, uint64_t n,
                        uint64_t base, const Ctx& ctx) {
  GammaArgs<T> a{alpha, beta, out, trials, n, base, ctx.stream_id,
                   make_round_keys(ctx.k0, ctx.k1, ctx.stream_id), ctx.err, ctx.work};
#if BRNG_GAMMA_DYN
  {
    cudaError_t e = cudaMemsetAsync(ctx.work, 0, sizeof(unsigned long long), ctx.stream);
    if (e != cudaSuccess) return e;
  }
#endif
  const uint64_t warps_needed = (n + kChunk - 1) / kChunk;
  const uint64_t ctas_needed = (warps_needed + (kThreads / 32) - 1) / (kThreads / 32);
#if BRNG_GAMMA_DYN
  const uint64_t cap = (uint64_t)ctx.num_sms * BRNG_GAMMA_MINB;   // one resident wave
#else
  const uint64_t cap = (uint64_t)ctx.num_sms * 8;  // two waves of 4 resident CTAs/SM
#endif
  const unsigned g = (unsigned)(ctas_needed < cap ? ctas_needed : cap);
  if (a.trials)
    gamma_kernel<T, true><<<g, kThreads, 0, ctx.stream>>>(a);
  else
    gamma_kernel<T, false><<<g, kThreads, 0, ctx.stream>>>(a);
  return cudaGetLastError();
}

int dir2_ctas_per_sm() {
  static int cached = [] {
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, dirichlet_2pass_kernel<float>,
                                                      kDirThreads, 0) != cudaSuccess ||
        v < 1)
      v = 1;
    return v;
  }();
  return cached;
}

template <typename T>
cudaError_t dirichlet_typed(const T* alpha, uint64_t n_rows, uint64_t k, T* out,
                            uint8_t* trials, uint64_t base, const Ctx& ctx) {
  DirArgs<T> a{alpha, out, trials, n_rows, k, base, ctx.stream_id,
                 make_round_keys(ctx.k0, ctx.k1, ctx.stream_id), ctx.err, 1u, ctx.work,
                 nullptr};
  const uint64_t ctas_needed = (n_rows + 3) / 4;
  // binary64 output parks the row's Gammas in the output row instead (no
  // shared-memory occupancy cost): faster from K = 1024 on (tools/dirichlet_k.py:
  // 2^27 components, K = 1024: 2.38 -> 2.12 ms, K = 2048: 3.71 -> 2.10 ms)
  const uint64_t smem_k = sizeof(T) == 8 ? (kDirSmemK < 512 ? kDirSmemK : 512)
                                         : (kDirSmemK < BRNG_DIR_SMEM_K32 ? kDirSmemK
                                                                          : BRNG_DIR_SMEM_K32);
  if (k <= smem_k) {
    const uint64_t r = kDirTarget / k;
    a.rpw = (uint32_t)(r < 1 ? 1 : (r > 8 ? 8 : r));
    const size_t smem = (size_t)4 * a.rpw * k * sizeof(double);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(dirichlet_smem_kernel<T, true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(dirichlet_smem_kernel<T, false>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    const uint64_t groups = (n_rows + a.rpw - 1) / a.rpw;
    const uint64_t ctas = (groups + 3) / 4;
#if BRNG_GAMMA_DYN
    // one resident wave of CTAs; warps take row groups from a counter
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, trials ? dirichlet_smem_kernel<T, true> : dirichlet_smem_kernel<T, false>,
            kDirThreads, smem) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    const uint64_t cap = (uint64_t)ctx.num_sms * per_sm;
    cudaError_t e0 = cudaMemsetAsync(ctx.work, 0, sizeof(unsigned long long), ctx.stream);
    if (e0 != cudaSuccess) return e0;
#else
    const uint64_t cap = (uint64_t)ctx.num_sms * 16 * 8;
#endif
    const unsigned g = (unsigned)(ctas < cap ? ctas : cap);
    if (trials)
      dirichlet_smem_kernel<T, true><<<g, kDirThreads, smem, ctx.stream>>>(a);
    else
      dirichlet_smem_kernel<T, false><<<g, kDirThreads, smem, ctx.stream>>>(a);
  } else {
    uint64_t cap = (uint64_t)ctx.num_sms * 16 * 8;
    if (sizeof(T) == 4 && ctx.dir_scratch) {
      // one resident wave; warp w parks its rows' Gammas in scratch row w
      a.scratch = ctx.dir_scratch;
      cap = (uint64_t)ctx.num_sms * dir2_ctas_per_sm();
      cudaError_t e0 = cudaMemsetAsync(ctx.work, 0, sizeof(unsigned long long), ctx.stream);
      if (e0 != cudaSuccess) return e0;
    }
    const unsigned g = (unsigned)(ctas_needed < cap ? ctas_needed : cap);
    dirichlet_2pass_kernel<T><<<g, kDirThreads, 0, ctx.stream>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gamma(int dtype, const void* alpha, const void* beta, void* out,
                         uint8_t* trials, uint64_t n, uint64_t base, const Ctx& ctx) {
  if (dtype == kF32)
    return gamma_typed<float>(static_cast<const float*>(alpha), static_cast<const float*>(beta),
                              static_cast<float*>(out), trials, n, base, ctx);
  return gamma_typed<double>(static_cast<const double*>(alpha),
                             static_cast<const double*>(beta), static_cast<double*>(out), trials,
                             n, base, ctx);
}

size_t dirichlet_scratch_len(int dtype, uint64_t k, const Ctx& ctx) {
  if (dtype != kF32 || k <= (kDirSmemK < BRNG_DIR_SMEM_K32 ? kDirSmemK : BRNG_DIR_SMEM_K32))
    return 0;
  return (size_t)ctx.num_sms * dir2_ctas_per_sm() * (kDirThreads / 32) * k;
}

cudaError_t launch_dirichlet(int dtype, const void* alpha, uint64_t n_rows, uint64_t k,
                             void* out, uint8_t* trials, uint64_t base, const Ctx& ctx) {
  if (dtype == kF32)
    return dirichlet_typed<float>(static_cast<const float*>(alpha), n_rows, k,
                                  static_cast<float*>(out), trials, base, ctx);
  return dirichlet_typed<double>(static_cast<const double*>(alpha), n_rows, k,
                                 static_cast<double*>(out), trials, base, ctx);
}

}  // namespace brng
