// lda.cu -- NEXT row N4: an LDA-shaped consumer of
// varying-parameter deviates, the paper's motivating use (PAPER.md P:L34:
// "in Gibbs sampling of Latent Dirichlet Allocation (LDA) models ... one must
// sample from a Dirichlet distribution whose parameters are updated during
// each iteration"), and the "BatchRNG as asynchronous service" idea (P:L136:
// a background batch service replenishing standard-deviate buffers in
// overlap with other computational work).
//
// The model is LDA fold-in: documents' topic proportions and token topics
// are sampled with a FIXED topic-word matrix phi (inference on new documents
// with trained topics).  One Gibbs iteration (reading R-33, include/brng.h):
//   theta_d ~ Dirichlet(alpha + n_d.)     (exactly brng_dirichlet_f64 at c_t)
//   z_j     ~ Categorical(theta_dk phi[w_j, k])   (u_j = std uniform f64 j)
// Documents are independent given phi, so every iteration is one launch
// with a warp per document (dynamic assignment: lengths vary).
//
// Three ways of getting the deviates, all giving the same bits:
//   INLINE  the consumer calls the public device API (brng_dev::gamma_f64,
//           std_uniform_f64) where it needs a deviate: the GPU form of the
//           paper's one-at-a-time getters (reading R-32);
//   RING    a producer kernel on a side stream fills a slot of a two-slot
//           ring with the iteration's PARAMETER-FREE standard deviates (the
//           trial-1 normal z and word w3 of every Gamma component, the boost
//           log-uniform ln(1-u), every token's uniform) while the consumer
//           runs the previous iteration; the consumer applies the parameters
//           (mt_accept_z, mt_boost_from_log) and recomputes only the rare
//           trials >= 2 inline -- the paper's asynchronous service;
//   BULK    synchronous batch calls per iteration: counts -> alpha + n rows,
//           the library's Dirichlet kernel, the library's uniform fill, then
//           the consumer reads theta and u from HBM.
#include <algorithm>

#include "brng_internal.h"
#include "philox.cuh"

namespace brng {
namespace {

constexpr int kLdaThreads = 128;            // 4 warps; a warp works on one document
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ double lda_nan() { return __longlong_as_double(0x7ff8000000000000ll); }

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  return s;
}

// Gamma(alpha, 1) of component i from the ring: trial 1 from the producer's
// normal and word, trials >= 2 inline (the same blocks the getter uses), the
// boost from the producer's log-uniform.  Bit-identical to
// brng_dev::gamma_f64(key, stream, base, i, alpha, 1.0).
__device__ __forceinline__ double gamma_ring(const LdaArgs& a, uint64_t i, double al) {
  if (!(isfinite(al) && al > 0.0)) return lda_nan();
  double d, g = 0.0;
  bool ok = brng_dev::mt_accept_z(a.zbuf[i], a.w3buf[i], al, d, g);
  const uint64_t b0 = a.base + (uint64_t)brng_dev::kGammaStride * i;
  for (uint32_t t = 2; !ok && t <= brng_dev::kGammaMaxTrial; ++t)
    ok = brng_dev::mt_trial(brng_dev::block(brng_dev::Key{a.k0, a.k1}, a.stream, b0 + t), al,
                            d, g);
  if (!ok) return lda_nan();
  if (al < 1.0) g = brng_dev::mt_boost_from_log(a.lbuf[i], g, al);
  return g * 1.0;
}

// z for one token (R-33): p_k = fl(theta_k phi_k), running sums c_k in k
// order, C = c_{K-1}, x = fl(u C); the first k with x < c_k, else the last k
// with p_k > 0.
//
// Blocked search, the same values as two plain passes over K: pass 1 forms
// C and records the running sum at the end of each of nb <= kCatNB blocks
// of B components (E[m], in this lane's column of the warp's checkpoint
// area).  When every p_k has a clear sign bit the sums never decrease, so
// the first k with x < c_k lies in the first block with x < E[m], and
// re-running that block's sums from E[m-1] reproduces its c_k bit for bit
// (the same multiplies and adds in the same order): pass 2 reads B
// components instead of up to K.  A negative p_k (or a NaN with the sign
// bit set) takes the plain second pass.  The last k with p_k > 0 is found
// by a backward scan, only when no c_k exceeds x (x = C after rounding,
// C = 0 or NaN).
//
// phi rows are read with 256-bit loads when K % 4 == 0 and phi is 32-byte
// aligned (V4), theta (shared memory, the same address in every lane) with
// 128-bit broadcasts.  The previous form -- scalar loads, two full passes --
// kept L1 at 99.6% of its throughput with 32 scattered rows per warp load
// (5.35 ms per iteration at the bench shape).
constexpr uint32_t kCatNB = 8;

__device__ __forceinline__ void ld_phi4(const double* p, double& a, double& b, double& c,
                                        double& d) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
      : "l"(p));
}

template <bool V4>
__device__ __forceinline__ uint32_t categorical(const double* th, const double* ph, uint32_t K,
                                                double u, double* E) {
  const uint32_t B = V4 ? ((K + 4 * kCatNB - 1) / (4 * kCatNB)) * 4 : (K + kCatNB - 1) / kCatNB;
  double C = 0.0;
  uint32_t sgn = 0;
  uint32_t nb = 0;
  for (uint32_t k = 0; k < K; ++nb) {
    const uint32_t k1 = min(k + B, K);
    if (V4) {
      for (; k < k1; k += 4) {
        double f0, f1, f2, f3;
        ld_phi4(ph + k, f0, f1, f2, f3);
        const double2 t01 = *reinterpret_cast<const double2*>(th + k);
        const double2 t23 = *reinterpret_cast<const double2*>(th + k + 2);
        const double p0 = __dmul_rn(t01.x, f0), p1 = __dmul_rn(t01.y, f1);
        const double p2 = __dmul_rn(t23.x, f2), p3 = __dmul_rn(t23.y, f3);
        C = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(C, p0), p1), p2), p3);
        sgn |= __double2hiint(p0) | __double2hiint(p1) | __double2hiint(p2) |
               __double2hiint(p3);
      }
    } else {
      for (; k < k1; ++k) {
        const double p = __dmul_rn(th[k], __ldg(ph + k));
        C = __dadd_rn(C, p);
        sgn |= __double2hiint(p);
      }
    }
    E[nb * 32] = C;
  }
  const double x = __dmul_rn(u, C);
  if (!(sgn >> 31)) {
    for (uint32_t m = 0; m < nb; ++m) {
      if (x < E[m * 32]) {
        double c = m ? E[(m - 1) * 32] : 0.0;
        const uint32_t k1 = min(m * B + B, K);
        if (V4) {
          for (uint32_t k = m * B; k < k1; k += 4) {
            double f[4];
            ld_phi4(ph + k, f[0], f[1], f[2], f[3]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              c = __dadd_rn(c, __dmul_rn(th[k + i], f[i]));
              if (x < c) return k + i;
            }
          }
        } else {
          for (uint32_t k = m * B; k < k1; ++k) {
            c = __dadd_rn(c, __dmul_rn(th[k], __ldg(ph + k)));
            if (x < c) return k;
          }
        }
        break;                                   // not reached: c_{k1-1} = E[m] > x
      }
    }
  } else {
    double c = 0.0;
    for (uint32_t k = 0; k < K; ++k) {
      c = __dadd_rn(c, __dmul_rn(th[k], __ldg(ph + k)));
      if (x < c) return k;
    }
  }
  for (uint32_t k = K; k-- > 0;)
    if (__dmul_rn(th[k], __ldg(ph + k)) > 0.0) return k;
  return 0;
}

// One iteration.  SRC: 0 inline getters, 1 ring slot, 2 bulk buffers.
// Shared memory per warp: theta[K] (f64) then counts[K] (u32).
template <int SRC>
__global__ void __launch_bounds__(kLdaThreads) lda_consumer_kernel(const __grid_constant__ LdaArgs a) {
  extern __shared__ __align__(32) double lsm[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t K = a.k;
  // per warp: checkpoints E[kCatNB][32 lanes] (f64), theta[K] (f64), counts[K] (u32)
  constexpr uint32_t kW = kLdaThreads / 32;
  double* E = lsm + (size_t)wid * kCatNB * 32 + lane;
  double* th = lsm + (size_t)kW * kCatNB * 32 + (size_t)wid * K;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(lsm + (size_t)kW * kCatNB * 32 + (size_t)kW * K) +
                  (size_t)wid * K;
  const bool v4 = (K & 3u) == 0 && (reinterpret_cast<uintptr_t>(a.phi) & 31u) == 0;
  const uint64_t ubase = a.base + (uint64_t)brng_dev::kGammaStride * a.n_docs * K;
  const brng_dev::Key key{a.k0, a.k1};
  uint32_t nbad = 0;
  for (;;) {
    unsigned long long dd = 0;
    if (lane == 0) dd = atomicAdd(a.work, 1ull);
    const uint64_t d = __shfl_sync(kFull, dd, 0);
    if (d >= a.n_docs) break;
    uint64_t j0 = a.doc_off[d], j1 = a.doc_off[d + 1];
    // a malformed document range (decreasing, or past n_tokens) is counted
    // and treated as empty: no access outside the caller's arrays
    if (j1 < j0 || j1 > a.n_tokens) {
      nbad += lane == 0 ? 1u : 0u;
      j0 = j1 = 0;
    }
    if (SRC != 2) {
      for (uint32_t k = lane; k < K; k += 32) cnt[k] = 0;
      __syncwarp();
      for (uint64_t j = j0 + lane; j < j1; j += 32) {
        const uint32_t zz = a.z[j];
        atomicAdd(&cnt[zz < K ? zz : K - 1], 1u);
      }
      __syncwarp();
      // theta_d ~ Dirichlet(alpha + n_d.): the bulk Dirichlet's arithmetic
      // (Gammas, lane-strided sum + xor tree, g * fl(1/S))
      double s = 0.0;
      for (uint32_t k = lane; k < K; k += 32) {
        const double al = a.alpha[k] + (double)cnt[k];
        const uint64_t i = d * K + k;
        const double g = SRC == 0 ? brng_dev::gamma_f64(key, a.stream, a.base, i, al, 1.0)
                                  : gamma_ring(a, i, al);
        nbad += isnan(g) ? 1u : 0u;
        th[k] = g;
        s += g;
      }
      s = warp_sum(s);
      const double inv = 1.0 / s;
      for (uint32_t k = lane; k < K; k += 32) {
        const double t = th[k] * inv;
        th[k] = t;
        if (a.theta_out) a.theta_out[d * K + k] = t;
      }
    } else {
      for (uint32_t k = lane; k < K; k += 32) {
        const double t = a.theta_in[d * K + k];
        th[k] = t;
        if (a.theta_out) a.theta_out[d * K + k] = t;
      }
    }
    __syncwarp();
    for (uint64_t j = j0 + lane; j < j1; j += 32) {
      const double u = SRC == 0 ? brng_dev::std_uniform_f64(key, a.stream, ubase, j) : a.ubuf[j];
      const uint32_t w = a.words[j];
      if (w >= a.v) {                         // word id out of range: counted, z unchanged
        ++nbad;
        continue;
      }
      const double* ph = a.phi + (uint64_t)w * K;
      a.z[j] = (uint16_t)(v4 ? categorical<true>(th, ph, K, u, E)
                             : categorical<false>(th, ph, K, u, E));
    }
    __syncwarp();
  }
  flush_errors(a.err, nbad);
}

struct LdaProdArgs {
  uint64_t base, ubase, n_comp, n_tokens;
  RoundKeys rk;
  double* zbuf;
  uint32_t* w3buf;
  double* lbuf;
  double* ubuf;
};

// Producer (RING): the iteration's parameter-free standard deviates.
// Components i = d K + k: trial-1 normal z_i and word w3_i from block
// base + 256 i + 1, boost log-uniform ln(1 - u53) from block base + 256 i;
// tokens: u_j from block ubase + j/2 (two per block).  Static grid-stride
// (no work counter: it runs concurrently with a consumer of the handle).
__global__ void __launch_bounds__(256) lda_producer_kernel(const __grid_constant__ LdaProdArgs p) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = tid; i < p.n_comp; i += nt) {
    const uint64_t b0 = p.base + (uint64_t)brng_dev::kGammaStride * i;
    const uint4 w1 = philox_block_rk(b0 + 1, p.rk);
    p.zbuf[i] = brng_dev::mt_normal(w1);
    p.w3buf[i] = w1.w;
    p.lbuf[i] = brng_dev::mt_boost_log(philox_block_rk(b0, p.rk));
  }
  const uint64_t npair = (p.n_tokens + 1) / 2;
  for (uint64_t q = tid; q < npair; q += nt) {
    const uint4 w = philox_block_rk(p.ubase + q, p.rk);
    p.ubuf[2 * q] = u53(w.x, w.y);
    if (2 * q + 1 < p.n_tokens) p.ubuf[2 * q + 1] = u53(w.z, w.w);
  }
}

// BULK step 1: the Dirichlet parameter rows alpha + n_d. (f64 [D][K]).
__global__ void __launch_bounds__(kLdaThreads) lda_rows_kernel(const __grid_constant__ LdaArgs a,
                                                               double* rows) {
  extern __shared__ double lsm[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t K = a.k;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(lsm) + (size_t)wid * K;
  const uint64_t warp = ((uint64_t)blockIdx.x * kLdaThreads + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * kLdaThreads) >> 5;
  for (uint64_t d = warp; d < a.n_docs; d += nw) {
    for (uint32_t k = lane; k < K; k += 32) cnt[k] = 0;
    __syncwarp();
    uint64_t j0 = a.doc_off[d], j1 = a.doc_off[d + 1];
    if (j1 < j0 || j1 > a.n_tokens) j0 = j1 = 0;     // malformed range (counted by the consumer)
    for (uint64_t j = j0 + lane; j < j1; j += 32) {
      const uint32_t zz = a.z[j];
      atomicAdd(&cnt[zz < K ? zz : K - 1], 1u);
    }
    __syncwarp();
    for (uint32_t k = lane; k < K; k += 32) rows[d * K + k] = a.alpha[k] + (double)cnt[k];
    __syncwarp();
  }
}

template <typename Kern>
int ctas_for(Kern kern, size_t smem, int num_sms) {
  int v = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, kLdaThreads, smem) != cudaSuccess ||
      v < 1)
    v = 1;
  return v * num_sms;
}

}  // namespace

size_t lda_consumer_smem(uint32_t k) {
  return (size_t)(kLdaThreads / 32) * (kCatNB * 32 * 8 + (size_t)k * (8 + 4));
}

cudaError_t launch_lda_consumer(int src, const LdaArgs& a, const Ctx& ctx) {
  const size_t smem = lda_consumer_smem(a.k);
  cudaError_t e = cudaMemsetAsync(a.work, 0, sizeof(unsigned long long), ctx.stream);
  if (e != cudaSuccess) return e;
  const uint64_t want = (a.n_docs + 3) / 4;
  // Shared-memory carve-out for kLdaCtasPerSm CTAs/SM.  Left to itself the
  // driver gives a low-register consumer (BULK: 42 registers) a carve-out
  // for 16 CTAs/SM, which leaves little L1 for the phi rows.  Carve-outs for
  // 4 / 8 / 12 / 16 CTAs measured 1.74 / 1.62 / 1.62 / 1.70 ms (inline) and
  // 1.73 / 1.69 / 1.78 / 2.35 ms (bulk) per iteration at the bench shape
  // (profiles/r02_lda_carveout.txt).
  constexpr int kLdaCtasPerSm = 8;
  const int carve = (int)std::min<size_t>(
      100, (kLdaCtasPerSm * (smem + 1024) * 100 + 228 * 1024 - 1) / (228 * 1024));
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) {
      cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem);
      if (e2 != cudaSuccess) return e2;
    }
    cudaError_t e3 = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          carve);
    if (e3 != cudaSuccess) return e3;
    const uint64_t cap = (uint64_t)ctas_for(kern, smem, ctx.num_sms);
    const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
    kern<<<g, kLdaThreads, smem, ctx.stream>>>(a);
    return cudaGetLastError();
  };
  if (src == 0) return go(lda_consumer_kernel<0>);
  if (src == 1) return go(lda_consumer_kernel<1>);
  return go(lda_consumer_kernel<2>);
}

cudaError_t launch_lda_producer(const LdaArgs& a, double* zbuf, uint32_t* w3buf, double* lbuf,
                                double* ubuf, const Ctx& ctx, cudaStream_t s) {
  LdaProdArgs p;
  p.base = a.base;
  p.ubase = a.base + (uint64_t)brng_dev::kGammaStride * a.n_docs * a.k;
  p.n_comp = a.n_docs * a.k;
  p.n_tokens = a.n_tokens;
  p.rk = make_round_keys(ctx.k0, ctx.k1, a.stream);
  p.zbuf = zbuf; p.w3buf = w3buf; p.lbuf = lbuf; p.ubuf = ubuf;
  const uint64_t work = p.n_comp > (p.n_tokens + 1) / 2 ? p.n_comp : (p.n_tokens + 1) / 2;
  const uint64_t want = (work + 255) / 256;
  const uint64_t cap = (uint64_t)ctx.num_sms * 8;
  const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
  lda_producer_kernel<<<g, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_lda_rows(const LdaArgs& a, double* rows, const Ctx& ctx) {
  const size_t smem = (size_t)(kLdaThreads / 32) * a.k * 4;
  const uint64_t want = (a.n_docs + 3) / 4;
  const uint64_t cap = (uint64_t)ctx.num_sms * 16;
  const unsigned g = (unsigned)(want < cap ? (want ? want : 1) : cap);
  lda_rows_kernel<<<g, kLdaThreads, smem, ctx.stream>>>(a, rows);
  return cudaGetLastError();
}

}  // namespace brng
