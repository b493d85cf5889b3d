// fill.cu -- K1/K2: Philox words, standard uniforms and the per-sample
// transforms of the reducible distributions ("a + (b - a) * x",
// P:L69 GetUniform/GetGaussian/GetExponential/GetLogUniform
// parameters read per sample from memory), plus the NEXT-row N2 getters
// GetLaplace / GetWeibull (algorithms R-30), as ONE fused streaming
// pass on sm_100a:
//
//   Philox4x32-10 block (4 words, registers) -> standard deviates (4 per block
//   for f32, 2 for f64; Laplace uses two words per sample) -> vector
//   streaming parameter loads -> per-sample transform -> vector streaming store.
//
// This is the BatchRNG idea recast for the GPU: the "buffer" of standard
// deviates is the four-word Philox block held in registers, refilled by
// counter (no buffer counter, no refill branch), so each sample costs its
// algorithmic HBM traffic only (f32: 8 B of parameters + 4 B out).
#include "brng_internal.h"
#include "philox.cuh"

namespace brng {
namespace {

constexpr int kThreads = 256;

template <typename T>
struct FillArgs {
  const T* p0;   // a | mu | lambda | alpha   (nullable for raw/std/log-uniform)
  const T* p1;   // b | sigma | beta
  T* out;
  uint64_t n;
  uint64_t base;
  uint64_t stream;
  RoundKeys rk;  // Philox round keys (constant bank)
  int vec;       // all arrays aligned to the vector width
  unsigned long long* err;
  T s0, s1;      // SCALAR mode: fixed parameters (the paper's VSL-Batch case)
};

template <int DIST>
constexpr int n_params() {
  return (DIST == kUniform || DIST == kGaussian || DIST == kLaplace || DIST == kWeibull) ? 2
         : (DIST == kExponential) ? 1 : 0;
}
// samples per Philox block
template <typename T, int DIST>
constexpr int spb() {
  return sizeof(T) == 4 ? (DIST == kLaplace ? 2 : 4) : (DIST == kLaplace ? 1 : 2);
}

// ---- vector load/store of N consecutive T (streaming cache hints) -----------
template <typename T, int N> struct Vec;
template <> struct Vec<float, 4> {
  static __device__ __forceinline__ void ld(const float* p, float v[4]) {
    const float4 x = __ldcs(reinterpret_cast<const float4*>(p));
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  }
  static __device__ __forceinline__ void st(float* p, const float v[4]) {
    __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
  }
};
template <> struct Vec<float, 2> {
  static __device__ __forceinline__ void ld(const float* p, float v[2]) {
    const float2 x = __ldcs(reinterpret_cast<const float2*>(p));
    v[0] = x.x; v[1] = x.y;
  }
  static __device__ __forceinline__ void st(float* p, const float v[2]) {
    __stcs(reinterpret_cast<float2*>(p), make_float2(v[0], v[1]));
  }
};
template <> struct Vec<double, 2> {
  static __device__ __forceinline__ void ld(const double* p, double v[2]) {
    const double2 x = __ldcs(reinterpret_cast<const double2*>(p));
    v[0] = x.x; v[1] = x.y;
  }
  static __device__ __forceinline__ void st(double* p, const double v[2]) {
    __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
  }
};
template <> struct Vec<double, 1> {
  static __device__ __forceinline__ void ld(const double* p, double v[1]) { v[0] = __ldcs(p); }
  static __device__ __forceinline__ void st(double* p, const double v[1]) { __stcs(p, v[0]); }
};

__device__ __forceinline__ float fnan() { return __int_as_float(0x7fffffff); }
__device__ __forceinline__ double dnan() { return __longlong_as_double(0x7ff8000000000000ll); }
// Weibull's e^(ln(e)/alpha): binary32 libm, binary64 the device API's
__device__ __forceinline__ float weibull_pow(float e, float alpha) {
  return expf(logf(e) / alpha);
}
__device__ __forceinline__ double weibull_pow(double e, double alpha) {
  return brng_dev::weibull_pow_f64(e, alpha);
}

// ---- per-sample transforms (validity -> NaN + count, R-23) --------
template <int DIST, typename T>
__device__ __forceinline__ T xform(T p0, T p1, T s, uint32_t& bad) {
  const T nanv = sizeof(T) == 4 ? (T)fnan() : (T)dnan();
  if (DIST == kUniform) {                 // a + (b - a) u
    const bool ok = isfinite(p0) && isfinite(p1) && (p0 < p1);
    bad += !ok;
    return ok ? fma(p1 - p0, s, p0) : nanv;
  } else if (DIST == kGaussian) {         // mu + sigma z
    const bool ok = isfinite(p0) && isfinite(p1) && (p1 >= T(0));
    bad += !ok;
    return ok ? fma(p1, s, p0) : nanv;
  } else if (DIST == kExponential) {      // e / lambda  (rate, R-07)
    const bool ok = isfinite(p0) && (p0 > T(0));
    bad += !ok;
    return ok ? s / p0 : nanv;
  } else if (DIST == kLaplace) {          // mu + beta (+-e)
    const bool ok = isfinite(p0) && isfinite(p1) && (p1 > T(0));
    bad += !ok;
    return ok ? fma(p1, s, p0) : nanv;
  } else if (DIST == kWeibull) {          // beta e^(1/alpha)
    const bool ok = isfinite(p0) && isfinite(p1) && (p0 > T(0)) && (p1 > T(0));
    bad += !ok;
    return ok ? p1 * weibull_pow(s, p0) : nanv;
  }
  return s;
}

// ---- standard deviates of one block -----------------------------------------
// f32: 4 x u24 words (uniform / exponential / log-uniform / Weibull), two
// Box-Muller pairs (R-06) or two Laplace (exponential, sign) pairs (R-30).
template <int DIST>
__device__ __forceinline__ void std_block(uint4 w, float* s) {
  if (DIST == kGaussian) {
    float sn, cs;
    const float r0 = sqrtf(-2.0f * logf(1.0f - u24(w.x)));
    brng_dev::dm::sincos2pi_u24(w.y, &sn, &cs);
    s[0] = r0 * cs; s[1] = r0 * sn;
    const float r1 = sqrtf(-2.0f * logf(1.0f - u24(w.z)));
    brng_dev::dm::sincos2pi_u24(w.w, &sn, &cs);
    s[2] = r1 * cs; s[3] = r1 * sn;
  } else if (DIST == kLaplace) {
    const float e0 = -logf(1.0f - u24(w.x)), e1 = -logf(1.0f - u24(w.z));
    s[0] = u24(w.y) < 0.5f ? -e0 : e0;
    s[1] = u24(w.w) < 0.5f ? -e1 : e1;
  } else {
    const float u[4] = {u24(w.x), u24(w.y), u24(w.z), u24(w.w)};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (DIST == kExponential || DIST == kWeibull) s[k] = -logf(1.0f - u[k]);
      else if (DIST == kLogUniform) s[k] = logf(1.0f - u[k]);
      else s[k] = u[k];
    }
  }
}
// f64: 2 x u53 (uniform / exponential / log-uniform / Weibull), one Box-Muller
// pair, or one Laplace sample.
// (binary64 transcendentals: the table-driven brng_dev::dm functions, the same
// ones the device-API getters use, so bulk and getter results are identical)
template <int DIST>
__device__ __forceinline__ void std_block(uint4 w, double* s) {
  namespace dm = brng_dev::dm;
  if (DIST == kGaussian) {
    dm::box_muller_f64(w, &s[0], &s[1]);
  } else if (DIST == kLaplace) {
    const double e = -dm::ln1m_u53(w.x, w.y);
    s[0] = u53(w.z, w.w) < 0.5 ? -e : e;
  } else {
    const uint32_t lo[2] = {w.x, w.z}, hi[2] = {w.y, w.w};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (DIST == kExponential || DIST == kWeibull) s[k] = -dm::ln1m_u53(lo[k], hi[k]);
      else if (DIST == kLogUniform) s[k] = dm::ln1m_u53(lo[k], hi[k]);
      else s[k] = u53(lo[k], hi[k]);
    }
  }
}

// ---- kernels ------------------------------------------------------------------
#ifndef BRNG_FILL_BPT
#define BRNG_FILL_BPT 2
#endif
constexpr int kBPT = BRNG_FILL_BPT;    // Philox blocks per thread per iteration

// SCALAR: every sample uses the fixed parameters (s0, s1) -- the fixed-
// parameter "Batch" scenario of the paper's Fig. 2, 4 B/sample.
// Each thread handles kBPT blocks per iteration (stride apart): all parameter
// loads are issued before any Philox work, for memory-level parallelism.
template <typename T, int DIST, bool SCALAR = false>
__global__ void __launch_bounds__(kThreads) fill_kernel(const __grid_constant__ FillArgs<T> a) {
  constexpr int S = spb<T, DIST>();
  constexpr int NP = SCALAR ? 0 : n_params<DIST>();
  const uint64_t nblk = (a.n + S - 1) / S;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  uint32_t bad = 0;
  for (uint64_t j0 = (uint64_t)blockIdx.x * kThreads + threadIdx.x; j0 < nblk;
       j0 += kBPT * stride) {
    T p0[kBPT][S], p1[kBPT][S];
    bool full[kBPT];
#pragma unroll
    for (int b = 0; b < kBPT; ++b) {
      const uint64_t j = j0 + b * stride;
      full[b] = a.vec && (j + 1) * S <= a.n;
      if (full[b]) {
        if (NP >= 1) Vec<T, S>::ld(a.p0 + j * S, p0[b]);
        if (NP >= 2) Vec<T, S>::ld(a.p1 + j * S, p1[b]);
      }
    }
#pragma unroll
    for (int b = 0; b < kBPT; ++b) {
      const uint64_t j = j0 + b * stride;
      if (j >= nblk) break;
      const uint4 w = philox_block_rk(a.base + j, a.rk);
      T s[S];
      std_block<DIST>(w, s);
      const uint64_t i0 = j * S;
      if (full[b]) {
        T o[S];
#pragma unroll
        for (int k = 0; k < S; ++k)
          o[k] = SCALAR ? xform<DIST>(a.s0, a.s1, s[k], bad)
                        : xform<DIST>(NP >= 1 ? p0[b][k] : T(0), NP >= 2 ? p1[b][k] : T(0), s[k],
                                      bad);
        Vec<T, S>::st(a.out + i0, o);
      } else {
#pragma unroll
        for (int k = 0; k < S; ++k) {
          const uint64_t i = i0 + k;
          if (i < a.n) {
            const T q0 = SCALAR ? a.s0 : (NP >= 1 ? a.p0[i] : T(0));
            const T q1 = SCALAR ? a.s1 : (NP >= 2 ? a.p1[i] : T(0));
            a.out[i] = xform<DIST>(q0, q1, s[k], bad);
          }
        }
      }
    }
  }
  if (SCALAR || NP > 0) flush_errors(a.err, bad);
}

__global__ void __launch_bounds__(kThreads) raw_u32_kernel(const __grid_constant__ FillArgs<uint32_t> a) {
  const uint64_t nblk = (a.n + 3) >> 2;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t j = (uint64_t)blockIdx.x * kThreads + threadIdx.x; j < nblk; j += stride) {
    const uint4 w = philox_block_rk(a.base + j, a.rk);
    const uint64_t i0 = j << 2;
    if (a.vec && i0 + 4 <= a.n) {
      __stcs(reinterpret_cast<uint4*>(a.out) + j, w);
    } else {
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
      for (int k = 0; k < 4; ++k)
        if (i0 + k < a.n) a.out[i0 + k] = ww[k];
    }
  }
}

inline bool aligned(const void* p, uintptr_t bytes) {
  return p == nullptr || ((uintptr_t)p & (bytes - 1)) == 0;
}

inline unsigned grid_for(uint64_t nblk, const Ctx& ctx) {
  const uint64_t want = (nblk + (uint64_t)kThreads * kBPT - 1) / ((uint64_t)kThreads * kBPT);
  const uint64_t cap = (uint64_t)ctx.num_sms * 8 * 4;  // 8 CTAs/SM resident x 4 waves
  return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

template <typename T, int DIST>
cudaError_t run_dist(const T* p0, const T* p1, T* out, uint64_t n, uint64_t base,
                     const Ctx& ctx, const double* scalars) {
  constexpr int S = spb<T, DIST>();
  const uintptr_t vb = sizeof(T) * S;
  FillArgs<T> a{p0, p1, out, n, base, ctx.stream_id, make_round_keys(ctx.k0, ctx.k1, ctx.stream_id),
                aligned(p0, vb) && aligned(p1, vb) && aligned(out, vb), ctx.err, T(0), T(0)};
  const unsigned g = grid_for((n + S - 1) / S, ctx);
  if (scalars) {
    a.s0 = (T)scalars[0];
    a.s1 = (T)scalars[1];
    fill_kernel<T, DIST, true><<<g, kThreads, 0, ctx.stream>>>(a);
  } else {
    fill_kernel<T, DIST, false><<<g, kThreads, 0, ctx.stream>>>(a);
  }
  return cudaGetLastError();
}

template <typename T>
cudaError_t run_typed(int dist, const T* p0, const T* p1, T* out, uint64_t n, uint64_t base,
                      const Ctx& ctx, const double* sc) {
  switch (dist) {
    case kStdUniform: return run_dist<T, kStdUniform>(p0, p1, out, n, base, ctx, nullptr);
    case kUniform: return run_dist<T, kUniform>(p0, p1, out, n, base, ctx, sc);
    case kGaussian: return run_dist<T, kGaussian>(p0, p1, out, n, base, ctx, sc);
    case kExponential: return run_dist<T, kExponential>(p0, p1, out, n, base, ctx, sc);
    case kLogUniform: return run_dist<T, kLogUniform>(p0, p1, out, n, base, ctx, nullptr);
    case kLaplace: return run_dist<T, kLaplace>(p0, p1, out, n, base, ctx, sc);
    case kWeibull: return run_dist<T, kWeibull>(p0, p1, out, n, base, ctx, sc);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

int samples_per_block(int dist, int dtype) {
  if (dist == kRaw) return 4;
  if (dtype == kF64) return dist == kLaplace ? 1 : 2;
  return dist == kLaplace ? 2 : 4;
}

cudaError_t launch_fill(int dist, int dtype, const void* p0, const void* p1, void* out,
                        uint64_t n, uint64_t base, const Ctx& ctx, const double* scalars) {
  if (dist == kRaw) {
    FillArgs<uint32_t> a{nullptr, nullptr, static_cast<uint32_t*>(out), n, base, ctx.stream_id,
                         make_round_keys(ctx.k0, ctx.k1, ctx.stream_id), aligned(out, 16), ctx.err};
    raw_u32_kernel<<<grid_for((n + 3) >> 2, ctx), kThreads, 0, ctx.stream>>>(a);
    return cudaGetLastError();
  }
  if (dtype == kF32)
    return run_typed<float>(dist, static_cast<const float*>(p0), static_cast<const float*>(p1),
                            static_cast<float*>(out), n, base, ctx, scalars);
  return run_typed<double>(dist, static_cast<const double*>(p0), static_cast<const double*>(p1),
                           static_cast<double*>(out), n, base, ctx, scalars);
}

}  // namespace brng
