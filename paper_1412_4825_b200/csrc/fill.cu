// fill.cu -- K1/K2: Philox words, standard uniforms and the per-sample
// transforms of the reducible distributions ("a + (b - a) * x",
// P:L69 GetUniform/GetGaussian/GetExponential, P:L87-92 parameters read per
// sample from memory), as ONE fused streaming pass on sm_100a:
//
//   Philox4x32-10 block (4 words, registers) -> 4 f32 / 2 f64 standard
//   deviates -> 128-bit streaming parameter loads -> per-sample transform ->
//   128-bit streaming store.
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
  const T* p0;   // a | mu | lambda (nullable for raw/std)
  const T* p1;   // b | sigma
  T* out;
  uint64_t n;
  uint64_t base;
  uint64_t stream;
  uint32_t k0, k1;
  int vec;       // all arrays 16-byte aligned
  unsigned long long* err;
};

// ---- per-sample transforms (validity -> NaN + count, R-23) -------
template <int DIST>
__device__ __forceinline__ float xform(float p0, float p1, float s, uint32_t& bad) {
  if (DIST == kUniform) {
    const bool ok = isfinite(p0) && isfinite(p1) && (p0 < p1);
    bad += !ok;
    return ok ? fmaf(p1 - p0, s, p0) : __int_as_float(0x7fffffff);
  } else if (DIST == kGaussian) {
    const bool ok = isfinite(p0) && isfinite(p1) && (p1 >= 0.0f);
    bad += !ok;
    return ok ? fmaf(p1, s, p0) : __int_as_float(0x7fffffff);
  } else if (DIST == kExponential) {
    const bool ok = isfinite(p0) && (p0 > 0.0f);
    bad += !ok;
    return ok ? (-logf(1.0f - s)) / p0 : __int_as_float(0x7fffffff);
  }
  return s;
}
template <int DIST>
__device__ __forceinline__ double xform(double p0, double p1, double s, uint32_t& bad) {
  if (DIST == kUniform) {
    const bool ok = isfinite(p0) && isfinite(p1) && (p0 < p1);
    bad += !ok;
    return ok ? fma(p1 - p0, s, p0) : __longlong_as_double(0x7ff8000000000000ll);
  } else if (DIST == kGaussian) {
    const bool ok = isfinite(p0) && isfinite(p1) && (p1 >= 0.0);
    bad += !ok;
    return ok ? fma(p1, s, p0) : __longlong_as_double(0x7ff8000000000000ll);
  } else if (DIST == kExponential) {
    const bool ok = isfinite(p0) && (p0 > 0.0);
    bad += !ok;
    return ok ? (-log(1.0 - s)) / p0 : __longlong_as_double(0x7ff8000000000000ll);
  }
  return s;
}

// ---- standard deviates of one block ----------------------------------------
// f32: four u24 uniforms, or two Box-Muller pairs (R-06).
template <int DIST>
__device__ __forceinline__ void std4(uint4 w, float s[4]) {
  if (DIST == kGaussian) {
    float sn, cs;
    const float r0 = sqrtf(-2.0f * logf(1.0f - u24(w.x)));
    sincospif(2.0f * u24(w.y), &sn, &cs);
    s[0] = r0 * cs; s[1] = r0 * sn;
    const float r1 = sqrtf(-2.0f * logf(1.0f - u24(w.z)));
    sincospif(2.0f * u24(w.w), &sn, &cs);
    s[2] = r1 * cs; s[3] = r1 * sn;
  } else {
    s[0] = u24(w.x); s[1] = u24(w.y); s[2] = u24(w.z); s[3] = u24(w.w);
  }
}
// f64: two u53 uniforms, or one Box-Muller pair.
template <int DIST>
__device__ __forceinline__ void std2(uint4 w, double s[2]) {
  if (DIST == kGaussian) {
    double sn, cs;
    const double r = sqrt(-2.0 * log(1.0 - u53(w.x, w.y)));
    sincospi(2.0 * u53(w.z, w.w), &sn, &cs);
    s[0] = r * cs; s[1] = r * sn;
  } else {
    s[0] = u53(w.x, w.y); s[1] = u53(w.z, w.w);
  }
}

// ---- kernels ------------------------------------------------------------------
template <int DIST>
__global__ void __launch_bounds__(kThreads) fill_f32_kernel(FillArgs<float> a) {
  const uint64_t nblk = (a.n + 3) >> 2;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  uint32_t bad = 0;
  for (uint64_t j = (uint64_t)blockIdx.x * kThreads + threadIdx.x; j < nblk; j += stride) {
    const uint4 w = philox_block(a.base + j, a.stream, a.k0, a.k1);
    float s[4];
    std4<DIST>(w, s);
    const uint64_t i0 = j << 2;
    if (a.vec && i0 + 4 <= a.n) {
      float4 p0 = make_float4(0.f, 0.f, 0.f, 0.f), p1 = p0;
      if (DIST == kUniform || DIST == kGaussian || DIST == kExponential)
        p0 = __ldcs(reinterpret_cast<const float4*>(a.p0) + j);
      if (DIST == kUniform || DIST == kGaussian)
        p1 = __ldcs(reinterpret_cast<const float4*>(a.p1) + j);
      float4 o;
      o.x = xform<DIST>(p0.x, p1.x, s[0], bad);
      o.y = xform<DIST>(p0.y, p1.y, s[1], bad);
      o.z = xform<DIST>(p0.z, p1.z, s[2], bad);
      o.w = xform<DIST>(p0.w, p1.w, s[3], bad);
      __stcs(reinterpret_cast<float4*>(a.out) + j, o);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t i = i0 + k;
        if (i < a.n) {
          const float p0 = (DIST >= kUniform) ? a.p0[i] : 0.f;
          const float p1 = (DIST == kUniform || DIST == kGaussian) ? a.p1[i] : 0.f;
          a.out[i] = xform<DIST>(p0, p1, s[k], bad);
        }
      }
    }
  }
  if (DIST >= kUniform) flush_errors(a.err, bad);
}

template <int DIST>
__global__ void __launch_bounds__(kThreads) fill_f64_kernel(FillArgs<double> a) {
  const uint64_t nblk = (a.n + 1) >> 1;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  uint32_t bad = 0;
  for (uint64_t j = (uint64_t)blockIdx.x * kThreads + threadIdx.x; j < nblk; j += stride) {
    const uint4 w = philox_block(a.base + j, a.stream, a.k0, a.k1);
    double s[2];
    std2<DIST>(w, s);
    const uint64_t i0 = j << 1;
    if (a.vec && i0 + 2 <= a.n) {
      double2 p0 = make_double2(0.0, 0.0), p1 = p0;
      if (DIST >= kUniform) p0 = __ldcs(reinterpret_cast<const double2*>(a.p0) + j);
      if (DIST == kUniform || DIST == kGaussian)
        p1 = __ldcs(reinterpret_cast<const double2*>(a.p1) + j);
      double2 o;
      o.x = xform<DIST>(p0.x, p1.x, s[0], bad);
      o.y = xform<DIST>(p0.y, p1.y, s[1], bad);
      __stcs(reinterpret_cast<double2*>(a.out) + j, o);
    } else {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const uint64_t i = i0 + k;
        if (i < a.n) {
          const double p0 = (DIST >= kUniform) ? a.p0[i] : 0.0;
          const double p1 = (DIST == kUniform || DIST == kGaussian) ? a.p1[i] : 0.0;
          a.out[i] = xform<DIST>(p0, p1, s[k], bad);
        }
      }
    }
  }
  if (DIST >= kUniform) flush_errors(a.err, bad);
}

__global__ void __launch_bounds__(kThreads) raw_u32_kernel(FillArgs<uint32_t> a) {
  const uint64_t nblk = (a.n + 3) >> 2;
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  for (uint64_t j = (uint64_t)blockIdx.x * kThreads + threadIdx.x; j < nblk; j += stride) {
    const uint4 w = philox_block(a.base + j, a.stream, a.k0, a.k1);
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

inline bool aligned16(const void* p) { return p == nullptr || ((uintptr_t)p & 15u) == 0; }

inline unsigned grid_for(uint64_t nblk, const Ctx& ctx) {
  const uint64_t want = (nblk + kThreads - 1) / kThreads;
  const uint64_t cap = (uint64_t)ctx.num_sms * 8 * 4;  // 8 CTAs/SM resident x 4 waves
  return (unsigned)(want < cap ? (want ? want : 1) : cap);
}

template <typename T>
cudaError_t run_typed(int dist, const T* p0, const T* p1, T* out, uint64_t n, uint64_t base,
                      const Ctx& ctx);

template <>
cudaError_t run_typed<float>(int dist, const float* p0, const float* p1, float* out, uint64_t n,
                             uint64_t base, const Ctx& ctx) {
  FillArgs<float> a{p0, p1, out, n, base, ctx.stream_id, ctx.k0, ctx.k1,
                    aligned16(p0) && aligned16(p1) && aligned16(out), ctx.err};
  const unsigned g = grid_for((n + 3) >> 2, ctx);
  switch (dist) {
    case kStdUniform: fill_f32_kernel<kStdUniform><<<g, kThreads, 0, ctx.stream>>>(a); break;
    case kUniform: fill_f32_kernel<kUniform><<<g, kThreads, 0, ctx.stream>>>(a); break;
    case kGaussian: fill_f32_kernel<kGaussian><<<g, kThreads, 0, ctx.stream>>>(a); break;
    case kExponential: fill_f32_kernel<kExponential><<<g, kThreads, 0, ctx.stream>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <>
cudaError_t run_typed<double>(int dist, const double* p0, const double* p1, double* out,
                              uint64_t n, uint64_t base, const Ctx& ctx) {
  FillArgs<double> a{p0, p1, out, n, base, ctx.stream_id, ctx.k0, ctx.k1,
                     aligned16(p0) && aligned16(p1) && aligned16(out), ctx.err};
  const unsigned g = grid_for((n + 1) >> 1, ctx);
  switch (dist) {
    case kStdUniform: fill_f64_kernel<kStdUniform><<<g, kThreads, 0, ctx.stream>>>(a); break;
    case kUniform: fill_f64_kernel<kUniform><<<g, kThreads, 0, ctx.stream>>>(a); break;
    case kGaussian: fill_f64_kernel<kGaussian><<<g, kThreads, 0, ctx.stream>>>(a); break;
    case kExponential: fill_f64_kernel<kExponential><<<g, kThreads, 0, ctx.stream>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fill(int dist, int dtype, const void* p0, const void* p1, void* out,
                        uint64_t n, uint64_t base, const Ctx& ctx) {
  if (dist == kRaw) {
    FillArgs<uint32_t> a{nullptr, nullptr, static_cast<uint32_t*>(out), n, base, ctx.stream_id,
                         ctx.k0, ctx.k1, aligned16(out), ctx.err};
    raw_u32_kernel<<<grid_for((n + 3) >> 2, ctx), kThreads, 0, ctx.stream>>>(a);
    return cudaGetLastError();
  }
  if (dtype == kF32)
    return run_typed<float>(dist, static_cast<const float*>(p0), static_cast<const float*>(p1),
                            static_cast<float*>(out), n, base, ctx);
  return run_typed<double>(dist, static_cast<const double*>(p0), static_cast<const double*>(p1),
                           static_cast<double*>(out), n, base, ctx);
}

}  // namespace brng
