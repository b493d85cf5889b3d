/*
 * brng_device.cuh -- header-only DEVICE API of brng (sm_100a): the paper's
 * one-at-a-time getters (GetUniform, GetGaussian,
 * GetExponential, GetLogUniform, GetLaplace, GetWeibull, GetGamma) as
 * counter-addressed __device__ functions that a user kernel calls inside its
 * own loop -- the GPU form of "BatchRNG as a service" (reading R-32):
 * with a counter-based engine there is nothing to replenish, the consumer
 * computes the deviate it needs where it needs it.
 *
 * Every function returns EXACTLY the value the corresponding bulk C-ABI call
 * (include/brng.h) produces for sample i when that call was enqueued at
 * cursor `base` on a handle with the same seed and stream_id -- same counter
 * map (R-02, R-12), same conversions and arithmetic.  Invalid parameters give
 * NaN (the device API has no error counter).
 *
 *   brng_dev::Key key = brng_dev::make_key(seed);
 *   double x = brng_dev::gaussian_f64(key, stream_id, base, i, mu, sigma);
 *
 * The library's own kernels are built from the same primitives (philox10,
 * u24/u53/u32d, mt_trial).
 */
#ifndef BRNG_DEVICE_CUH
#define BRNG_DEVICE_CUH

#include <stdint.h>
#include <cuda_runtime.h>

namespace brng_dev {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;
constexpr uint32_t kGammaStride = 256u;     // blocks reserved per Gamma sample (R-11)
constexpr uint32_t kGammaMaxTrial = 255u;

struct Key {
  uint32_t k0, k1;
};
__host__ __device__ __forceinline__ Key make_key(uint64_t seed) {
  return Key{(uint32_t)seed, (uint32_t)(seed >> 32)};
}

// ---- Philox4x32-10 (R-01, R-02) -----------------------------------------------
// One round: (c0,c1,c2,c3) -> (hi(M1 c2)^c1^k0, lo(M1 c2), hi(M0 c0)^c3^k1, lo(M0 c0)).
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
__device__ __forceinline__ uint4 philox10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r)
    c = philox_round(c, k0 + (uint32_t)r * kPhiloxW0, k1 + (uint32_t)r * kPhiloxW1);
  return c;
}
// Block `pos` of stream `stream`: counter (lo pos, hi pos, lo stream, hi stream).
__device__ __forceinline__ uint4 philox_block(uint64_t pos, uint64_t stream, uint32_t k0,
                                              uint32_t k1) {
  return philox10(make_uint4((uint32_t)pos, (uint32_t)(pos >> 32), (uint32_t)stream,
                             (uint32_t)(stream >> 32)),
                  k0, k1);
}
__device__ __forceinline__ uint4 block(const Key& k, uint64_t stream, uint64_t pos) {
  return philox_block(pos, stream, k.k0, k.k1);
}
__device__ __forceinline__ uint32_t word(const uint4& w, int j) {
  return j == 0 ? w.x : j == 1 ? w.y : j == 2 ? w.z : w.w;
}

// ---- word -> standard uniform (R-04), all exact ---------------------------------
__device__ __forceinline__ float u24(uint32_t w) { return __uint2float_rn(w >> 8) * 0x1p-24f; }
__device__ __forceinline__ double u53(uint32_t lo, uint32_t hi) {
  return fma((double)(lo >> 11), 0x1p-53, (double)hi * 0x1p-32);
}
__device__ __forceinline__ double u32d(uint32_t w) { return (double)w * 0x1p-32; }

// ---- Marsaglia-Tsang trial (R-08, R-09) -----------------------------------------
// d = alpha' - 1/3, c = 1/sqrt(9 d) (rsqrt, ~1 ulp).
__device__ __forceinline__ void mt_consts(double alpha, double& d, double& c) {
  const double ap = alpha < 1.0 ? alpha + 1.0 : alpha;
  d = ap - 1.0 / 3.0;
  c = rsqrt(9.0 * d);
}
// One trial from one Philox block: z = sqrt(-2 ln(1-u53(w0,w1))) cos(2 pi
// u32d(w2)), U = 1 - u32d(w3); reject if 1+cz <= 0, else v = (1+cz)^3 and
// accept iff ln U < z^2/2 + d - d v + d ln v; g = d v (binary64).  The
// decision is evaluated in binary32 on the cancellation-free form
// z^2/2 + d (log1p(w) - w), w = v - 1, whose error is < 1e-6 (1 + z^2/2 +
// d|w| + |ln U|); margins inside a 10x band re-run the exact binary64 test in
// the contract's operation order, so decisions are the binary64 contract's.
// d is returned; alpha is consumed only after z (hides its load latency).
__device__ __forceinline__ bool mt_trial(uint4 w, double alpha, double& d, double& g) {
  const double L = log(1.0 - u53(w.x, w.y));
  const double z = __dmul_rn(sqrt(-2.0 * L), cospi(2.0 * u32d(w.z)));
  double c;
  mt_consts(alpha, d, c);
  const double cz = __dmul_rn(c, z);
  const double t = __dadd_rn(1.0, cz);
  if (!(t > 0.0)) return false;
  const double v = __dmul_rn(__dmul_rn(t, t), t);
  g = __dmul_rn(d, v);
  const double U = 1.0 - u32d(w.w);
  const double wv = cz * (3.0 + cz * (3.0 + cz));
  const float wf = (float)wv;
  const float lf = log1pf(wf) - wf;
  const float lnu = logf((float)U);
  const double z2h = 0.5 * z * z;
  const double m = fma(d, (double)lf, z2h) - (double)lnu;
  const double band = 1e-5 * (1.0 + z2h + d * fabs(wv) + fabs((double)lnu));
  if (m > band) return true;
  if (m < -band) return false;
  const double rhs = __dadd_rn(__dsub_rn(__dadd_rn(__dmul_rn(__dmul_rn(z, z), 0.5), d),
                                         __dmul_rn(d, v)),
                               __dmul_rn(d, log(v)));
  return log(U) < rhs;
}
// alpha < 1 boost (R-10): g * exp(ln(1-u53(w0,w1)) / alpha) from block 256 i.
__device__ __forceinline__ double mt_boost(uint4 wb, double g, double alpha) {
  return g * exp(log(1.0 - u53(wb.x, wb.y)) / alpha);
}

// ---- per-sample getters: value of sample i of the bulk call at cursor base --------
__device__ __forceinline__ float nanf_() { return __int_as_float(0x7fffffff); }
__device__ __forceinline__ double nan_() { return __longlong_as_double(0x7ff8000000000000ll); }

__device__ __forceinline__ float std_uniform_f32(const Key& k, uint64_t stream, uint64_t base,
                                                 uint64_t i) {
  return u24(word(block(k, stream, base + i / 4), (int)(i % 4)));
}
__device__ __forceinline__ double std_uniform_f64(const Key& k, uint64_t stream, uint64_t base,
                                                  uint64_t i) {
  const uint4 w = block(k, stream, base + i / 2);
  return (i % 2) ? u53(w.z, w.w) : u53(w.x, w.y);
}
// GetUniform: a + (b - a) u
__device__ __forceinline__ float uniform_f32(const Key& k, uint64_t stream, uint64_t base,
                                             uint64_t i, float a, float b) {
  const float u = std_uniform_f32(k, stream, base, i);
  return (isfinite(a) && isfinite(b) && a < b) ? fmaf(b - a, u, a) : nanf_();
}
__device__ __forceinline__ double uniform_f64(const Key& k, uint64_t stream, uint64_t base,
                                              uint64_t i, double a, double b) {
  const double u = std_uniform_f64(k, stream, base, i);
  return (isfinite(a) && isfinite(b) && a < b) ? fma(b - a, u, a) : nan_();
}
// GetGaussian (R-06): Box-Muller, f32 pairs (2p, 2p+1) of block i/4, f64 block i/2
__device__ __forceinline__ float std_gaussian_f32(const Key& k, uint64_t stream, uint64_t base,
                                                  uint64_t i) {
  const uint4 w = block(k, stream, base + i / 4);
  const int p = (int)((i % 4) / 2);
  const float r = sqrtf(-2.0f * logf(1.0f - u24(word(w, 2 * p))));
  float sn, cs;
  sincospif(2.0f * u24(word(w, 2 * p + 1)), &sn, &cs);
  return (i % 2) ? r * sn : r * cs;
}
__device__ __forceinline__ double std_gaussian_f64(const Key& k, uint64_t stream, uint64_t base,
                                                   uint64_t i) {
  const uint4 w = block(k, stream, base + i / 2);
  const double r = sqrt(-2.0 * log(1.0 - u53(w.x, w.y)));
  double sn, cs;
  sincospi(2.0 * u53(w.z, w.w), &sn, &cs);
  return (i % 2) ? r * sn : r * cs;
}
__device__ __forceinline__ float gaussian_f32(const Key& k, uint64_t stream, uint64_t base,
                                              uint64_t i, float mu, float sigma) {
  const float z = std_gaussian_f32(k, stream, base, i);
  return (isfinite(mu) && isfinite(sigma) && sigma >= 0.0f) ? fmaf(sigma, z, mu) : nanf_();
}
__device__ __forceinline__ double gaussian_f64(const Key& k, uint64_t stream, uint64_t base,
                                               uint64_t i, double mu, double sigma) {
  const double z = std_gaussian_f64(k, stream, base, i);
  return (isfinite(mu) && isfinite(sigma) && sigma >= 0.0) ? fma(sigma, z, mu) : nan_();
}
// GetExponential (R-07, rate lambda) and GetLogUniform
__device__ __forceinline__ float exponential_f32(const Key& k, uint64_t stream, uint64_t base,
                                                 uint64_t i, float lambda) {
  const float e = -logf(1.0f - std_uniform_f32(k, stream, base, i));
  return (isfinite(lambda) && lambda > 0.0f) ? e / lambda : nanf_();
}
__device__ __forceinline__ double exponential_f64(const Key& k, uint64_t stream, uint64_t base,
                                                  uint64_t i, double lambda) {
  const double e = -log(1.0 - std_uniform_f64(k, stream, base, i));
  return (isfinite(lambda) && lambda > 0.0) ? e / lambda : nan_();
}
__device__ __forceinline__ double log_uniform_f64(const Key& k, uint64_t stream, uint64_t base,
                                                  uint64_t i) {
  return log(1.0 - std_uniform_f64(k, stream, base, i));
}
// GetLaplace (R-30): mu + beta s e; f32 words (2j, 2j+1) of block i/2, f64 block i
__device__ __forceinline__ double laplace_f64(const Key& k, uint64_t stream, uint64_t base,
                                              uint64_t i, double mu, double beta) {
  const uint4 w = block(k, stream, base + i);
  const double e = -log(1.0 - u53(w.x, w.y));
  const double s = u53(w.z, w.w) < 0.5 ? -e : e;
  return (isfinite(mu) && isfinite(beta) && beta > 0.0) ? fma(beta, s, mu) : nan_();
}
// GetWeibull (R-30): beta e^(1/alpha)
__device__ __forceinline__ double weibull_f64(const Key& k, uint64_t stream, uint64_t base,
                                              uint64_t i, double alpha, double beta) {
  const double e = -log(1.0 - std_uniform_f64(k, stream, base, i));
  return (isfinite(alpha) && isfinite(beta) && alpha > 0.0 && beta > 0.0)
             ? beta * exp(log(e) / alpha) : nan_();
}
// GetGamma (R-08..R-11): shape alpha, scale beta; *trial = accepting trial
// (0 when invalid / capped).  Trials run sequentially here; the bulk kernel
// runs the same per-sample trials under warp compaction.
__device__ __forceinline__ double gamma_f64(const Key& k, uint64_t stream, uint64_t base,
                                            uint64_t i, double alpha, double beta,
                                            uint32_t* trial = nullptr) {
  if (trial) *trial = 0;
  if (!(isfinite(alpha) && isfinite(beta) && alpha > 0.0 && beta > 0.0)) return nan_();
  const uint64_t b0 = base + (uint64_t)kGammaStride * i;
  for (uint32_t t = 1; t <= kGammaMaxTrial; ++t) {
    double d, g;
    if (mt_trial(block(k, stream, b0 + t), alpha, d, g)) {
      if (trial) *trial = t;
      if (alpha < 1.0) g = mt_boost(block(k, stream, b0), g, alpha);
      return g * beta;
    }
  }
  return nan_();
}
// One Gibbs sweep on the triangle (R-16): chain stream, block pos.
__device__ __forceinline__ void gibbs_sweep(const Key& k, uint64_t stream, uint64_t pos,
                                            double& x, double& y) {
  const uint4 w = block(k, stream, pos);
  x = __dmul_rn(__dsub_rn(1.0, y), u53(w.x, w.y));
  y = __dmul_rn(__dsub_rn(1.0, x), u53(w.z, w.w));
}

}  // namespace brng_dev

#endif  // BRNG_DEVICE_CUH
