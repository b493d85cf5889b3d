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
 *
 * A Gamma trial also splits into its parameter-free part and the part that
 * uses alpha (mt_normal + mt_accept_z; mt_boost_log + mt_boost_from_log), so
 * a producer can precompute the former into a buffer and a consumer apply
 * the latter with bit-identical results -- the "BatchRNG as asynchronous
 * service" reading R-33 (brng_lda_gibbs's RING mode does this).
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

// ---- binary64 math of the Gamma trial and boost ---------------------------------
// The Gamma path is bound by instruction issue (DESIGN.md §7 K3), and
// libdevice's log/cospi/exp/sqrt are general-purpose (special-case branches,
// 60-100 instructions each, double constants rematerialised per use).  These
// versions cover exactly the arguments the trial produces: lookup tables
// (brng_device_tables.cuh) plus short Taylor polynomials whose truncation
// error is < 1e-19, coefficients in the constant bank (DFMA reads them as
// operands), no special-case branches.  Errors are ~1-2 ulp (tests/
// test_gpu_device_api.py pins them against mpmath), far inside the 1e-12
// value tolerance, and relative-accurate where the trial needs it.
}  // namespace brng_dev
#include "brng_device_tables.cuh"
namespace brng_dev {
namespace dm {
enum {
  kL7, kL6, kL5, kL4, kL3, kL2,          // ln: 1/7, -1/6, 1/5, -1/4, 1/3, -1/2
  kLn2Hi, kLn2Lo, kRndM128,              // ln 2 split; 1.5*2^52 - 128
  kS7, kS5, kS3, kC6, kC4, kTwoPi32,     // sin/cos Taylor; 2 pi / 2^32
  kE6, kE5, kE4, kE3, kInvLn2x64, kLn2Hi64, kLn2Lo64, kRnd,
  kNewton3, kThird,                      // 3/8 (rsqrt step); 1/3 (M-T d)
  kNumConst
};
static __constant__ double kC[kNumConst] = {
    1.0 / 7.0, -1.0 / 6.0, 0.2, -0.25, 1.0 / 3.0, -0.5,
    0x1.62e42feep-1,                 // 32 significant bits: e * ln2_hi is exact
    0x1.a39ef35793c76p-33,           // ln 2 - ln2_hi
    6755399441055744.0 - 128.0,
    -1.0 / 5040.0, 1.0 / 120.0, -1.0 / 6.0, -1.0 / 720.0, 1.0 / 24.0,
    0x1.921fb54442d18p-30,           // 2 pi / 2^32
    1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0,
    0x1.71547652b82fep+6,            // 64 / ln 2
    0x1.62e42feep-7, 0x1.a39ef35793c76p-39,   // ln2_hi / 64, ln2_lo / 64
    6755399441055744.0,              // 1.5 * 2^52: round-to-integer shifter
    0.375, 1.0 / 3.0,
};
// Where the lookup tables are read from.  GlobalTables: the __device__ arrays
// through the read-only path (any user kernel).  A kernel may instead stage
// the same arrays elsewhere (e.g. shared memory) behind the same interface:
// same values, so the same results bit for bit.
struct GlobalTables {
  // constant i of kC (a table type may keep some of them in registers)
  __device__ __forceinline__ double k(int i) const { return kC[i]; }
  __device__ __forceinline__ double2 ln(int j) const { return __ldg(&tab::kLn[j]); }
  __device__ __forceinline__ double2 cs(uint32_t j) const { return __ldg(&tab::kCos[j]); }
  __device__ __forceinline__ double exp2(int j) const { return __ldg(&tab::kExp2[j]); }
};
// exact binary64 of a 32-bit signed integer: one I2F.F64.S32 (XU pipe).  The
// bit-built form (2^52 + 2^31 + v) - (2^52 + 2^31) -- the same values -- took
// an IMAD.MOV of the constant high word, a LOP3 and a DADD per use: Gamma
// 0.830 -> 0.820 ms and Dirichlet 3.964 -> 3.915 ms with the conversion
// (identical outputs; profiles/r02_i2d.txt).
__device__ __forceinline__ double i2d(int v) { return (double)v; }
// 1 - u53(lo, hi), exactly, from the bits: with k = (hi:lo) >> 11 (53 bits),
// D = 2^52 + (k mod 2^52) and t = bit 52 of k, 1 - k 2^-53 = (t ? 1 : 1.5) -
// D 2^-53 (one exact FMA; no integer->double conversion).
__device__ __forceinline__ double one_minus_u53(uint32_t lo, uint32_t hi) {
  const double D = __hiloint2double(0x43300000 | ((hi >> 11) & 0xFFFFF),
                                    (int)__funnelshift_r(lo, hi, 11));
  const double C = __hiloint2double(0x3FF80000 ^ ((hi >> 12) & 0x80000), 0);
  return fma(D, -0x1p-53, C);
}
// ln x for a positive normal x.  x = 2^e m, m in [sqrt(1/2), sqrt(2));
// j = round(128 (m-1)), c_j ~ 1/(1+j/128), r = m c_j - 1 (one rounding, |r| <
// 0.0056); ln x = e ln2 - ln c_j + log1p(r), log1p by its Taylor series to
// r^7.  c_0 = 1 and ln c_0 = 0, so for x near 1 the result is log1p(x-1)
// to ~1 ulp relative.
// ln of the positive normal binary64 with high word hx and low word lx
template <class Tab = GlobalTables>
__device__ __forceinline__ double ln_pos_bits(int hx, int lx, const Tab& tb = Tab()) {
  const int e = (hx - 0x3FE6A09E) >> 20;
  const double m = __hiloint2double(hx - e * (1 << 20), lx);
  const int j = __double2loint(fma(m, 128.0, tb.k(kRndM128)));
  const double2 ct = tb.ln(j + tab::kLnOff);
  const double r = fma(m, ct.x, -1.0);
  double q = fma(r, tb.k(kL7), kC[kL6]);
  q = fma(r, q, kC[kL5]);
  q = fma(r, q, kC[kL4]);
  q = fma(r, q, kC[kL3]);
  q = fma(r, q, kC[kL2]);
  const double de = i2d(e);
  const double lo = fma(r * r, q, de * kC[kLn2Lo]) + r;
  return fma(de, kC[kLn2Hi], ct.y) + lo;
}
template <class Tab = GlobalTables>
__device__ __forceinline__ double ln_pos(double x, const Tab& tb = Tab()) {
  return ln_pos_bits(__double2hiint(x), __double2loint(x), tb);
}
// cos(2 pi w 2^-32): j = round(w / 2^24) mod 256, b = 2 pi (w - j 2^24) 2^-32
// (|b| <= pi/256); cos(a_j + b) = C_j cos b - S_j sin b with Taylor cos b - 1
// to b^6 and sin b to b^7.  Absolute error ~1e-16.
template <class Tab = GlobalTables>
__device__ __forceinline__ double cos2pi_u32(uint32_t w, const Tab& tb = Tab()) {
  const uint32_t j = (w + 0x800000u) >> 24;
  const double b = i2d((int)(w - (j << 24))) * kC[kTwoPi32];
  const double2 cs = tb.cs(j);
  const double b2 = b * b;
  const double s = fma(b2 * b, fma(b2, fma(b2, tb.k(kS7), kC[kS5]), kC[kS3]), b);
  const double cm1 = b2 * fma(b2, fma(b2, tb.k(kC6), kC[kC4]), -0.5);
  return cs.x + fma(cs.x, cm1, -cs.y * s);
}
// e^y for finite y <= 0: k = round(64 y / ln 2), r = y - k ln2/64 (|r| <=
// 0.0055, Cody-Waite), e^y = 2^(k>>6) 2^((k&63)/64) e^r, e^r - 1 by Taylor
// to r^6.  y < -700 (result near/below the normal range) takes libdevice.
template <class Tab = GlobalTables>
__device__ __forceinline__ double exp_nonpos(double y, const Tab& tb = Tab()) {
  if (y < -700.0) return exp(y);
  const double t = fma(y, tb.k(kInvLn2x64), kC[kRnd]);
  const int k = __double2loint(t);
  const double kd = t - kC[kRnd];
  double r = fma(kd, -kC[kLn2Hi64], y);
  r = fma(kd, -kC[kLn2Lo64], r);
  double q = fma(r, tb.k(kE6), kC[kE5]);
  q = fma(r, q, kC[kE4]);
  q = fma(r, q, kC[kE3]);
  q = fma(r, q, 0.5);
  const double p = fma(r * r, q, r);
  const double T = tb.exp2(k & 63);
  const double v = fma(T, p, T);
  return __hiloint2double(__double2hiint(v) + (k >> 6) * (1 << 20), __double2loint(v));
}
// 1/sqrt(x) for a positive normal x: MUFU.RSQ64H seed (~2^-22) and one
// cubic Newton step y (1 + e/2 + 3e^2/8), e = 1 - x y^2: ~1 ulp.
template <class Tab = GlobalTables>
__device__ __forceinline__ double rsqrt_pos(double x, const Tab& tb = Tab()) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x * y, y, 1.0);
  return fma(y * e, fma(e, tb.k(kNewton3), 0.5), y);
}
// sqrt(x) for x = 0 or a positive normal: x * rsqrt(x) (~2 ulp).
template <class Tab = GlobalTables>
__device__ __forceinline__ double sqrt_nonneg(double x, const Tab& tb = Tab()) {
  return x > 0.0 ? x * rsqrt_pos(x, tb) : 0.0;
}
// ln x in binary32 by MUFU.LG2 (flushes subnormal x to 0 -> -inf).  Error
// <= 2^-22 ln2 absolute for x in [1/2, 2], else <= 2 ulp of log2 x.
__device__ __forceinline__ float ln_approx_f32(float x) {
  float l;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(x));
  return l * 0.69314718f;
}
// {sin, cos}(2 pi u24(w)), u24(w) = (w >> 8) 2^-24, in binary32: k = w >> 8,
// j = round(k / 2^18) mod 64, b = 2 pi (k - j 2^18) 2^-24 (|b| <= pi/64);
// table {C_j, S_j} (exact 0/+-1 at the quarter turns, so results near the
// zeros of sin/cos are relative-accurate) and Taylor sin b to b^5, cos b - 1
// to b^4 (truncation < 2e-11).  ~1e-7 absolute, vs ~3x the instructions of
// sincospif.
__device__ __forceinline__ void sincos2pi_u24(uint32_t w, float* sn, float* cs) {
  const uint32_t k = w >> 8;
  const uint32_t j = ((k + 0x20000u) >> 18) & 63u;
  const int rem = (int)((k - (j << 18)) << 14) >> 14;   // sign-extended 18 bits
  const float b = (float)rem * 0x1.921fb6p-22f;          // 2 pi / 2^24
  const float2 t = __ldg(&tab::kSinCos32[j]);
  const float b2 = b * b;
  const float sb = fmaf(b2 * b, fmaf(b2, 1.0f / 120.0f, -1.0f / 6.0f), b);
  const float cm1 = b2 * fmaf(b2, 1.0f / 24.0f, -0.5f);
  *cs = t.x + fmaf(t.x, cm1, -t.y * sb);
  *sn = t.y + fmaf(t.y, cm1, t.x * sb);
}
// {sin, cos}(2 pi u53(lo, hi)) for the binary64 Box-Muller angle: k = the
// 53-bit integer, j = round(k / 2^45) mod 256, rem = k - j 2^45 (|rem| <=
// 2^44, exact in binary64), b = 2 pi rem 2^-53; table {C_j, S_j} and Taylor
// sin b to b^7, cos b - 1 to b^6.  ~1e-16 absolute; exact 0/+-1 at the
// quarter turns, relative-accurate next to the zeros.
template <class Tab = GlobalTables>
__device__ __forceinline__ void sincos2pi_u53(uint32_t lo, uint32_t hi, double* sn, double* cs,
                                              const Tab& tb = Tab()) {
  const uint64_t k = ((uint64_t)hi << 21) | (lo >> 11);
  const uint32_t j = (uint32_t)((k + (1ull << 44)) >> 45) & 255u;
  const int64_t rem = (int64_t)((k - ((uint64_t)j << 45)) << 18) >> 18;
  const double b = (double)rem * 0x1.921fb54442d18p-51;     // 2 pi / 2^53
  const double2 t = tb.cs(j);
  const double b2 = b * b;
  const double sb = fma(b2 * b, fma(b2, fma(b2, kC[kS7], kC[kS5]), kC[kS3]), b);
  const double cm1 = b2 * fma(b2, fma(b2, kC[kC6], kC[kC4]), -0.5);
  *cs = t.x + fma(t.x, cm1, -t.y * sb);
  *sn = t.y + fma(t.y, cm1, t.x * sb);
}
// ln(1 - u53(lo, hi)) (<= 0; exact 0 at u = 0)
// 1 - u53 = N 2^-53 with N = 2^53 - k (k the 53-bit integer of the words),
// exact: N is converted by one I2F.F64.U64 (XU pipe) and the 2^-53 applied to
// its exponent field -- the same binary64 value as one_minus_u53, without its
// DFMA and the constant's zero low word (Gamma 0.815 -> 0.807 ms, Dirichlet
// 3.735 -> 3.693 ms, identical outputs; profiles/r02_ln1m.txt)
template <class Tab = GlobalTables>
__device__ __forceinline__ double ln1m_u53(uint32_t lo, uint32_t hi, const Tab& tb = Tab()) {
  const uint64_t k = (((uint64_t)hi << 32) | lo) >> 11;
  const double D = __ull2double_rn((1ull << 53) - k);
  return ln_pos_bits(__double2hiint(D) - (53 << 20), __double2loint(D), tb);
}
// e^y for |y| <= 700 by the table path of exp_nonpos (positive k scales the
// exponent up, no overflow below 709); libdevice beyond.
template <class Tab = GlobalTables>
__device__ __forceinline__ double exp_small(double y, const Tab& tb = Tab()) {
  if (!(fabs(y) <= 700.0)) return exp(y);
  const double t = fma(y, kC[kInvLn2x64], kC[kRnd]);
  const int k = __double2loint(t);
  const double kd = t - kC[kRnd];
  double r = fma(kd, -kC[kLn2Hi64], y);
  r = fma(kd, -kC[kLn2Lo64], r);
  double q = fma(r, kC[kE6], kC[kE5]);
  q = fma(r, q, kC[kE4]);
  q = fma(r, q, kC[kE3]);
  q = fma(r, q, 0.5);
  const double p = fma(r * r, q, r);
  const double T = tb.exp2(k & 63);
  const double v = fma(T, p, T);
  return __hiloint2double(__double2hiint(v) + (k >> 6) * (1 << 20), __double2loint(v));
}
// Box-Muller pair from one block (R-06, binary64): r = sqrt(-2 ln(1-u53(w0,
// w1))), theta = 2 pi u53(w2, w3); {r cos, r sin}.
template <class Tab = GlobalTables>
__device__ __forceinline__ void box_muller_f64(uint4 w, double* z0, double* z1,
                                               const Tab& tb = Tab()) {
  const double r = sqrt_nonneg(-2.0 * ln1m_u53(w.x, w.y, tb));
  double sn, cs;
  sincos2pi_u53(w.z, w.w, &sn, &cs, tb);
  *z0 = r * cs;
  *z1 = r * sn;
}
}  // namespace dm

// ---- Marsaglia-Tsang trial (R-08, R-09) -----------------------------------------
// d = alpha' - 1/3, c = 1/sqrt(9 d) (~1 ulp).
template <class Tab = dm::GlobalTables>
__device__ __forceinline__ void mt_consts(double alpha, double& d, double& c,
                                          const Tab& tb = Tab()) {
  const double ap = alpha < 1.0 ? alpha + 1.0 : alpha;
  d = ap - dm::kC[dm::kThird];
  c = dm::rsqrt_pos(9.0 * d, tb);
}
// The binary32 screen of the acceptance test (see mt_trial): +1 accept,
// -1 reject, 0 = margin inside the error band (decide with mt_exact).
__device__ __forceinline__ int mt_screen(double z, double d, double t, uint32_t w3) {
  const float tf = (float)t, zf = (float)z, df = (float)d;
  const float z2hf = 0.5f * zf * zf;
  const float wf = fmaf(tf * tf, tf, -1.0f);
  const float lnt = dm::ln_approx_f32(tf);
  const float lnu = dm::ln_approx_f32(fmaf(__uint2float_rn(~w3), 0x1p-32f, 0x1p-32f));
  const float m = fmaf(df, fmaf(3.0f, lnt, -wf), z2hf) - lnu;
  const float band =
      0x1p-17f * (1.0f + z2hf + df * (1.0f + fabsf(wf) + 3.0f * fabsf(lnt)) + fabsf(lnu));
  return m > band ? 1 : (m < -band ? -1 : 0);
}
// The exact binary64 test in the contract's operation order (R-09):
// ln U < ((z z) 0.5 + d) - d v + d ln v, U = 1 - u32d(w3).
__device__ __forceinline__ bool mt_exact(double z, double d, double v, uint32_t w3) {
  const double U = 1.0 - u32d(w3);
  const double rhs = __dadd_rn(__dsub_rn(__dadd_rn(__dmul_rn(__dmul_rn(z, z), 0.5), d),
                                         __dmul_rn(d, v)),
                               __dmul_rn(d, log(v)));
  return log(U) < rhs;
}
// One trial from one Philox block: z = sqrt(-2 ln(1-u53(w0,w1))) cos(2 pi
// u32d(w2)), U = 1 - u32d(w3); reject if 1+cz <= 0, else v = (1+cz)^3 and
// accept iff ln U < z^2/2 + d - d v + d ln v; g = d v (binary64 values).
//
// Decision.  A binary32 screen evaluates the margin on the form
//   m = z^2/2 + d (3 ln t - w) - ln U,   t = 1 + cz, w = t^3 - 1,
// (equal to rhs - ln U in exact arithmetic) with MUFU.LG2 logs.  Its error is
// below 2^-19.4 (1 + z^2/2 + d (1 + |w| + 3|ln t|) + |ln U|) (DESIGN.md §7:
// lg2.approx 2^-22 absolute on [1/2,2] / 2 ulp elsewhere, 2^-24 per rounding);
// margins outside 2^-17 times that sum are decided by their sign, the rest
// (~0.1% of trials) re-run the exact binary64 test in the contract's
// operation order.  Decisions are therefore the binary64 contract's.
// d is returned; alpha is consumed only after z (hides its load latency).
// The trial splits into its parameter-free part (the standard normal z of the
// block: the paper's buffered Gaussian) and the part that uses the
// sample's alpha; mt_trial is exactly their composition, so a consumer that
// gets z (and the block's word w3) from a producer's buffer (NEXT row N4,
// reading R-33) computes the same decision and value bit for bit.
template <class Tab = dm::GlobalTables>
__device__ __forceinline__ double mt_normal(uint4 w, const Tab& tb = Tab()) {
  const double L = dm::ln1m_u53(w.x, w.y, tb);
  return __dmul_rn(dm::sqrt_nonneg(-2.0 * L, tb), dm::cos2pi_u32(w.z, tb));
}
template <class Tab = dm::GlobalTables>
__device__ __forceinline__ bool mt_accept_z(double z, uint32_t w3, double alpha, double& d,
                                            double& g,
                                            const Tab& tb = Tab()) {
  double c;
  mt_consts(alpha, d, c, tb);
  const double cz = __dmul_rn(c, z);
  const double t = __dadd_rn(1.0, cz);
  if (!(t > 0.0)) return false;
  const double v = __dmul_rn(__dmul_rn(t, t), t);
  g = __dmul_rn(d, v);
  const int sc = mt_screen(z, d, t, w3);
  if (sc != 0) return sc > 0;
  return mt_exact(z, d, v, w3);
}
template <class Tab = dm::GlobalTables>
__device__ __forceinline__ bool mt_trial(uint4 w, double alpha, double& d, double& g,
                                         const Tab& tb = Tab()) {
  return mt_accept_z(mt_normal(w, tb), w.w, alpha, d, g, tb);
}
// ln(1 - u53(w0, w1)) of the boost block: the parameter-free part of the boost
// (the paper's log-uniform buffer)
template <class Tab = dm::GlobalTables>
__device__ __forceinline__ double mt_boost_log(uint4 wb, const Tab& tb = Tab()) {
  return dm::ln1m_u53(wb.x, wb.y, tb);
}
template <class Tab = dm::GlobalTables>
__device__ __forceinline__ double mt_boost_from_log(double L, double g, double alpha,
                                                    const Tab& tb = Tab()) {
  return g * dm::exp_nonpos(L / alpha, tb);
}
// alpha < 1 boost (R-10): g * exp(ln(1-u53(w0,w1)) / alpha) from block 256 i.
template <class Tab = dm::GlobalTables>
__device__ __forceinline__ double mt_boost(uint4 wb, double g, double alpha,
                                           const Tab& tb = Tab()) {
  return mt_boost_from_log(mt_boost_log(wb, tb), g, alpha, tb);
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
  dm::sincos2pi_u24(word(w, 2 * p + 1), &sn, &cs);
  return (i % 2) ? r * sn : r * cs;
}
__device__ __forceinline__ double std_gaussian_f64(const Key& k, uint64_t stream, uint64_t base,
                                                   uint64_t i) {
  const uint4 w = block(k, stream, base + i / 2);
  double z0, z1;
  dm::box_muller_f64(w, &z0, &z1);
  return (i % 2) ? z1 : z0;
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
// the word pair of binary64 sample i (two samples per block)
__device__ __forceinline__ uint2 pair_f64(const Key& k, uint64_t stream, uint64_t base,
                                          uint64_t i) {
  const uint4 w = block(k, stream, base + i / 2);
  return (i % 2) ? make_uint2(w.z, w.w) : make_uint2(w.x, w.y);
}
__device__ __forceinline__ double exponential_f64(const Key& k, uint64_t stream, uint64_t base,
                                                  uint64_t i, double lambda) {
  const uint2 p = pair_f64(k, stream, base, i);
  const double e = -dm::ln1m_u53(p.x, p.y);
  return (isfinite(lambda) && lambda > 0.0) ? e / lambda : nan_();
}
__device__ __forceinline__ double log_uniform_f64(const Key& k, uint64_t stream, uint64_t base,
                                                  uint64_t i) {
  const uint2 p = pair_f64(k, stream, base, i);
  return dm::ln1m_u53(p.x, p.y);
}
// GetLaplace (R-30): mu + beta s e; f32 words (2j, 2j+1) of block i/2, f64 block i
__device__ __forceinline__ double laplace_f64(const Key& k, uint64_t stream, uint64_t base,
                                              uint64_t i, double mu, double beta) {
  const uint4 w = block(k, stream, base + i);
  const double e = -dm::ln1m_u53(w.x, w.y);
  const double s = u53(w.z, w.w) < 0.5 ? -e : e;
  return (isfinite(mu) && isfinite(beta) && beta > 0.0) ? fma(beta, s, mu) : nan_();
}
// e^(ln(e) / alpha) of the Weibull transform (binary64): e = 0 gives 0
__device__ __forceinline__ double weibull_pow_f64(double e, double alpha) {
  return dm::exp_small((e > 0.0 ? dm::ln_pos(e) : -INFINITY) / alpha);
}
// GetWeibull (R-30): beta e^(1/alpha)
__device__ __forceinline__ double weibull_f64(const Key& k, uint64_t stream, uint64_t base,
                                              uint64_t i, double alpha, double beta) {
  const uint2 p = pair_f64(k, stream, base, i);
  const double e = -dm::ln1m_u53(p.x, p.y);
  return (isfinite(alpha) && isfinite(beta) && alpha > 0.0 && beta > 0.0)
             ? beta * weibull_pow_f64(e, alpha) : nan_();
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
