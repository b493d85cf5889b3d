// A "user" translation unit that draws its deviates through the public device
// API (include/brng_device.cuh) one sample at a time -- the paper's
// one-at-a-time getters called inside the consumer's own loop.  Used by
// tests/test_gpu_device_api.py to check the getters against the bulk C ABI.
#include <brng_device.cuh>

namespace {
__global__ void k_fill(int dist, uint64_t seed, uint64_t stream, uint64_t base, const double* p0,
                       const double* p1, double* out, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const brng_dev::Key k = brng_dev::make_key(seed);
  double v = 0.0;
  switch (dist) {
    case 2: v = brng_dev::uniform_f64(k, stream, base, i, p0[i], p1[i]); break;
    case 3: v = brng_dev::gaussian_f64(k, stream, base, i, p0[i], p1[i]); break;
    case 4: v = brng_dev::exponential_f64(k, stream, base, i, p0[i]); break;
    case 5: v = brng_dev::log_uniform_f64(k, stream, base, i); break;
    case 6: v = brng_dev::laplace_f64(k, stream, base, i, p0[i], p1[i]); break;
    case 7: v = brng_dev::weibull_f64(k, stream, base, i, p0[i], p1[i]); break;
  }
  out[i] = v;
}
__global__ void k_fill32(int dist, uint64_t seed, uint64_t stream, uint64_t base, const float* p0,
                         const float* p1, float* out, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const brng_dev::Key k = brng_dev::make_key(seed);
  float v = 0.0f;
  switch (dist) {
    case 2: v = brng_dev::uniform_f32(k, stream, base, i, p0[i], p1[i]); break;
    case 3: v = brng_dev::gaussian_f32(k, stream, base, i, p0[i], p1[i]); break;
    case 4: v = brng_dev::exponential_f32(k, stream, base, i, p0[i]); break;
  }
  out[i] = v;
}
__global__ void k_gamma(uint64_t seed, uint64_t stream, uint64_t base, const double* alpha,
                        const double* beta, double* out, unsigned char* trials, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t t;
  out[i] = brng_dev::gamma_f64(brng_dev::make_key(seed), stream, base, i, alpha[i], beta[i], &t);
  trials[i] = (unsigned char)t;
}
// The split trial (N4, R-33): a "producer" computes the parameter-free parts
// (trial-1 normal + word, boost log-uniform) into buffers, a "consumer"
// applies the parameters with mt_accept_z / mt_boost_from_log and runs any
// later trial with mt_trial -- must equal gamma_f64 bit for bit.
__global__ void k_gamma_split(uint64_t seed, uint64_t stream, uint64_t base, const double* alpha,
                              const double* beta, double* out, unsigned char* trials,
                              uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const brng_dev::Key k = brng_dev::make_key(seed);
  const uint64_t b0 = base + (uint64_t)brng_dev::kGammaStride * i;
  // producer part
  const uint4 w1 = brng_dev::block(k, stream, b0 + 1);
  const double z1 = brng_dev::mt_normal(w1);
  const uint32_t w3 = w1.w;
  const double L = brng_dev::mt_boost_log(brng_dev::block(k, stream, b0));
  // consumer part
  const double al = alpha[i], be = beta[i];
  double d, g = 0.0;
  unsigned t = 0;
  if (isfinite(al) && isfinite(be) && al > 0.0 && be > 0.0) {
    if (brng_dev::mt_accept_z(z1, w3, al, d, g)) {
      t = 1;
    } else {
      for (unsigned tt = 2; tt <= brng_dev::kGammaMaxTrial; ++tt)
        if (brng_dev::mt_trial(brng_dev::block(k, stream, b0 + tt), al, d, g)) { t = tt; break; }
    }
  }
  if (t == 0) { out[i] = brng_dev::nan_(); trials[i] = 0; return; }
  if (al < 1.0) g = brng_dev::mt_boost_from_log(L, g, al);
  out[i] = g * be;
  trials[i] = (unsigned char)t;
}
// Fig. 1 of the paper as a user kernel: one chain per thread.
__global__ void k_gibbs(uint64_t seed, uint64_t stream_id, uint64_t base, uint64_t n_chains,
                        uint64_t n_sweeps, double* out_x, double* out_y) {
  const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_chains) return;
  const brng_dev::Key k = brng_dev::make_key(seed);
  double x = 0.5, y = 0.5;
  for (uint64_t s = 0; s < n_sweeps; ++s) {
    brng_dev::gibbs_sweep(k, stream_id + c, base + s, x, y);
    out_x[s * n_chains + c] = x;
    out_y[s * n_chains + c] = y;
  }
}
// The table-driven binary64 math of the Gamma path (brng_dev::dm), one
// function per `fn`: 0 ln_pos(x), 1 cos2pi_u32(w), 2 exp_nonpos(x),
// 3 one_minus_u53(w[2i], w[2i+1]), 4 rsqrt_pos(x), 5 sqrt_nonneg(x),
// 6/7 sin/cos of sincos2pi_u24(w) (binary32), 8/9 sin/cos of
// sincos2pi_u53(w[2i], w[2i+1]), 10 exp_small(x), 11/12 ln(1 - u53) two ways.
__global__ void k_math(int fn, const double* x, const uint32_t* w, double* out, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  namespace dm = brng_dev::dm;
  out[i] = fn == 0 ? dm::ln_pos(x[i])
         : fn == 1 ? dm::cos2pi_u32(w[i])
         : fn == 2 ? dm::exp_nonpos(x[i])
         : fn == 3 ? dm::one_minus_u53(w[2 * i], w[2 * i + 1])
         : fn == 4 ? dm::rsqrt_pos(x[i])
         : fn == 5 ? dm::sqrt_nonneg(x[i])
                   : 0.0;
  if (fn == 6 || fn == 7) {
    float sn, cs;
    dm::sincos2pi_u24(w[i], &sn, &cs);
    out[i] = fn == 6 ? (double)sn : (double)cs;
  }
  if (fn == 8 || fn == 9) {
    double sn, cs;
    dm::sincos2pi_u53(w[2 * i], w[2 * i + 1], &sn, &cs);
    out[i] = fn == 8 ? sn : cs;
  }
  if (fn == 10) out[i] = dm::exp_small(x[i]);
  // 11 ln1m_u53 (1 - u53 converted by I2F, exponent adjusted), 12 the same
  // value through the bit-built one_minus_u53 and ln_pos
  if (fn == 11) out[i] = dm::ln1m_u53(w[2 * i], w[2 * i + 1]);
  if (fn == 12) out[i] = dm::ln_pos(dm::one_minus_u53(w[2 * i], w[2 * i + 1]));
}
// The Marsaglia-Tsang decision pieces on given Philox words: the binary32
// screen (+1/-1/0) and the exact binary64 test, for trials with 1 + cz > 0
// (screen = 2 marks 1 + cz <= 0).  Same steps as brng_dev::mt_trial.
__global__ void k_screen(const uint32_t* w, const double* alpha, signed char* screen,
                         signed char* exact, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  namespace dm = brng_dev::dm;
  const uint4 b = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
  const double L = dm::ln_pos(dm::one_minus_u53(b.x, b.y));
  const double z = __dmul_rn(dm::sqrt_nonneg(-2.0 * L), dm::cos2pi_u32(b.z));
  double d, c;
  brng_dev::mt_consts(alpha[i], d, c);
  const double t = __dadd_rn(1.0, __dmul_rn(c, z));
  if (!(t > 0.0)) { screen[i] = 2; exact[i] = 0; return; }
  const double v = __dmul_rn(__dmul_rn(t, t), t);
  screen[i] = (signed char)brng_dev::mt_screen(z, d, t, b.w);
  exact[i] = brng_dev::mt_exact(z, d, v, b.w) ? 1 : 0;
}
unsigned grid(uint64_t n) { return (unsigned)((n + 255) / 256); }
}  // namespace

extern "C" {
int dev_fill(int dist, uint64_t seed, uint64_t stream, uint64_t base, const double* p0,
             const double* p1, double* out, uint64_t n, void* s) {
  k_fill<<<grid(n), 256, 0, (cudaStream_t)s>>>(dist, seed, stream, base, p0, p1, out, n);
  return (int)cudaGetLastError();
}
int dev_fill32(int dist, uint64_t seed, uint64_t stream, uint64_t base, const float* p0,
               const float* p1, float* out, uint64_t n, void* s) {
  k_fill32<<<grid(n), 256, 0, (cudaStream_t)s>>>(dist, seed, stream, base, p0, p1, out, n);
  return (int)cudaGetLastError();
}
int dev_gamma(uint64_t seed, uint64_t stream, uint64_t base, const double* a, const double* b,
              double* out, unsigned char* tr, uint64_t n, void* s) {
  k_gamma<<<grid(n), 256, 0, (cudaStream_t)s>>>(seed, stream, base, a, b, out, tr, n);
  return (int)cudaGetLastError();
}
int dev_gamma_split(uint64_t seed, uint64_t stream, uint64_t base, const double* a,
                    const double* b, double* out, unsigned char* tr, uint64_t n, void* s) {
  k_gamma_split<<<grid(n), 256, 0, (cudaStream_t)s>>>(seed, stream, base, a, b, out, tr, n);
  return (int)cudaGetLastError();
}
int dev_math(int fn, const double* x, const uint32_t* w, double* out, uint64_t n, void* s) {
  k_math<<<grid(n), 256, 0, (cudaStream_t)s>>>(fn, x, w, out, n);
  return (int)cudaGetLastError();
}
int dev_screen(const uint32_t* w, const double* alpha, signed char* screen, signed char* exact,
               uint64_t n, void* s) {
  k_screen<<<grid(n), 256, 0, (cudaStream_t)s>>>(w, alpha, screen, exact, n);
  return (int)cudaGetLastError();
}
int dev_gibbs(uint64_t seed, uint64_t stream_id, uint64_t base, uint64_t nc, uint64_t ns,
              double* ox, double* oy, void* s) {
  k_gibbs<<<grid(nc), 256, 0, (cudaStream_t)s>>>(seed, stream_id, base, nc, ns, ox, oy);
  return (int)cudaGetLastError();
}
}
