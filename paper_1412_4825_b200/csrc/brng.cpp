// brng.cpp -- the C ABI (include/brng.h): handle, cursor, validation, host
// buffer staging and kernel launches.  The handle is the GPU recast of the
// paper's BatchRNG object: engine state = (seed,
// stream_id, block cursor); the "buffer counter" is the Philox block cursor,
// advanced at enqueue time (R-12).
#include "../../include/brng.h"

#include <cuda_runtime.h>

#include <limits>
#include <new>
#include <vector>

#include "brng_internal.h"

struct brng_handle_s {
  uint64_t seed;
  uint64_t stream_id;
  uint64_t cursor;
  int device;
  int num_sms;
  cudaStream_t stream;
  unsigned long long* d_err;   // invalid-sample counter
  double* d_partials;          // Gibbs per-CTA partials
  size_t partials_cap;         // in doubles
};

namespace {

using brng::Ctx;

int cuda_status(cudaError_t e) { return e == cudaSuccess ? BRNG_OK : BRNG_ERR_CUDA; }

Ctx make_ctx(brng_t h) {
  Ctx c;
  c.stream = h->stream;
  c.num_sms = h->num_sms;
  c.k0 = (uint32_t)h->seed;
  c.k1 = (uint32_t)(h->seed >> 32);
  c.stream_id = h->stream_id;
  c.err = h->d_err;
  return c;
}

int check_device(brng_t h) {
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return BRNG_ERR_CUDA;
  if (dev != h->device) {
    // Launch on the handle's device regardless of the caller's current device.
    if (cudaSetDevice(h->device) != cudaSuccess) return BRNG_ERR_STATE;
  }
  return BRNG_OK;
}

// span = ceil(n / per) * mult with overflow checks; cursor + span <= 2^64.
int reserve(brng_t h, uint64_t n, uint64_t per, uint64_t mult, uint64_t* base) {
  const uint64_t blocks = n / per + (n % per != 0);
  if (mult != 0 && blocks > std::numeric_limits<uint64_t>::max() / mult) return BRNG_ERR_OVERFLOW;
  const uint64_t span = blocks * mult;
  if (span > std::numeric_limits<uint64_t>::max() - h->cursor) return BRNG_ERR_OVERFLOW;
  *base = h->cursor;
  return BRNG_OK;
}
void commit(brng_t h, uint64_t n, uint64_t per, uint64_t mult) {
  h->cursor += (n / per + (n % per != 0)) * mult;
}

bool is_device_ptr(const void* p) {
  if (p == nullptr) return true;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Host-buffer staging (include/brng.h "Pointers"): host inputs are copied to
// stream-ordered device allocations, host outputs are copied back after the
// kernel, and the call synchronises before returning.
struct Stage {
  cudaStream_t s;
  struct Out { void* host; void* dev; size_t bytes; };
  std::vector<void*> allocs;
  std::vector<Out> outs;
  bool any_host = false;
  cudaError_t err = cudaSuccess;

  explicit Stage(cudaStream_t st) : s(st) {}
  const void* in(const void* p, size_t bytes) {
    if (p == nullptr || bytes == 0 || is_device_ptr(p)) return p;
    any_host = true;
    void* d = nullptr;
    if (err == cudaSuccess) err = cudaMallocAsync(&d, bytes, s);
    if (err == cudaSuccess) { allocs.push_back(d); err = cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, s); }
    return d;
  }
  void* out(void* p, size_t bytes) {
    if (p == nullptr || bytes == 0 || is_device_ptr(p)) return p;
    any_host = true;
    void* d = nullptr;
    if (err == cudaSuccess) err = cudaMallocAsync(&d, bytes, s);
    if (err == cudaSuccess) { allocs.push_back(d); outs.push_back({p, d, bytes}); }
    return d;
  }
  cudaError_t finish(cudaError_t launch) {
    if (err == cudaSuccess) err = launch;
    for (auto& o : outs)
      if (err == cudaSuccess) err = cudaMemcpyAsync(o.host, o.dev, o.bytes, cudaMemcpyDeviceToHost, s);
    for (void* d : allocs) cudaFreeAsync(d, s);
    if (any_host) {
      cudaError_t e2 = cudaStreamSynchronize(s);
      if (err == cudaSuccess) err = e2;
    }
    return err;
  }
};

bool mul_ok(uint64_t a, uint64_t b) { return b == 0 || a <= std::numeric_limits<uint64_t>::max() / b; }

int fill_common(brng_t h, int dist, int dtype, const void* p0, const void* p1, void* out,
                uint64_t n, size_t esize) {
  if (!h || !out) return BRNG_ERR_NULL;
  if ((dist == brng::kUniform || dist == brng::kGaussian) && (!p0 || !p1)) return BRNG_ERR_NULL;
  if (dist == brng::kExponential && !p0) return BRNG_ERR_NULL;
  if (n == 0) return BRNG_OK;
  if (!mul_ok(n, esize)) return BRNG_ERR_SIZE;
  int st = check_device(h);
  if (st) return st;
  const uint64_t per = (dtype == brng::kF64) ? 2 : 4;
  uint64_t base;
  if ((st = reserve(h, n, per, 1, &base))) return st;
  Stage sg(h->stream);
  const size_t bytes = (size_t)n * esize;
  const void* d0 = sg.in(p0, p0 ? bytes : 0);
  const void* d1 = sg.in(p1, p1 ? bytes : 0);
  void* dout = sg.out(out, bytes);
  cudaError_t e = sg.err == cudaSuccess
                      ? brng::launch_fill(dist, dtype, d0, d1, dout, n, base, make_ctx(h))
                      : sg.err;
  e = sg.finish(e);
  if (e != cudaSuccess) return BRNG_ERR_CUDA;
  commit(h, n, per, 1);
  return BRNG_OK;
}

int gamma_common(brng_t h, int dtype, const void* alpha, const void* beta, void* out,
                 uint64_t n, uint8_t* trials, size_t esize) {
  if (!h || !alpha || !beta || !out) return BRNG_ERR_NULL;
  if (n == 0) return BRNG_OK;
  if (!mul_ok(n, esize)) return BRNG_ERR_SIZE;
  int st = check_device(h);
  if (st) return st;
  uint64_t base;
  if ((st = reserve(h, n, 1, BRNG_GAMMA_STRIDE, &base))) return st;
  Stage sg(h->stream);
  const size_t bytes = (size_t)n * esize;
  const void* da = sg.in(alpha, bytes);
  const void* db = sg.in(beta, bytes);
  void* dout = sg.out(out, bytes);
  uint8_t* dtr = static_cast<uint8_t*>(sg.out(trials, trials ? (size_t)n : 0));
  cudaError_t e = sg.err == cudaSuccess
                      ? brng::launch_gamma(dtype, da, db, dout, dtr, n, base, make_ctx(h))
                      : sg.err;
  e = sg.finish(e);
  if (e != cudaSuccess) return BRNG_ERR_CUDA;
  commit(h, n, 1, BRNG_GAMMA_STRIDE);
  return BRNG_OK;
}

int dirichlet_common(brng_t h, int dtype, const void* alpha, uint64_t n_rows, uint64_t k,
                     void* out, uint8_t* trials, size_t esize) {
  if (!h || !alpha || !out) return BRNG_ERR_NULL;
  if (k == 0) return BRNG_ERR_SIZE;
  if (n_rows == 0) return BRNG_OK;
  if (!mul_ok(n_rows, k)) return BRNG_ERR_SIZE;
  const uint64_t n = n_rows * k;
  if (!mul_ok(n, esize)) return BRNG_ERR_SIZE;
  int st = check_device(h);
  if (st) return st;
  uint64_t base;
  if ((st = reserve(h, n, 1, BRNG_GAMMA_STRIDE, &base))) return st;
  Stage sg(h->stream);
  const size_t bytes = (size_t)n * esize;
  const void* da = sg.in(alpha, bytes);
  void* dout = sg.out(out, bytes);
  uint8_t* dtr = static_cast<uint8_t*>(sg.out(trials, trials ? (size_t)n : 0));
  cudaError_t e = sg.err == cudaSuccess
                      ? brng::launch_dirichlet(dtype, da, n_rows, k, dout, dtr, base, make_ctx(h))
                      : sg.err;
  e = sg.finish(e);
  if (e != cudaSuccess) return BRNG_ERR_CUDA;
  commit(h, n, 1, BRNG_GAMMA_STRIDE);
  return BRNG_OK;
}

}  // namespace

extern "C" {

int brng_version(void) { return BRNG_VERSION; }

const char* brng_status_string(int s) {
  switch (s) {
    case BRNG_OK: return "ok";
    case BRNG_ERR_NULL: return "null handle or pointer";
    case BRNG_ERR_SIZE: return "invalid size";
    case BRNG_ERR_CUDA: return "CUDA runtime error";
    case BRNG_ERR_PARAM: return "invalid parameter";
    case BRNG_ERR_OVERFLOW: return "Philox cursor overflow";
    case BRNG_ERR_STATE: return "handle used on another device";
    default: return "unknown status";
  }
}

int brng_create(uint64_t seed, uint64_t stream_id, brng_t* out) {
  if (!out) return BRNG_ERR_NULL;
  *out = nullptr;
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return BRNG_ERR_CUDA;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return BRNG_ERR_CUDA;
  brng_handle_s* h = new (std::nothrow) brng_handle_s();
  if (!h) return BRNG_ERR_CUDA;
  h->seed = seed; h->stream_id = stream_id; h->cursor = 0;
  h->device = dev; h->num_sms = sms; h->stream = nullptr;
  h->d_partials = nullptr; h->partials_cap = 0;
  if (cudaMalloc(&h->d_err, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemset(h->d_err, 0, sizeof(unsigned long long)) != cudaSuccess) {
    delete h;
    return BRNG_ERR_CUDA;
  }
  *out = h;
  return BRNG_OK;
}

int brng_destroy(brng_t h) {
  if (!h) return BRNG_ERR_NULL;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  cudaFree(h->d_err);
  if (h->d_partials) cudaFree(h->d_partials);
  delete h;
  return BRNG_OK;
}

int brng_set_cuda_stream(brng_t h, void* s) {
  if (!h) return BRNG_ERR_NULL;
  h->stream = static_cast<cudaStream_t>(s);
  return BRNG_OK;
}
int brng_get_offset(brng_t h, uint64_t* c) {
  if (!h || !c) return BRNG_ERR_NULL;
  *c = h->cursor;
  return BRNG_OK;
}
int brng_set_offset(brng_t h, uint64_t c) {
  if (!h) return BRNG_ERR_NULL;
  h->cursor = c;
  return BRNG_OK;
}
int brng_get_key(brng_t h, uint64_t* seed, uint64_t* stream_id) {
  if (!h || !seed || !stream_id) return BRNG_ERR_NULL;
  *seed = h->seed; *stream_id = h->stream_id;
  return BRNG_OK;
}
int brng_synchronize(brng_t h) {
  if (!h) return BRNG_ERR_NULL;
  return cuda_status(cudaStreamSynchronize(h->stream));
}
int brng_device_errors(brng_t h, uint64_t* n) {
  if (!h || !n) return BRNG_ERR_NULL;
  unsigned long long v = 0;
  cudaError_t e = cudaMemcpyAsync(&v, h->d_err, sizeof(v), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  *n = v;
  return cuda_status(e);
}
int brng_reset_device_errors(brng_t h) {
  if (!h) return BRNG_ERR_NULL;
  return cuda_status(cudaMemsetAsync(h->d_err, 0, sizeof(unsigned long long), h->stream));
}

int brng_raw_u32(brng_t h, uint32_t* out, uint64_t n) {
  return fill_common(h, brng::kRaw, brng::kU32, nullptr, nullptr, out, n, 4);
}
int brng_std_uniform_f32(brng_t h, float* out, uint64_t n) {
  return fill_common(h, brng::kStdUniform, brng::kF32, nullptr, nullptr, out, n, 4);
}
int brng_std_uniform_f64(brng_t h, double* out, uint64_t n) {
  return fill_common(h, brng::kStdUniform, brng::kF64, nullptr, nullptr, out, n, 8);
}
int brng_uniform_f32(brng_t h, const float* a, const float* b, float* out, uint64_t n) {
  return fill_common(h, brng::kUniform, brng::kF32, a, b, out, n, 4);
}
int brng_uniform_f64(brng_t h, const double* a, const double* b, double* out, uint64_t n) {
  return fill_common(h, brng::kUniform, brng::kF64, a, b, out, n, 8);
}
int brng_gaussian_f32(brng_t h, const float* mu, const float* sigma, float* out, uint64_t n) {
  return fill_common(h, brng::kGaussian, brng::kF32, mu, sigma, out, n, 4);
}
int brng_gaussian_f64(brng_t h, const double* mu, const double* sigma, double* out, uint64_t n) {
  return fill_common(h, brng::kGaussian, brng::kF64, mu, sigma, out, n, 8);
}
int brng_exponential_f32(brng_t h, const float* lambda, float* out, uint64_t n) {
  return fill_common(h, brng::kExponential, brng::kF32, lambda, nullptr, out, n, 4);
}
int brng_exponential_f64(brng_t h, const double* lambda, double* out, uint64_t n) {
  return fill_common(h, brng::kExponential, brng::kF64, lambda, nullptr, out, n, 8);
}

int brng_gamma_f32(brng_t h, const float* alpha, const float* beta, float* out, uint64_t n,
                   uint8_t* trials) {
  return gamma_common(h, brng::kF32, alpha, beta, out, n, trials, 4);
}
int brng_gamma_f64(brng_t h, const double* alpha, const double* beta, double* out, uint64_t n,
                   uint8_t* trials) {
  return gamma_common(h, brng::kF64, alpha, beta, out, n, trials, 8);
}
int brng_dirichlet_f32(brng_t h, const float* alpha, uint64_t n_rows, uint64_t k, float* out,
                       uint8_t* trials) {
  return dirichlet_common(h, brng::kF32, alpha, n_rows, k, out, trials, 4);
}
int brng_dirichlet_f64(brng_t h, const double* alpha, uint64_t n_rows, uint64_t k, double* out,
                       uint8_t* trials) {
  return dirichlet_common(h, brng::kF64, alpha, n_rows, k, out, trials, 8);
}

int brng_gibbs_triangle(brng_t h, uint64_t n_chains, uint64_t n_sweeps, const double* x0,
                        const double* y0, uint64_t burn_in, double* out_x, double* out_y,
                        double* chain_stats, double* final_xy, double* totals) {
  if (!h) return BRNG_ERR_NULL;
  if (burn_in > n_sweeps) return BRNG_ERR_SIZE;
  if (n_sweeps >= (1ull << 23)) return BRNG_ERR_SIZE;   // u32 shared histogram bound
  if (n_chains == 0) return BRNG_OK;
  if (!mul_ok(n_chains, n_sweeps) || !mul_ok(n_chains * n_sweeps, 8) || !mul_ok(n_chains, 40))
    return BRNG_ERR_SIZE;
  if (n_chains > std::numeric_limits<uint64_t>::max() - h->stream_id) return BRNG_ERR_OVERFLOW;
  int st = check_device(h);
  if (st) return st;
  uint64_t base;
  if ((st = reserve(h, n_sweeps, 1, 1, &base))) return st;
  Ctx ctx = make_ctx(h);
  const size_t need = brng::gibbs_partials_len(n_chains, ctx);
  if (need > h->partials_cap) {
    if (h->d_partials) {
      cudaStreamSynchronize(h->stream);
      cudaFree(h->d_partials);
      h->d_partials = nullptr; h->partials_cap = 0;
    }
    if (cudaMalloc(&h->d_partials, need * sizeof(double)) != cudaSuccess) return BRNG_ERR_CUDA;
    h->partials_cap = need;
  }
  Stage sg(h->stream);
  const size_t nc8 = (size_t)n_chains * 8;
  const double* dx0 = static_cast<const double*>(sg.in(x0, x0 ? nc8 : 0));
  const double* dy0 = static_cast<const double*>(sg.in(y0, y0 ? nc8 : 0));
  double* dox = static_cast<double*>(sg.out(out_x, out_x ? nc8 * n_sweeps : 0));
  double* doy = static_cast<double*>(sg.out(out_y, out_y ? nc8 * n_sweeps : 0));
  double* dst = static_cast<double*>(sg.out(chain_stats, chain_stats ? nc8 * 5 : 0));
  double* dfx = static_cast<double*>(sg.out(final_xy, final_xy ? nc8 * 2 : 0));
  double* dtot = static_cast<double*>(sg.out(totals, totals ? BRNG_TOTALS_LEN * 8 : 0));
  cudaError_t e = sg.err == cudaSuccess
                      ? brng::launch_gibbs(n_chains, n_sweeps, dx0, dy0, burn_in, dox, doy, dst,
                                           dfx, dtot, h->d_partials, base, ctx)
                      : sg.err;
  e = sg.finish(e);
  if (e != cudaSuccess) return BRNG_ERR_CUDA;
  commit(h, n_sweeps, 1, 1);
  return BRNG_OK;
}

}  // extern "C"
