// fake_kernels.cpp -- TEST INFRASTRUCTURE ONLY: stand-ins for the sm_100a
// launches (paper_1412_4825_b200/csrc/brng_internal.h) used by the host-logic
// sanitizer harness.  Each "kernel" runs on the host at launch time and
// writes a value that encodes the GLOBAL unit it was given (from the cursor /
// stream the C ABI passed for the chunk, plus the chunk-local index) and the
// staged inputs, so the driver can check that every chunk was launched at the
// right counter position with the right slices of the caller's arrays.
#include <cstring>

#include "../../paper_1412_4825_b200/csrc/brng_internal.h"

namespace brng {

int samples_per_block(int dist, int dtype) {     // the contract's span rule (include/brng.h)
  if (dist == kRaw) return 4;
  if (dtype == kF64) return dist == kLaplace ? 1 : 2;
  return dist == kLaplace ? 2 : 4;
}

double fake_fill_value(uint64_t g, double p0, double p1) {
  return (double)(g % 1000003u) + p0 + 2.0 * p1;
}

cudaError_t launch_fill(int dist, int dtype, const void* p0, const void* p1, void* out,
                        uint64_t n, uint64_t base, const Ctx&, const double* scalars) {
  const uint64_t per = (uint64_t)samples_per_block(dist, dtype);
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t g = base * per + i;          // global sample index (cursor 0 call)
    double a = 0.0, b = 0.0;
    if (scalars) {
      a = scalars[0]; b = scalars[1];
    } else if (dtype == kF64) {
      if (p0) a = static_cast<const double*>(p0)[i];
      if (p1) b = static_cast<const double*>(p1)[i];
    } else if (dtype == kF32) {
      if (p0) a = static_cast<const float*>(p0)[i];
      if (p1) b = static_cast<const float*>(p1)[i];
    }
    const double v = fake_fill_value(g, a, b);
    if (dtype == kF64) static_cast<double*>(out)[i] = v;
    else if (dtype == kF32) static_cast<float*>(out)[i] = (float)v;
    else static_cast<uint32_t*>(out)[i] = (uint32_t)g;
  }
  return cudaSuccess;
}

cudaError_t launch_gamma(int dtype, const void* alpha, const void* beta, void* out,
                         uint8_t* trials, uint64_t n, uint64_t base, const Ctx&) {
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t g = base / 256 + i;
    double a, b;
    if (dtype == kF64) {
      a = static_cast<const double*>(alpha)[i]; b = static_cast<const double*>(beta)[i];
    } else {
      a = static_cast<const float*>(alpha)[i]; b = static_cast<const float*>(beta)[i];
    }
    const double v = fake_fill_value(g, a, b);
    if (dtype == kF64) static_cast<double*>(out)[i] = v;
    else static_cast<float*>(out)[i] = (float)v;
    if (trials) trials[i] = (uint8_t)(g & 0xff);
  }
  return cudaSuccess;
}

size_t dirichlet_scratch_len(int dtype, uint64_t k, const Ctx& ctx) {
  return (dtype == kF32 && k > 1024) ? (size_t)ctx.num_sms * 4 * 4 * k : 0;
}

cudaError_t launch_dirichlet(int dtype, const void* alpha, uint64_t n_rows, uint64_t k,
                             void* out, uint8_t* trials, uint64_t base, const Ctx& ctx) {
  if (dirichlet_scratch_len(dtype, k, ctx) && ctx.dir_scratch)   // touch the whole scratch
    std::memset(ctx.dir_scratch, 0, dirichlet_scratch_len(dtype, k, ctx) * sizeof(double));
  for (uint64_t i = 0; i < n_rows * k; ++i) {
    const uint64_t g = base / 256 + i;
    const double a = dtype == kF64 ? static_cast<const double*>(alpha)[i]
                                   : (double)static_cast<const float*>(alpha)[i];
    const double v = fake_fill_value(g, a, 0.0);
    if (dtype == kF64) static_cast<double*>(out)[i] = v;
    else static_cast<float*>(out)[i] = (float)v;
    if (trials) trials[i] = (uint8_t)(g & 0xff);
  }
  return cudaSuccess;
}

uint64_t gibbs_wave_chains(const Ctx& ctx) { return (uint64_t)ctx.num_sms * 2 * 256 * 3; }
size_t gibbs_partials_len(uint64_t, const Ctx& ctx) { return (size_t)ctx.num_sms * 2 * 272; }

cudaError_t launch_gibbs(uint64_t n_chains, uint64_t n_sweeps, const double* x0,
                         const double* y0, uint64_t, double* out_x, double* out_y,
                         double* chain_stats, double* final_xy, double* totals,
                         double* partials, uint64_t base, const Ctx& ctx,
                         bool accumulate_totals) {
  std::memset(partials, 0, gibbs_partials_len(n_chains, ctx) * sizeof(double));
  for (uint64_t c = 0; c < n_chains; ++c) {
    const double id = (double)(ctx.stream_id + c);          // global chain (stream)
    const double x = x0 ? x0[c] : 0.5, y = y0 ? y0[c] : 0.5;
    for (uint64_t s = 0; s < n_sweeps; ++s) {
      if (out_x) out_x[s * n_chains + c] = id + 1e-3 * (double)(base + s) + x;
      if (out_y) out_y[s * n_chains + c] = id + 1e-3 * (double)(base + s) + y;
    }
    if (chain_stats)
      for (int q = 0; q < 5; ++q) chain_stats[q * n_chains + c] = 10.0 * id + q;
    if (final_xy) { final_xy[c] = id; final_xy[n_chains + c] = -id; }
  }
  if (totals) {
    if (!accumulate_totals) std::memset(totals, 0, 272 * sizeof(double));
    totals[8] += (double)n_chains;
    totals[9] += (double)(n_chains * n_sweeps);
  }
  return cudaSuccess;
}

size_t lda_consumer_smem(uint32_t k) { return (size_t)4 * k * 12; }
cudaError_t launch_lda_consumer(int, const LdaArgs&, const Ctx&) { return cudaSuccess; }
cudaError_t launch_lda_producer(const LdaArgs&, double*, uint32_t*, double*, double*, const Ctx&,
                                cudaStream_t) {
  return cudaSuccess;
}
cudaError_t launch_lda_rows(const LdaArgs&, double*, const Ctx&) { return cudaSuccess; }

}  // namespace brng
