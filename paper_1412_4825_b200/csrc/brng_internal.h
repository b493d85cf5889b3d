// brng_internal.h -- launch interface between the C ABI (brng.cpp) and the
// sm_100a kernels (fill.cu, gamma.cu, gibbs.cu).  Not part of the public ABI.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace brng {

enum Dist : int {
  kRaw = 0, kStdUniform = 1, kUniform = 2, kGaussian = 3, kExponential = 4,
  kLogUniform = 5, kLaplace = 6, kWeibull = 7     // NEXT row N2 (R-30)
};
enum DType : int { kF32 = 0, kF64 = 1, kU32 = 2 };

struct Ctx {
  cudaStream_t stream;
  int num_sms;
  uint32_t k0, k1;           // Philox key = (lo32 seed, hi32 seed)
  uint64_t stream_id;        // Philox stream of fills / Gamma / Dirichlet
  unsigned long long* err;   // device invalid-sample counter
  unsigned long long* work;  // device work counter (dynamic chunk assignment)
  double* dir_scratch = nullptr;   // binary32 large-K Dirichlet: one row of Gammas per warp
};

// K1/K2: raw words, standard uniforms and per-sample-parameter transforms.
int samples_per_block(int dist, int dtype);
// scalars != nullptr: fixed parameters scalars[0..1] for every sample (batch).
cudaError_t launch_fill(int dist, int dtype, const void* p0, const void* p1, void* out,
                        uint64_t n, uint64_t base, const Ctx& ctx,
                        const double* scalars = nullptr);
// K3: Marsaglia-Tsang Gamma with warp compaction.
cudaError_t launch_gamma(int dtype, const void* alpha, const void* beta, void* out,
                         uint8_t* trials, uint64_t n, uint64_t base, const Ctx& ctx);
// K4: Dirichlet rows (Gamma + warp-shuffle normalisation).
// Doubles of scratch the binary32 large-K Dirichlet launch uses (0: none,
// the rows are recomputed instead): one row of K Gammas per resident warp.
size_t dirichlet_scratch_len(int dtype, uint64_t k, const Ctx& ctx);
cudaError_t launch_dirichlet(int dtype, const void* alpha, uint64_t n_rows, uint64_t k,
                             void* out, uint8_t* trials, uint64_t base, const Ctx& ctx);
// K5-K7: Gibbs chains + stats + histogram, then the fixed-order reduction.
// partials: device scratch of at least gibbs_partials_len(...) doubles.
size_t gibbs_partials_len(uint64_t n_chains, const Ctx& ctx);
// Chains one resident wave of the bulk Gibbs launch holds (host-staged calls
// cut chunks at multiples of it: no partly filled last round per chunk).
uint64_t gibbs_wave_chains(const Ctx& ctx);
cudaError_t launch_gibbs(uint64_t n_chains, uint64_t n_sweeps, const double* x0,
                         const double* y0, uint64_t burn_in, double* out_x, double* out_y,
                         double* chain_stats, double* final_xy, double* totals,
                         double* partials, uint64_t base, const Ctx& ctx,
                         bool accumulate_totals = false);

// NEXT row N4: LDA fold-in Gibbs consumer (lda.cu; reading R-33).
struct LdaArgs {
  uint64_t n_docs, n_tokens, base;     // base: cursor of this iteration
  uint32_t k, v;
  uint32_t k0, k1;                     // Philox key
  uint64_t stream;
  const uint64_t* doc_off;
  const uint32_t* words;
  const double* phi;                   // [v][k]
  const double* alpha;                 // [k]
  uint16_t* z;                         // [n_tokens], in/out
  double* theta_out;                   // nullable [n_docs][k]
  const double* zbuf;                  // RING slot: trial-1 normals [n_docs k]
  const uint32_t* w3buf;               //            trial-1 words   [n_docs k]
  const double* lbuf;                  //            boost ln(1-u)   [n_docs k]
  const double* ubuf;                  // RING / BULK: token uniforms [n_tokens]
  const double* theta_in;              // BULK: theta [n_docs][k]
  unsigned long long* work;
  unsigned long long* err;
};
size_t lda_consumer_smem(uint32_t k);
// src: 0 inline device-API getters, 1 ring slot, 2 bulk buffers
cudaError_t launch_lda_consumer(int src, const LdaArgs& a, const Ctx& ctx);
cudaError_t launch_lda_producer(const LdaArgs& a, double* zbuf, uint32_t* w3buf, double* lbuf,
                                double* ubuf, const Ctx& ctx, cudaStream_t s);
cudaError_t launch_lda_rows(const LdaArgs& a, double* rows, const Ctx& ctx);

}  // namespace brng
