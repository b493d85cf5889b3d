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
constexpr uint64_t kChunk = 1024;          // samples per warp queue (Gamma)
constexpr uint32_t kStride = 256;          // blocks per sample (R-11)
constexpr uint32_t kMaxTrial = 255;
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ll); }

// One Marsaglia-Tsang trial from one Philox block.  The squeeze
// U < 1 - 0.0331 z^4 is an exact subset of the acceptance region, so it only
// skips the two logarithms; the decision is the contract's.
__device__ __forceinline__ bool mt_trial(uint4 w, double d, double c, double& g) {
  const double L = log(1.0 - u53(w.x, w.y));
  const double z = sqrt(-2.0 * L) * cospi(2.0 * u32d(w.z));
  const double t = fma(c, z, 1.0);
  if (!(t > 0.0)) return false;
  const double v = t * t * t;
  const double U = 1.0 - u32d(w.w);
  const double z2 = z * z;
  if (U < 1.0 - 0.0331 * (z2 * z2)) { g = d * v; return true; }
  if (log(U) < 0.5 * z2 + d - d * v + d * log(v)) { g = d * v; return true; }
  return false;
}

// Warp-cooperative Gamma queue over sample indices [beg, end).
//   load(i, alpha, beta)  -- parameters of sample i
//   sink(i, value, trial) -- value = g * beta (NaN when invalid / capped)
// All 32 lanes must call it (ballots use the full mask).
template <typename Load, typename Sink>
__device__ __forceinline__ void mt_queue(uint64_t beg, uint64_t end, uint64_t base,
                                         uint64_t stream, uint32_t k0, uint32_t k1, Load load,
                                         Sink sink, uint32_t& nbad) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t head = beg + 32;
  uint64_t i = beg + lane;
  bool active = i < end;
  double alpha = 1.0, beta = 1.0, d = 0.0, c = 0.0;
  bool valid = false;
  uint32_t t = 1;
  auto setup = [&]() {
    load(i, alpha, beta);
    valid = isfinite(alpha) && isfinite(beta) && alpha > 0.0 && beta > 0.0;
    const double ap = alpha < 1.0 ? alpha + 1.0 : alpha;
    d = ap - 1.0 / 3.0;
    c = 1.0 / sqrt(9.0 * d);
    t = 1;
  };
  if (active) setup();
  while (__any_sync(kFull, active)) {
    bool done = false;
    double g = 0.0;
    if (active) {
      if (!valid) {
        done = true; t = 0; ++nbad;
      } else {
        const uint4 w = philox_block(base + (uint64_t)kStride * i + t, stream, k0, k1);
        if (mt_trial(w, d, c, g)) {
          done = true;
        } else if (++t > kMaxTrial) {
          done = true; t = 0; ++nbad;
        }
      }
      if (done) {
        double val = qnan();
        if (t != 0) {
          if (alpha < 1.0) {  // U^(1/alpha) boost (R-10)
            const uint4 wb = philox_block(base + (uint64_t)kStride * i, stream, k0, k1);
            g = g * exp(log(1.0 - u53(wb.x, wb.y)) / alpha);
          }
          val = g * beta;
        }
        sink(i, val, t);
      }
    }
    const uint32_t dm = __ballot_sync(kFull, done);
    if (done) {
      i = head + __popc(dm & lanemask_lt());
      active = i < end;
      if (active) setup();
    }
    head += __popc(dm);
  }
}

template <typename T>
struct GammaArgs {
  const T* alpha;
  const T* beta;
  T* out;
  uint8_t* trials;
  uint64_t n, base, stream;
  uint32_t k0, k1;
  unsigned long long* err;
};

template <typename T>
__global__ void __launch_bounds__(kThreads) gamma_kernel(GammaArgs<T> a) {
  const uint64_t warp = ((uint64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint64_t n_warps = ((uint64_t)gridDim.x * kThreads) >> 5;
  uint32_t nbad = 0;
  for (uint64_t beg = warp * kChunk; beg < a.n; beg += n_warps * kChunk) {
    const uint64_t end = beg + kChunk < a.n ? beg + kChunk : a.n;
    mt_queue(
        beg, end, a.base, a.stream, a.k0, a.k1,
        [&](uint64_t i, double& al, double& be) {
          al = (double)__ldg(a.alpha + i);
          be = (double)__ldg(a.beta + i);
        },
        [&](uint64_t i, double v, uint32_t t) {
          a.out[i] = (T)v;
          if (a.trials) a.trials[i] = (uint8_t)t;
        },
        nbad);
  }
  flush_errors(a.err, nbad);
}

template <typename T>
struct DirArgs {
  const T* alpha;
  T* out;
  uint8_t* trials;
  uint64_t n_rows, k, base, stream;
  uint32_t k0, k1;
  unsigned long long* err;
};

constexpr int kDirThreads = 128;     // 4 warps / CTA, one row per warp
constexpr uint64_t kDirSmemK = 2048; // rows up to this K are staged in smem

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  return s;
}

// K <= kDirSmemK: Gammas of the row staged in shared memory (8 K bytes/warp),
// summed lane-strided then by a fixed xor-shuffle tree, normalised, stored
// coalesced.
template <typename T>
__global__ void __launch_bounds__(kDirThreads) dirichlet_smem_kernel(DirArgs<T> a) {
  extern __shared__ double gsm[];
  const uint32_t lane = threadIdx.x & 31;
  double* g_row = gsm + (threadIdx.x >> 5) * a.k;
  const uint64_t warp = ((uint64_t)blockIdx.x * kDirThreads + threadIdx.x) >> 5;
  const uint64_t n_warps = ((uint64_t)gridDim.x * kDirThreads) >> 5;
  uint32_t nbad = 0;
  for (uint64_t row = warp; row < a.n_rows; row += n_warps) {
    const uint64_t beg = row * a.k;
    mt_queue(
        beg, beg + a.k, a.base, a.stream, a.k0, a.k1,
        [&](uint64_t i, double& al, double& be) {
          al = (double)__ldg(a.alpha + i);
          be = 1.0;
        },
        [&](uint64_t i, double v, uint32_t t) {
          g_row[i - beg] = v;
          if (a.trials) a.trials[i] = (uint8_t)t;
        },
        nbad);
    __syncwarp();
    double s = 0.0;
    for (uint64_t j = lane; j < a.k; j += 32) s += g_row[j];
    s = warp_sum(s);
    const double inv = 1.0 / s;
    for (uint64_t j = lane; j < a.k; j += 32) a.out[beg + j] = (T)(g_row[j] * inv);
    __syncwarp();
  }
  flush_errors(a.err, nbad);
}

// Any K: two passes over the row's Gamma samples (the second recomputes them
// from their counters -- exact, no scratch).
template <typename T>
__global__ void __launch_bounds__(kDirThreads) dirichlet_2pass_kernel(DirArgs<T> a) {
  const uint64_t warp = ((uint64_t)blockIdx.x * kDirThreads + threadIdx.x) >> 5;
  const uint64_t n_warps = ((uint64_t)gridDim.x * kDirThreads) >> 5;
  uint32_t nbad = 0, nbad2 = 0;
  for (uint64_t row = warp; row < a.n_rows; row += n_warps) {
    const uint64_t beg = row * a.k;
    auto load = [&](uint64_t i, double& al, double& be) {
      al = (double)__ldg(a.alpha + i);
      be = 1.0;
    };
    double s = 0.0;
    mt_queue(beg, beg + a.k, a.base, a.stream, a.k0, a.k1, load,
             [&](uint64_t, double v, uint32_t) { s += v; }, nbad);
    s = warp_sum(s);
    const double inv = 1.0 / s;
    mt_queue(beg, beg + a.k, a.base, a.stream, a.k0, a.k1, load,
             [&](uint64_t i, double v, uint32_t t) {
               a.out[i] = (T)(v * inv);
               if (a.trials) a.trials[i] = (uint8_t)t;
             },
             nbad2);
  }
  flush_errors(a.err, nbad);
}

template <typename T>
cudaError_t gamma_typed(const T* alpha, const T* beta, T* out, uint8_t* trials, uint64_t n,
                        uint64_t base, const Ctx& ctx) {
  GammaArgs<T> a{alpha, beta, out, trials, n, base, ctx.stream_id, ctx.k0, ctx.k1, ctx.err};
  const uint64_t warps_needed = (n + kChunk - 1) / kChunk;
  const uint64_t ctas_needed = (warps_needed + (kThreads / 32) - 1) / (kThreads / 32);
  const uint64_t cap = (uint64_t)ctx.num_sms * 8;  // one full-occupancy wave
  const unsigned g = (unsigned)(ctas_needed < cap ? ctas_needed : cap);
  gamma_kernel<T><<<g, kThreads, 0, ctx.stream>>>(a);
  return cudaGetLastError();
}

template <typename T>
cudaError_t dirichlet_typed(const T* alpha, uint64_t n_rows, uint64_t k, T* out,
                            uint8_t* trials, uint64_t base, const Ctx& ctx) {
  DirArgs<T> a{alpha, out, trials, n_rows, k, base, ctx.stream_id, ctx.k0, ctx.k1, ctx.err};
  const uint64_t ctas_needed = (n_rows + 3) / 4;
  if (k <= kDirSmemK) {
    const size_t smem = (size_t)4 * k * sizeof(double);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(dirichlet_smem_kernel<T>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
    }
    const uint64_t cap = (uint64_t)ctx.num_sms * 16 * 8;
    const unsigned g = (unsigned)(ctas_needed < cap ? ctas_needed : cap);
    dirichlet_smem_kernel<T><<<g, kDirThreads, smem, ctx.stream>>>(a);
  } else {
    const uint64_t cap = (uint64_t)ctx.num_sms * 16 * 8;
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

cudaError_t launch_dirichlet(int dtype, const void* alpha, uint64_t n_rows, uint64_t k,
                             void* out, uint8_t* trials, uint64_t base, const Ctx& ctx) {
  if (dtype == kF32)
    return dirichlet_typed<float>(static_cast<const float*>(alpha), n_rows, k,
                                  static_cast<float*>(out), trials, base, ctx);
  return dirichlet_typed<double>(static_cast<const double*>(alpha), n_rows, k,
                                 static_cast<double*>(out), trials, base, ctx);
}

}  // namespace brng
