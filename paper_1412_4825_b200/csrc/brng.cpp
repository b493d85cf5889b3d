// brng.cpp -- the C ABI (include/brng.h): handle, cursor, validation, host
// buffer staging and kernel launches.  The handle is the GPU recast of the
// paper's BatchRNG object: engine state = (seed,
// stream_id, block cursor); the "buffer counter" is the Philox block cursor,
// advanced at enqueue time (R-12).
//
// Host buffers are streamed through the GPU in chunks with a three-stream
// pipeline (H2D copy stream -> kernel on the handle's stream -> D2H copy
// stream, two staging slots), so PCIe transfers in both directions overlap
// each other and the kernels.  Chunks are cut on sample (fills: Philox-block;
// Dirichlet: row; Gibbs: chain) boundaries and every chunk is launched at the
// cursor / stream its first unit has in the unchunked call, so every sample,
// per-chain statistic, final state and histogram count is identical to a
// device-pointer call.  The Gibbs moment totals (totals[0..7]) are sums over
// chains whose order depends on the chunking (each chunk's K7 sum is added to
// the running totals), so they agree to rounding (~1e-15 relative), not bit
// for bit.
#include "../../include/brng.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <new>
#include <vector>

#include "brng_internal.h"

namespace {
// Staging slots per handle: H2D may run this many chunks ahead of D2H.  More
// than double buffering matters when the handle's kernels share the GPU with
// another stream's long launches: the chunks that became ready during such a
// launch then all run back to back at its boundary (6 x 64 MB per array).
#ifndef BRNG_STAGE_SLOTS
#define BRNG_STAGE_SLOTS 6
#endif
constexpr int kSlots = BRNG_STAGE_SLOTS;
constexpr size_t kChunkBytes = size_t(64) << 20;     // target staging chunk per array
}  // namespace

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
  double* d_totals;            // Gibbs totals scratch for host `totals` pointers
  double* d_dir_scratch;       // binary32 large-K Dirichlet rows (grown on demand)
  size_t dir_scratch_cap;      // in doubles
  cudaEvent_t ev_switch;       // orders work across brng_set_cuda_stream
  // host-staging pipeline (created on the first host-pointer call)
  cudaStream_t s_in, s_out;
  cudaEvent_t ev_in[kSlots], ev_k[kSlots], ev_out[kSlots];
  void* stage[kSlots];
  size_t stage_cap;
  int stage_n;                 // slots allocated (at stage_cap bytes each)
  bool pipe_ready;
  // scratch buffers replaced by a larger one stay allocated until
  // brng_destroy: a CUDA graph captured earlier may still reference them
  std::vector<void*> retired;
  // LDA consumer (NEXT row N4): producer stream, ring / bulk scratch
  bool lda_ready;
  cudaStream_t s_prod;
  cudaEvent_t ev_prod[2], ev_cons[2], ev_lda;
  void* lda_buf;
  size_t lda_cap;              // bytes
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
  c.work = h->d_err + 1;
  return c;
}

// Makes the handle's device current for one C-ABI call and restores the
// caller's current device when the call returns (the library never leaves a
// different device current behind).
class DeviceGuard {
 public:
  explicit DeviceGuard(brng_t h) {
    if (cudaGetDevice(&prev_) != cudaSuccess) {
      status_ = BRNG_ERR_CUDA;
      return;
    }
    if (prev_ != h->device) {
      if (cudaSetDevice(h->device) != cudaSuccess) {
        status_ = BRNG_ERR_STATE;
        return;
      }
      changed_ = true;
    }
  }
  ~DeviceGuard() {
    if (changed_) cudaSetDevice(prev_);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
  int status() const { return status_; }

 private:
  int prev_ = -1;
  bool changed_ = false;
  int status_ = BRNG_OK;
};

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

bool mul_ok(uint64_t a, uint64_t b) {
  return b == 0 || a <= std::numeric_limits<uint64_t>::max() / b;
}

// One array of a call.  A unit is a sample / row / chain; an array holds
// `rows` rows of n_units * unit_bytes bytes (rows > 1: Gibbs [k][n_chains]).
struct Arr {
  const void* ptr;
  size_t unit_bytes;
  bool out;
  size_t rows = 1;
  bool host = false;
  size_t slot_off = 0;        // offset of this array inside a staging slot
};

// BRNG_TRACE=1: host-staged calls report enqueue / wait times on stderr
// (diagnostics for the host-buffer path; off by default).
bool trace_on() {
  static const bool on = [] {
    const char* v = std::getenv("BRNG_TRACE");
    return v != nullptr && v[0] == '1';
  }();
  return on;
}

// Stream-capture state of the handle's stream (scratch growth must not
// synchronise or free inside a capture).
bool capturing(brng_t h) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(h->stream, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone;
}

// Grow a handle-owned device scratch to at least `need` elements of `esize`
// bytes.  The old buffer is retired (kept until brng_destroy), never freed
// here, so graphs captured with it stay valid and no synchronisation is
// needed.  Returns false when the allocation fails.
bool grow_scratch(brng_t h, void** buf, size_t* cap, size_t need, size_t esize) {
  if (need <= *cap) return true;
  void* nb = nullptr;
  if (cudaMalloc(&nb, need * esize) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (*buf) h->retired.push_back(*buf);
  *buf = nb;
  *cap = need;
  return true;
}

int ensure_pipe(brng_t h, size_t slot_bytes, int n_slots) {
  if (!h->pipe_ready) {
    if (cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking) != cudaSuccess)
      return BRNG_ERR_CUDA;
    for (int b = 0; b < kSlots; ++b) {
      if (cudaEventCreateWithFlags(&h->ev_in[b], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&h->ev_k[b], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&h->ev_out[b], cudaEventDisableTiming) != cudaSuccess)
        return BRNG_ERR_CUDA;
      h->stage[b] = nullptr;
    }
    h->stage_cap = 0;
    h->stage_n = 0;
    h->pipe_ready = true;
  }
  // staging slots are reused across calls: earlier transfers on the copy
  // streams must be done before a slot is freed
  if (slot_bytes > h->stage_cap) {
    cudaStreamSynchronize(h->s_in);
    cudaStreamSynchronize(h->s_out);
    for (int b = 0; b < kSlots; ++b) {
      if (h->stage[b]) cudaFree(h->stage[b]);
      h->stage[b] = nullptr;
    }
    h->stage_cap = slot_bytes;
    h->stage_n = 0;
  }
  // only as many slots as the call has chunks (a one-chunk call needs one)
  for (; h->stage_n < n_slots; ++h->stage_n)
    if (cudaMalloc(&h->stage[h->stage_n], h->stage_cap) != cudaSuccess) return BRNG_ERR_CUDA;
  return BRNG_OK;
}

// Launch callback for units [u0, u0 + nu) with per-array device pointers.
using Launch =
    std::function<cudaError_t(uint64_t u0, uint64_t nu, const std::vector<void*>& dptr, bool first)>;

// Run a call over n_units.  All-device arrays: one direct launch on the
// handle's stream (asynchronous).  Any host array: chunked pipeline; returns
// after every host output is written.
// max_units (0 = none) caps a chunk below the byte target.
// soft_align: `align` is a performance preference (may be dropped), not a
// counter-alignment requirement.
int run(brng_t h, std::vector<Arr>& arrs, uint64_t n_units, uint64_t align, const Launch& launch,
        uint64_t max_units = 0, bool soft_align = false) {
  auto prefer_only_align_ok = [&](uint64_t al, size_t w) {
    return !soft_align || (uint64_t)w <= kChunkBytes / al;
  };
  bool any_host = false;
  for (auto& a : arrs) {
    a.host = a.ptr != nullptr && !is_device_ptr(a.ptr);
    any_host |= a.host;
  }
  // chunked runs launch on chunk-local [rows][chunk] layouts, so multi-row
  // DEVICE arrays are staged too (copies use cudaMemcpyDefault / UVA)
  if (any_host)
    for (auto& a : arrs)
      if (a.ptr != nullptr && a.rows > 1) a.host = true;
  if (!any_host) {
    std::vector<void*> d;
    for (auto& a : arrs) d.push_back(const_cast<void*>(a.ptr));
    return cuda_status(launch(0, n_units, d, true));
  }
  // chunk: <= kChunkBytes of the widest host array, a multiple of align
  size_t widest = 1;
  for (auto& a : arrs)
    if (a.host) widest = std::max(widest, a.unit_bytes * a.rows);
  // an alignment that is only a performance preference (Gibbs: whole
  // resident waves) is dropped when one aligned chunk would exceed the byte
  // target (host out_x/out_y rows: a wave of chains x n_sweeps x 8 B)
  if (align > 1 && !prefer_only_align_ok(align, widest)) align = 1;
  uint64_t chunk = std::max<uint64_t>(align, (kChunkBytes / widest) / align * align);
  if (max_units) chunk = std::min<uint64_t>(chunk, std::max<uint64_t>(align, max_units / align * align));
  chunk = std::min<uint64_t>(chunk, n_units);
  size_t slot = 0;
  for (auto& a : arrs)
    if (a.host) {
      a.slot_off = slot;
      slot += (a.unit_bytes * a.rows * chunk + 255) & ~size_t(255);
    }
  const auto t_beg = std::chrono::steady_clock::now();
  const uint64_t n_chunks = (n_units + chunk - 1) / chunk;
  int st = ensure_pipe(h, slot, (int)std::min<uint64_t>(kSlots, n_chunks));
  if (st) return st;
  // the first copies must not overtake earlier work of this handle's stream
  cudaError_t e = cudaEventRecord(h->ev_k[0], h->stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(h->s_in, h->ev_k[0], 0);
  for (uint64_t j = 0; j < n_chunks && e == cudaSuccess; ++j) {
    const int b = (int)(j % kSlots);
    const uint64_t u0 = j * chunk, nu = std::min(chunk, n_units - u0);
    char* base = static_cast<char*>(h->stage[b]);
    if (j >= kSlots) e = cudaStreamWaitEvent(h->s_in, h->ev_out[b], 0);   // slot free again
    std::vector<void*> d;
    for (auto& a : arrs) {
      if (!a.host) {
        d.push_back(a.ptr ? static_cast<char*>(const_cast<void*>(a.ptr)) + u0 * a.unit_bytes
                          : nullptr);
        continue;
      }
      char* dp = base + a.slot_off;
      d.push_back(dp);
      if (!a.out && e == cudaSuccess) {
        const char* hp = static_cast<const char*>(a.ptr) + u0 * a.unit_bytes;
        e = cudaMemcpy2DAsync(dp, nu * a.unit_bytes, hp, n_units * a.unit_bytes,
                              nu * a.unit_bytes, a.rows, cudaMemcpyDefault, h->s_in);
      }
    }
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_in[b], h->s_in);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->stream, h->ev_in[b], 0);
    if (e == cudaSuccess) e = launch(u0, nu, d, j == 0);
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_k[b], h->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->s_out, h->ev_k[b], 0);
    for (size_t k = 0; k < arrs.size() && e == cudaSuccess; ++k) {
      const Arr& a = arrs[k];
      if (!a.host || !a.out) continue;
      char* hp = static_cast<char*>(const_cast<void*>(a.ptr)) + u0 * a.unit_bytes;
      e = cudaMemcpy2DAsync(hp, n_units * a.unit_bytes, d[k], nu * a.unit_bytes,
                            nu * a.unit_bytes, a.rows, cudaMemcpyDefault, h->s_out);
    }
    if (e == cudaSuccess) e = cudaEventRecord(h->ev_out[b], h->s_out);
  }
  const auto t_enq = std::chrono::steady_clock::now();
  cudaError_t e2 = cudaStreamSynchronize(h->s_out);
  cudaError_t e3 = cudaStreamSynchronize(h->stream);
  if (trace_on()) {
    const auto t_end = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[brng] staged call: %llu units, %llu chunks, enqueue %.2f ms, wait %.2f ms\n",
                 (unsigned long long)n_units, (unsigned long long)n_chunks,
                 std::chrono::duration<double, std::milli>(t_enq - t_beg).count(),
                 std::chrono::duration<double, std::milli>(t_end - t_enq).count());
  }
  if (e == cudaSuccess) e = e2;
  if (e == cudaSuccess) e = e3;
  return cuda_status(e);
}

int fill_common(brng_t h, int dist, int dtype, const void* p0, const void* p1, void* out,
                uint64_t n, size_t esize) {
  if (!h || !out) return BRNG_ERR_NULL;
  if ((dist == brng::kUniform || dist == brng::kGaussian || dist == brng::kLaplace ||
       dist == brng::kWeibull) && (!p0 || !p1))
    return BRNG_ERR_NULL;
  if (dist == brng::kExponential && !p0) return BRNG_ERR_NULL;
  if (n == 0) return BRNG_OK;
  if (!mul_ok(n, esize)) return BRNG_ERR_SIZE;
  DeviceGuard dg(h);
  int st = dg.status();
  if (st) return st;
  const uint64_t per = (uint64_t)brng::samples_per_block(dist, dtype);
  uint64_t base;
  if ((st = reserve(h, n, per, 1, &base))) return st;
  std::vector<Arr> arrs = {{p0, esize, false}, {p1, esize, false}, {out, esize, true}};
  const Ctx ctx = make_ctx(h);
  st = run(h, arrs, n, per, [&](uint64_t u0, uint64_t nu, const std::vector<void*>& d, bool) {
    return brng::launch_fill(dist, dtype, d[0], d[1], d[2], nu, base + u0 / per, ctx);
  });
  if (st) return st;
  commit(h, n, per, 1);
  return BRNG_OK;
}

// Fixed-parameter batch fill (the paper's VSL-Batch scenario).
int batch_common(brng_t h, int dist, int dtype, double p0, double p1, void* out, uint64_t n) {
  if (!h || !out) return BRNG_ERR_NULL;
  if (dist < brng::kUniform || dist > brng::kWeibull || dist == brng::kLogUniform)
    return BRNG_ERR_PARAM;
  if (dtype != brng::kF32 && dtype != brng::kF64) return BRNG_ERR_PARAM;
  if (n == 0) return BRNG_OK;
  const size_t esize = dtype == brng::kF64 ? 8 : 4;
  if (!mul_ok(n, esize)) return BRNG_ERR_SIZE;
  DeviceGuard dg(h);
  int st = dg.status();
  if (st) return st;
  const uint64_t per = (uint64_t)brng::samples_per_block(dist, dtype);
  uint64_t base;
  if ((st = reserve(h, n, per, 1, &base))) return st;
  std::vector<Arr> arrs = {{out, esize, true}};
  const Ctx ctx = make_ctx(h);
  const double sc[2] = {p0, p1};
  st = run(h, arrs, n, per, [&](uint64_t u0, uint64_t nu, const std::vector<void*>& d, bool) {
    return brng::launch_fill(dist, dtype, nullptr, nullptr, d[0], nu, base + u0 / per, ctx, sc);
  });
  if (st) return st;
  commit(h, n, per, 1);
  return BRNG_OK;
}

int gamma_common(brng_t h, int dtype, const void* alpha, const void* beta, void* out,
                 uint64_t n, uint8_t* trials, size_t esize) {
  if (!h || !alpha || !beta || !out) return BRNG_ERR_NULL;
  if (n == 0) return BRNG_OK;
  if (!mul_ok(n, esize)) return BRNG_ERR_SIZE;
  DeviceGuard dg(h);
  int st = dg.status();
  if (st) return st;
  uint64_t base;
  if ((st = reserve(h, n, 1, BRNG_GAMMA_STRIDE, &base))) return st;
  std::vector<Arr> arrs = {{alpha, esize, false}, {beta, esize, false}, {out, esize, true},
                           {trials, 1, true}};
  const Ctx ctx = make_ctx(h);
  st = run(h, arrs, n, 1, [&](uint64_t u0, uint64_t nu, const std::vector<void*>& d, bool) {
    return brng::launch_gamma(dtype, d[0], d[1], d[2], static_cast<uint8_t*>(d[3]), nu,
                              base + (uint64_t)BRNG_GAMMA_STRIDE * u0, ctx);
  });
  if (st) return st;
  commit(h, n, 1, BRNG_GAMMA_STRIDE);
  return BRNG_OK;
}

int dirichlet_common(brng_t h, int dtype, const void* alpha, uint64_t n_rows, uint64_t k,
                     void* out, uint8_t* trials, size_t esize) {
  if (!h || !alpha || !out) return BRNG_ERR_NULL;
  if (k == 0 || k >= (1ull << 24)) return BRNG_ERR_SIZE;   // the kernels' 24-bit row offsets
  if (n_rows == 0) return BRNG_OK;
  if (!mul_ok(n_rows, k)) return BRNG_ERR_SIZE;
  const uint64_t n = n_rows * k;
  if (!mul_ok(n, esize)) return BRNG_ERR_SIZE;
  DeviceGuard dg(h);
  int st = dg.status();
  if (st) return st;
  uint64_t base;
  if ((st = reserve(h, n, 1, BRNG_GAMMA_STRIDE, &base))) return st;
  std::vector<Arr> arrs = {{alpha, esize * k, false}, {out, esize * k, true}, {trials, k, true}};
  Ctx ctx = make_ctx(h);
  // binary32 rows too long for shared memory park their Gammas in a
  // handle-owned scratch (one row per resident warp) instead of recomputing
  // them; above 2 GB of scratch the kernel recomputes
  const size_t scr = brng::dirichlet_scratch_len(dtype, k, ctx);
  // (no growth inside a stream capture: the rows are recomputed instead)
  if (scr && scr <= (size_t(1) << 28)) {
    if (scr > h->dir_scratch_cap && !capturing(h))
      grow_scratch(h, reinterpret_cast<void**>(&h->d_dir_scratch), &h->dir_scratch_cap, scr,
                   sizeof(double));                 // failure: recompute the rows
    if (scr <= h->dir_scratch_cap) ctx.dir_scratch = h->d_dir_scratch;
  }
  st = run(h, arrs, n_rows, 1, [&](uint64_t r0, uint64_t nr, const std::vector<void*>& d, bool) {
    return brng::launch_dirichlet(dtype, d[0], nr, k, d[1], static_cast<uint8_t*>(d[2]),
                                  base + (uint64_t)BRNG_GAMMA_STRIDE * r0 * k, ctx);
  });
  if (st) return st;
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
  h->d_partials = nullptr; h->partials_cap = 0; h->d_totals = nullptr;
  h->d_dir_scratch = nullptr; h->dir_scratch_cap = 0;
  h->pipe_ready = false; h->stage_cap = 0; h->stage_n = 0;
  h->lda_ready = false; h->lda_buf = nullptr; h->lda_cap = 0;
  if (cudaMalloc(&h->d_err, 2 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemset(h->d_err, 0, 2 * sizeof(unsigned long long)) != cudaSuccess) {
    delete h;
    return BRNG_ERR_CUDA;
  }
  if (cudaEventCreateWithFlags(&h->ev_switch, cudaEventDisableTiming) != cudaSuccess) {
    cudaFree(h->d_err);
    delete h;
    return BRNG_ERR_CUDA;
  }
  *out = h;
  return BRNG_OK;
}

int brng_destroy(brng_t h) {
  if (!h) return BRNG_ERR_NULL;
  DeviceGuard dg(h);
  cudaStreamSynchronize(h->stream);
  cudaFree(h->d_err);
  cudaEventDestroy(h->ev_switch);
  if (h->d_partials) cudaFree(h->d_partials);
  if (h->d_totals) cudaFree(h->d_totals);
  if (h->d_dir_scratch) cudaFree(h->d_dir_scratch);
  for (void* p : h->retired) cudaFree(p);
  if (h->lda_buf) cudaFree(h->lda_buf);
  if (h->lda_ready) {
    cudaStreamSynchronize(h->s_prod);
    for (int b = 0; b < 2; ++b) {
      cudaEventDestroy(h->ev_prod[b]);
      cudaEventDestroy(h->ev_cons[b]);
    }
    cudaEventDestroy(h->ev_lda);
    cudaStreamDestroy(h->s_prod);
  }
  if (h->pipe_ready) {
    cudaStreamSynchronize(h->s_in);
    cudaStreamSynchronize(h->s_out);
    for (int b = 0; b < kSlots; ++b) {
      if (h->stage[b]) cudaFree(h->stage[b]);
      cudaEventDestroy(h->ev_in[b]);
      cudaEventDestroy(h->ev_k[b]);
      cudaEventDestroy(h->ev_out[b]);
    }
    cudaStreamDestroy(h->s_in);
    cudaStreamDestroy(h->s_out);
  }
  delete h;
  return BRNG_OK;
}

int brng_set_cuda_stream(brng_t h, void* s) {
  if (!h) return BRNG_ERR_NULL;
  cudaStream_t ns = static_cast<cudaStream_t>(s);
  if (ns != h->stream) {
    // The handle's device scratch (work counter, Gibbs partials) is reused by
    // every call: work already enqueued on the old stream must finish before
    // the new stream's calls touch it.
    DeviceGuard dg(h);
    if (dg.status()) return dg.status();
    cudaError_t e = cudaEventRecord(h->ev_switch, h->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ns, h->ev_switch, 0);
    if (e != cudaSuccess) return BRNG_ERR_CUDA;
    h->stream = ns;
  }
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
  *seed = h->seed;
  *stream_id = h->stream_id;
  return BRNG_OK;
}
int brng_synchronize(brng_t h) {
  if (!h) return BRNG_ERR_NULL;
  DeviceGuard dg(h);
  if (dg.status()) return dg.status();
  return cuda_status(cudaStreamSynchronize(h->stream));
}
int brng_device_errors(brng_t h, uint64_t* n) {
  if (!h || !n) return BRNG_ERR_NULL;
  DeviceGuard dg(h);
  if (dg.status()) return dg.status();
  unsigned long long v = 0;
  cudaError_t e = cudaMemcpyAsync(&v, h->d_err, sizeof(v), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  *n = v;
  return cuda_status(e);
}
int brng_reset_device_errors(brng_t h) {
  if (!h) return BRNG_ERR_NULL;
  DeviceGuard dg(h);
  if (dg.status()) return dg.status();
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

int brng_batch_fill(brng_t h, int dist, int dtype, double p0, double p1, void* out,
                    uint64_t n) {
  return batch_common(h, dist, dtype, p0, p1, out, n);
}

int brng_log_uniform_f32(brng_t h, float* out, uint64_t n) {
  return fill_common(h, brng::kLogUniform, brng::kF32, nullptr, nullptr, out, n, 4);
}
int brng_log_uniform_f64(brng_t h, double* out, uint64_t n) {
  return fill_common(h, brng::kLogUniform, brng::kF64, nullptr, nullptr, out, n, 8);
}
int brng_laplace_f32(brng_t h, const float* mu, const float* beta, float* out, uint64_t n) {
  return fill_common(h, brng::kLaplace, brng::kF32, mu, beta, out, n, 4);
}
int brng_laplace_f64(brng_t h, const double* mu, const double* beta, double* out, uint64_t n) {
  return fill_common(h, brng::kLaplace, brng::kF64, mu, beta, out, n, 8);
}
int brng_weibull_f32(brng_t h, const float* alpha, const float* beta, float* out, uint64_t n) {
  return fill_common(h, brng::kWeibull, brng::kF32, alpha, beta, out, n, 4);
}
int brng_weibull_f64(brng_t h, const double* alpha, const double* beta, double* out,
                     uint64_t n) {
  return fill_common(h, brng::kWeibull, brng::kF64, alpha, beta, out, n, 8);
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
  // u32 shared-memory histogram: a CTA round holds at most 768 chains, so
  // < 768 * 2^22 < 2^32 counts per bin by construction
  if (n_sweeps >= (1ull << 22)) return BRNG_ERR_SIZE;
  if (n_chains == 0) return BRNG_OK;
  if (!mul_ok(n_chains, n_sweeps) || !mul_ok(n_chains * n_sweeps, 8) || !mul_ok(n_chains, 40))
    return BRNG_ERR_SIZE;
  if (n_chains > std::numeric_limits<uint64_t>::max() - h->stream_id) return BRNG_ERR_OVERFLOW;
  DeviceGuard dg(h);
  int st = dg.status();
  if (st) return st;
  uint64_t base;
  if ((st = reserve(h, n_sweeps, 1, 1, &base))) return st;
  const Ctx ctx = make_ctx(h);
  const size_t need = brng::gibbs_partials_len(n_chains, ctx);
  if (need > h->partials_cap) {
    // a capture cannot allocate: make one eager call of this size first
    if (capturing(h)) return BRNG_ERR_STATE;
    if (!grow_scratch(h, reinterpret_cast<void**>(&h->d_partials), &h->partials_cap, need,
                      sizeof(double)))
      return BRNG_ERR_CUDA;
  }
  // totals belongs to the call, not to a chain: a host totals pointer gets a
  // device scratch that every chunk accumulates into
  double* dtot = totals;
  const bool host_tot = totals != nullptr && !is_device_ptr(totals);
  // (a handle-owned buffer, allocated once: a per-call cudaMallocAsync /
  // cudaFreeAsync pair was measured to stall some calls by 0.3-0.6 s)
  if (host_tot && h->d_totals == nullptr && capturing(h)) return BRNG_ERR_STATE;
  if (host_tot && h->d_totals == nullptr &&
      cudaMalloc(reinterpret_cast<void**>(&h->d_totals), BRNG_TOTALS_LEN * 8) != cudaSuccess)
    return BRNG_ERR_CUDA;
  if (host_tot) dtot = h->d_totals;
  std::vector<Arr> arrs = {{x0, 8, false},
                           {y0, 8, false},
                           {out_x, 8, true, (size_t)n_sweeps},
                           {out_y, 8, true, (size_t)n_sweeps},
                           {chain_stats, 8, true, 5},
                           {final_xy, 8, true, 2}};
  // Gibbs chunks: whole resident waves (no partly filled last round), two
  // per chunk, so a chunk is a few ms of kernel: kernels of other streams
  // (e.g. a concurrent host-staged fill) find a launch boundary that often
  // instead of waiting behind one long-lived wave of persistent CTAs.
#ifndef BRNG_GIBBS_CHUNK_WAVES
#define BRNG_GIBBS_CHUNK_WAVES 2
#endif
  const uint64_t wave = brng::gibbs_wave_chains(ctx);
  const uint64_t align = (BRNG_GIBBS_CHUNK_WAVES && n_chains >= wave) ? wave : 1;
  st = run(h, arrs, n_chains, align,
           [&](uint64_t c0, uint64_t nc, const std::vector<void*>& d, bool first) {
             Ctx cc = ctx;
             cc.stream_id = ctx.stream_id + c0;
             return brng::launch_gibbs(nc, n_sweeps, static_cast<const double*>(d[0]),
                                       static_cast<const double*>(d[1]), burn_in,
                                       static_cast<double*>(d[2]), static_cast<double*>(d[3]),
                                       static_cast<double*>(d[4]), static_cast<double*>(d[5]),
                                       dtot, h->d_partials, base, cc, !first);
           },
           BRNG_GIBBS_CHUNK_WAVES * wave, /*soft_align=*/true);
  if (host_tot) {
    cudaError_t e = cudaMemcpyAsync(totals, dtot, BRNG_TOTALS_LEN * 8, cudaMemcpyDeviceToHost,
                                    h->stream);
    cudaError_t e2 = cudaStreamSynchronize(h->stream);
    if (!st && (e != cudaSuccess || e2 != cudaSuccess)) st = BRNG_ERR_CUDA;
  }
  if (st) return st;
  commit(h, n_sweeps, 1, 1);
  return BRNG_OK;
}

// ---- NEXT row N4: LDA fold-in Gibbs consumer (R-33) --------
int brng_lda_gibbs(brng_t h, uint64_t n_docs, uint32_t k, uint32_t v, uint64_t n_tokens,
                   const uint64_t* doc_off, const uint32_t* words, const double* phi,
                   const double* alpha, uint16_t* z, double* theta, uint32_t n_iter, int mode) {
  if (!h || !doc_off || !words || !phi || !alpha || !z) return BRNG_ERR_NULL;
  if (k == 0 || k > BRNG_LDA_MAX_K || v == 0) return BRNG_ERR_SIZE;
  if (mode < BRNG_LDA_INLINE || mode > BRNG_LDA_BULK) return BRNG_ERR_PARAM;
  if (n_docs == 0 || n_iter == 0) return BRNG_OK;
  for (const void* p : {(const void*)doc_off, (const void*)words, (const void*)phi,
                        (const void*)alpha, (const void*)z, (const void*)theta})
    if (p && !is_device_ptr(p)) return BRNG_ERR_PARAM;          // device pointers only
  if (!mul_ok(n_docs, k) || !mul_ok(n_docs * k, BRNG_GAMMA_STRIDE) || !mul_ok(n_tokens, 16))
    return BRNG_ERR_SIZE;
  const uint64_t dk = n_docs * k;
  const uint64_t gspan = dk * BRNG_GAMMA_STRIDE;
  const uint64_t uspan = n_tokens / 2 + (n_tokens % 2);
  if (gspan > std::numeric_limits<uint64_t>::max() - uspan) return BRNG_ERR_OVERFLOW;
  const uint64_t span = gspan + uspan;
  DeviceGuard dg(h);
  int st = dg.status();
  if (st) return st;
  uint64_t base;
  if ((st = reserve(h, n_iter, 1, span, &base))) return st;
  Ctx ctx = make_ctx(h);
  brng::LdaArgs a{};
  a.n_docs = n_docs; a.n_tokens = n_tokens; a.k = k; a.v = v;
  a.k0 = ctx.k0; a.k1 = ctx.k1; a.stream = ctx.stream_id;
  a.doc_off = doc_off; a.words = words; a.phi = phi; a.alpha = alpha; a.z = z;
  a.work = ctx.work; a.err = ctx.err;
  // scratch: RING two slots of {z f64, w3 u32, ln(1-u) f64}[dk] + u f64[T];
  // BULK {alpha + n rows f64, theta f64}[dk] + u f64[T]
  auto al256 = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t slot = al256(dk * 8) + al256(dk * 4) + al256(dk * 8) + al256(n_tokens * 8);
  const size_t need = mode == BRNG_LDA_RING ? 2 * slot
                    : mode == BRNG_LDA_BULK ? al256(dk * 8) * 2 + al256(n_tokens * 8) : 0;
  if (need > h->lda_cap) {
    if (capturing(h)) return BRNG_ERR_STATE;
    if (!grow_scratch(h, &h->lda_buf, &h->lda_cap, need, 1)) return BRNG_ERR_CUDA;
  }
  char* buf = static_cast<char*>(h->lda_buf);
  cudaError_t e = cudaSuccess;
  if (mode == BRNG_LDA_INLINE) {
    for (uint32_t t = 0; t < n_iter && e == cudaSuccess; ++t) {
      a.base = base + (uint64_t)t * span;
      a.theta_out = t + 1 == n_iter ? theta : nullptr;
      e = brng::launch_lda_consumer(0, a, ctx);
    }
  } else if (mode == BRNG_LDA_BULK) {
    double* rows = reinterpret_cast<double*>(buf);
    double* th = reinterpret_cast<double*>(buf + al256(dk * 8));
    double* ub = reinterpret_cast<double*>(buf + 2 * al256(dk * 8));
    a.theta_in = th; a.ubuf = ub;
    for (uint32_t t = 0; t < n_iter && e == cudaSuccess; ++t) {
      a.base = base + (uint64_t)t * span;
      a.theta_out = t + 1 == n_iter ? theta : nullptr;
      e = brng::launch_lda_rows(a, rows, ctx);
      if (e == cudaSuccess) e = brng::launch_dirichlet(brng::kF64, rows, n_docs, k, th, nullptr,
                                                       a.base, ctx);
      if (e == cudaSuccess) e = brng::launch_fill(brng::kStdUniform, brng::kF64, nullptr,
                                                  nullptr, ub, n_tokens, a.base + gspan, ctx);
      if (e == cudaSuccess) e = brng::launch_lda_consumer(2, a, ctx);
    }
  } else {
    if (!h->lda_ready) {
      // all-or-nothing: a partial failure releases what was created
      cudaStream_t sp = nullptr;
      cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
      bool ok = cudaStreamCreateWithFlags(&sp, cudaStreamNonBlocking) == cudaSuccess;
      for (int b = 0; b < 5 && ok; ++b)
        ok = cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming) == cudaSuccess;
      if (!ok) {
        for (cudaEvent_t x : ev)
          if (x) cudaEventDestroy(x);
        if (sp) cudaStreamDestroy(sp);
        return BRNG_ERR_CUDA;
      }
      h->s_prod = sp;
      h->ev_prod[0] = ev[0]; h->ev_prod[1] = ev[1];
      h->ev_cons[0] = ev[2]; h->ev_cons[1] = ev[3];
      h->ev_lda = ev[4];
      h->lda_ready = true;
    }
    struct Slot { double* zb; uint32_t* w3; double* lb; double* ub; } sl[2];
    for (int b = 0; b < 2; ++b) {
      char* p = buf + b * slot;
      sl[b].zb = reinterpret_cast<double*>(p);
      sl[b].w3 = reinterpret_cast<uint32_t*>(p + al256(dk * 8));
      sl[b].lb = reinterpret_cast<double*>(p + al256(dk * 8) + al256(dk * 4));
      sl[b].ub = reinterpret_cast<double*>(p + al256(dk * 8) + al256(dk * 4) + al256(dk * 8));
    }
    // the producer of iteration t + 1 runs on the side stream while the
    // consumer of iteration t runs on the handle's stream; slot t % 2
    e = cudaEventRecord(h->ev_lda, h->stream);                     // earlier work first
    if (e == cudaSuccess) e = cudaStreamWaitEvent(h->s_prod, h->ev_lda, 0);
    auto produce = [&](uint32_t t) {
      brng::LdaArgs pa = a;
      pa.base = base + (uint64_t)t * span;
      const Slot& q = sl[t % 2];
      cudaError_t e2 = cudaSuccess;
      if (t >= 2) e2 = cudaStreamWaitEvent(h->s_prod, h->ev_cons[t % 2], 0);   // slot free
      if (e2 == cudaSuccess) e2 = brng::launch_lda_producer(pa, q.zb, q.w3, q.lb, q.ub, ctx,
                                                            h->s_prod);
      if (e2 == cudaSuccess) e2 = cudaEventRecord(h->ev_prod[t % 2], h->s_prod);
      return e2;
    };
    if (e == cudaSuccess) e = produce(0);
    for (uint32_t t = 0; t < n_iter && e == cudaSuccess; ++t) {
      if (t + 1 < n_iter) e = produce(t + 1);
      const Slot& q = sl[t % 2];
      a.base = base + (uint64_t)t * span;
      a.theta_out = t + 1 == n_iter ? theta : nullptr;
      a.zbuf = q.zb; a.w3buf = q.w3; a.lbuf = q.lb; a.ubuf = q.ub;
      if (e == cudaSuccess) e = cudaStreamWaitEvent(h->stream, h->ev_prod[t % 2], 0);
      if (e == cudaSuccess) e = brng::launch_lda_consumer(1, a, ctx);
      if (e == cudaSuccess) e = cudaEventRecord(h->ev_cons[t % 2], h->stream);
    }
  }
  if (e != cudaSuccess) return BRNG_ERR_CUDA;
  commit(h, n_iter, 1, span);
  return BRNG_OK;
}

}  // extern "C"
