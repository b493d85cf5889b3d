// driver.cpp -- TEST INFRASTRUCTURE ONLY: exercises the host logic of the C
// ABI (paper_1412_4825_b200/csrc/brng.cpp) under ASan + UBSan with the fake
// runtime (fake_cuda.cpp) and fake launches (fake_kernels.cpp): error paths,
// cursor reservation and overflow, device-pointer calls, and multi-chunk
// host-staged calls of every entry-point family, checking that every output
// element came from the right chunk launch with the right input slice, and
// that destroy releases every allocation.  Prints "host_asan ok" on success.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/brng.h"

size_t fake_cuda_live_allocs();
size_t fake_cuda_peak_bytes(bool reset);
namespace brng { double fake_fill_value(uint64_t g, double p0, double p1); }

static int g_fail = 0;
#define CHECK(c)                                                         \
  do {                                                                   \
    if (!(c)) {                                                          \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++g_fail;                                                          \
    }                                                                    \
  } while (0)

static void errors() {
  brng_t h = nullptr;
  CHECK(brng_create(1, 0, nullptr) == BRNG_ERR_NULL);
  CHECK(brng_create(1, 0, &h) == BRNG_OK && h);
  float f[8] = {0};
  double d[8] = {0};
  uint64_t c = 0;
  CHECK(brng_uniform_f32(nullptr, f, f, f, 8) == BRNG_ERR_NULL);
  CHECK(brng_uniform_f32(h, nullptr, f, f, 8) == BRNG_ERR_NULL);
  CHECK(brng_gamma_f64(h, d, nullptr, d, 8, nullptr) == BRNG_ERR_NULL);
  CHECK(brng_dirichlet_f64(h, d, 2, 0, d, nullptr) == BRNG_ERR_SIZE);
  CHECK(brng_gibbs_triangle(h, 4, 3, nullptr, nullptr, 4, nullptr, nullptr, nullptr, nullptr,
                            nullptr) == BRNG_ERR_SIZE);
  CHECK(brng_gibbs_triangle(h, 4, 1ull << 22, nullptr, nullptr, 0, nullptr, nullptr, nullptr,
                            nullptr, nullptr) == BRNG_ERR_SIZE);
  CHECK(brng_batch_fill(h, 99, 0, 0.0, 1.0, f, 4) == BRNG_ERR_PARAM);
  CHECK(brng_batch_fill(h, BRNG_DIST_UNIFORM, 7, 0.0, 1.0, f, 4) == BRNG_ERR_PARAM);
  CHECK(brng_get_offset(h, &c) == BRNG_OK && c == 0);
  // size overflow: n * element size past 2^64
  CHECK(brng_uniform_f64(h, d, d, d, (uint64_t)1 << 62) == BRNG_ERR_SIZE);
  CHECK(brng_dirichlet_f32(h, f, (uint64_t)1 << 40, (uint64_t)1 << 30, f, nullptr) ==
        BRNG_ERR_SIZE);
  // cursor overflow past 2^64: no launch, cursor unchanged
  CHECK(brng_set_offset(h, ~0ull - 1000) == BRNG_OK);
  CHECK(brng_gamma_f64(h, d, d, d, 8, nullptr) == BRNG_ERR_OVERFLOW);
  CHECK(brng_get_offset(h, &c) == BRNG_OK && c == ~0ull - 1000);
  CHECK(brng_gibbs_triangle(h, 4, 2000, nullptr, nullptr, 0, nullptr, nullptr, nullptr, nullptr,
                            nullptr) == BRNG_ERR_OVERFLOW);
  // stream overflow of a Gibbs call
  brng_t h2 = nullptr;
  CHECK(brng_create(1, ~0ull - 2, &h2) == BRNG_OK);
  CHECK(brng_gibbs_triangle(h2, 8, 4, nullptr, nullptr, 0, nullptr, nullptr, nullptr, nullptr,
                            nullptr) == BRNG_ERR_OVERFLOW);
  CHECK(brng_destroy(h2) == BRNG_OK);
  // n == 0: no-op
  CHECK(brng_set_offset(h, 5) == BRNG_OK);
  CHECK(brng_uniform_f32(h, f, f, f, 0) == BRNG_OK);
  CHECK(brng_get_offset(h, &c) == BRNG_OK && c == 5);
  for (int s = 0; s >= -7; --s) CHECK(brng_status_string(s) != nullptr);
  CHECK(brng_version() == BRNG_VERSION);
  CHECK(brng_destroy(h) == BRNG_OK);
  CHECK(brng_destroy(nullptr) == BRNG_ERR_NULL);
}

// host-staged f32 uniform fill over several 64 MB chunks + a ragged tail
static void fills_host() {
  const uint64_t n = (uint64_t)20 * 1000 * 1000 + 3;       // 80 MB per array -> 2 chunks
  std::vector<float> a(n), b(n), o(n, -1.0f);
  for (uint64_t i = 0; i < n; ++i) { a[i] = (float)(i % 7); b[i] = (float)(i % 5) + 8.0f; }
  brng_t h;
  CHECK(brng_create(3, 0, &h) == BRNG_OK);
  CHECK(brng_uniform_f32(h, a.data(), b.data(), o.data(), n) == BRNG_OK);
  uint64_t c;
  CHECK(brng_get_offset(h, &c) == BRNG_OK && c == (n + 3) / 4);
  uint64_t bad = 0;
  for (uint64_t i = 0; i < n; ++i)
    bad += o[i] != (float)brng::fake_fill_value(i, a[i], b[i]);
  CHECK(bad == 0);
  // f64 host fill starting at a nonzero cursor, and a batch fill
  const uint64_t m = (uint64_t)9 * 1000 * 1000 + 1;        // 72 MB per array
  std::vector<double> mu(m, 1.0), sg(m, 0.5), od(m);
  CHECK(brng_set_offset(h, 10) == BRNG_OK);
  CHECK(brng_gaussian_f64(h, mu.data(), sg.data(), od.data(), m) == BRNG_OK);
  bad = 0;
  for (uint64_t i = 0; i < m; ++i) bad += od[i] != brng::fake_fill_value(20 + i, 1.0, 0.5);
  CHECK(bad == 0);
  CHECK(brng_batch_fill(h, BRNG_DIST_GAUSSIAN, BRNG_DTYPE_F64, 2.0, 3.0, od.data(), m) == BRNG_OK);
  CHECK(brng_get_offset(h, &c) == BRNG_OK && c == 10 + 2 * ((m + 1) / 2));
  std::vector<uint32_t> w(1001);
  CHECK(brng_raw_u32(h, w.data(), w.size()) == BRNG_OK);
  CHECK(brng_destroy(h) == BRNG_OK);
}

static void gamma_dirichlet_host() {
  brng_t h;
  CHECK(brng_create(4, 0, &h) == BRNG_OK);
  const uint64_t n = (uint64_t)9 * 1000 * 1000 + 17;       // 72 MB of f64 -> 2 chunks
  std::vector<double> al(n), be(n), o(n);
  std::vector<uint8_t> tr(n);
  for (uint64_t i = 0; i < n; ++i) { al[i] = (double)(i % 11); be[i] = 0.25; }
  CHECK(brng_set_offset(h, 256 * 3) == BRNG_OK);
  CHECK(brng_gamma_f64(h, al.data(), be.data(), o.data(), n, tr.data()) == BRNG_OK);
  uint64_t bad = 0;
  for (uint64_t i = 0; i < n; ++i)
    bad += o[i] != brng::fake_fill_value(3 + i, al[i], 0.25) || tr[i] != (uint8_t)((3 + i) & 0xff);
  CHECK(bad == 0);
  // Dirichlet f32 rows over several chunks (k = 300), then a scratch-path k
  const uint64_t k = 300, rows = 120001;                   // 144 MB -> 3 chunks
  std::vector<float> a(rows * k), x(rows * k);
  for (uint64_t i = 0; i < rows * k; ++i) a[i] = (float)(i % 3);
  CHECK(brng_set_offset(h, 0) == BRNG_OK);
  CHECK(brng_dirichlet_f32(h, a.data(), rows, k, x.data(), nullptr) == BRNG_OK);
  bad = 0;
  for (uint64_t i = 0; i < rows * k; ++i) bad += x[i] != (float)brng::fake_fill_value(i, a[i], 0);
  CHECK(bad == 0);
  for (uint64_t kk : {2048ull, 4096ull, 2048ull}) {          // scratch grows, then is reused
    std::vector<float> a2(9 * kk, 1.0f), x2(9 * kk);
    CHECK(brng_dirichlet_f32(h, a2.data(), 9, kk, x2.data(), nullptr) == BRNG_OK);
  }
  CHECK(brng_destroy(h) == BRNG_OK);
}

static void gibbs_host() {
  brng_t h;
  CHECK(brng_create(42, 100, &h) == BRNG_OK);
  const uint64_t wave = 148ull * 2 * 256 * 3;
  const uint64_t nc = wave + 1017, ns = 64;               // host samples: chunk capped by bytes
  std::vector<double> ox(ns * nc), oy(ns * nc), st(5 * nc), fx(2 * nc), tot(BRNG_TOTALS_LEN);
  CHECK(brng_set_offset(h, 7) == BRNG_OK);
  fake_cuda_peak_bytes(true);
  CHECK(brng_gibbs_triangle(h, nc, ns, nullptr, nullptr, 0, ox.data(), oy.data(), st.data(),
                            fx.data(), tot.data()) == BRNG_OK);
  uint64_t bad = 0;
  for (uint64_t s = 0; s < ns; ++s)
    for (uint64_t c = 0; c < nc; ++c) {
      const double id = (double)(100 + c), v = id + 1e-3 * (double)(7 + s) + 0.5;
      bad += ox[s * nc + c] != v || oy[s * nc + c] != v;
    }
  for (uint64_t c = 0; c < nc; ++c) {
    for (int q = 0; q < 5; ++q) bad += st[q * nc + c] != 10.0 * (double)(100 + c) + q;
    bad += fx[c] != (double)(100 + c) || fx[nc + c] != -(double)(100 + c);
  }
  CHECK(bad == 0);
  CHECK(tot[8] == (double)nc && tot[9] == (double)(nc * ns));
  // staging stays near the 64 MB-per-array chunk target (a
  // wave-aligned chunk of host samples needed ~22 GB at 1000 sweeps)
  const size_t peak = fake_cuda_peak_bytes(false);
  std::printf("gibbs host-samples staging peak: %.1f MB\n", peak / 1048576.0);
  CHECK(peak < (size_t)512 << 20);
  uint64_t c;
  CHECK(brng_get_offset(h, &c) == BRNG_OK && c == 7 + ns);
  // host start states + host chain stats only, many chunks
  const uint64_t nc2 = 3 * wave + 5;
  std::vector<double> x0(nc2, 0.25), y0(nc2, 0.125), st2(5 * nc2);
  CHECK(brng_gibbs_triangle(h, nc2, 16, x0.data(), y0.data(), 0, nullptr, nullptr, st2.data(),
                            nullptr, tot.data()) == BRNG_OK);
  bad = 0;
  for (uint64_t c2 = 0; c2 < nc2; ++c2) bad += st2[c2] != 10.0 * (double)(100 + c2);
  CHECK(bad == 0 && tot[8] == (double)nc2);
  CHECK(brng_destroy(h) == BRNG_OK);
}

// LDA consumer entry point (N4): argument checks, device-pointer rule,
// cursor span, RING / BULK scratch growth and release
static void lda() {
  brng_t h;
  CHECK(brng_create(5, 0, &h) == BRNG_OK);
  const uint64_t D = 50, T = 777;
  const uint32_t K = 16, V = 30;
  void *off, *w, *phi, *al, *z, *th;
  CHECK(cudaMalloc(&off, (D + 1) * 8) == cudaSuccess && cudaMalloc(&w, T * 4) == cudaSuccess);
  CHECK(cudaMalloc(&phi, V * K * 8) == cudaSuccess && cudaMalloc(&al, K * 8) == cudaSuccess);
  CHECK(cudaMalloc(&z, T * 2) == cudaSuccess && cudaMalloc(&th, D * K * 8) == cudaSuccess);
  auto off_p = static_cast<const uint64_t*>(off);
  auto w_p = static_cast<const uint32_t*>(w);
  auto phi_p = static_cast<const double*>(phi);
  auto al_p = static_cast<const double*>(al);
  auto z_p = static_cast<uint16_t*>(z);
  auto th_p = static_cast<double*>(th);
  std::vector<uint16_t> host_z(T);
  CHECK(brng_lda_gibbs(h, D, 0, V, T, off_p, w_p, phi_p, al_p, z_p, th_p, 1, 0) == BRNG_ERR_SIZE);
  CHECK(brng_lda_gibbs(h, D, BRNG_LDA_MAX_K + 1, V, T, off_p, w_p, phi_p, al_p, z_p, th_p, 1, 0) ==
        BRNG_ERR_SIZE);
  CHECK(brng_lda_gibbs(h, D, K, V, T, off_p, w_p, phi_p, al_p, z_p, th_p, 1, 9) == BRNG_ERR_PARAM);
  CHECK(brng_lda_gibbs(h, D, K, V, T, off_p, w_p, phi_p, al_p, host_z.data(), th_p, 1, 0) ==
        BRNG_ERR_PARAM);
  CHECK(brng_lda_gibbs(h, D, K, V, T, nullptr, w_p, phi_p, al_p, z_p, th_p, 1, 0) == BRNG_ERR_NULL);
  uint64_t c = 0;
  CHECK(brng_get_offset(h, &c) == BRNG_OK && c == 0);
  const uint64_t span = 256ull * D * K + (T + 1) / 2;
  for (int mode : {BRNG_LDA_INLINE, BRNG_LDA_RING, BRNG_LDA_BULK, BRNG_LDA_RING})
    CHECK(brng_lda_gibbs(h, D, K, V, T, off_p, w_p, phi_p, al_p, z_p, th_p, 3, mode) == BRNG_OK);
  CHECK(brng_get_offset(h, &c) == BRNG_OK && c == 4 * 3 * span);
  CHECK(brng_lda_gibbs(h, D, K, V, T, off_p, w_p, phi_p, al_p, z_p, nullptr, 0, 0) == BRNG_OK);
  CHECK(brng_destroy(h) == BRNG_OK);
  for (void* p : {off, w, phi, al, z, th}) cudaFree(p);
}

int main() {
  errors();
  lda();
  fills_host();
  gamma_dirichlet_host();
  gibbs_host();
  CHECK(fake_cuda_live_allocs() == 0);
  if (g_fail) {
    std::fprintf(stderr, "host_asan: %d failures\n", g_fail);
    return 1;
  }
  std::printf("host_asan ok\n");
  return 0;
}
