/* oracle_driver.c -- TEST INFRASTRUCTURE ONLY: runs every entry point of the
 * CPU oracle (oracle/oracle.c) at small sizes, with edge and invalid
 * parameters, each output in its own exactly-sized heap block, under
 * AddressSanitizer + UndefinedBehaviorSanitizer.  Results are
 * checked only for basic sanity here (the pins live in tests/test_oracle_*.py);
 * the point is that no call reads or writes outside its arrays or hits
 * undefined behaviour.  Prints "oracle_asan ok". */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]);
void orc_block(uint64_t seed, uint64_t stream, uint64_t pos, uint32_t out[4]);
double orc_u24(uint32_t w);
double orc_u53(uint32_t lo, uint32_t hi);
double orc_u32d(uint32_t w);
double orc_cos2pi(double u);
double orc_sin2pi(double u);
double orc_box_muller(double u_r, double u_theta, int use_sin);
void orc_raw_u32(uint64_t, uint64_t, uint64_t, uint32_t*, uint64_t);
void orc_std_uniform_f32(uint64_t, uint64_t, uint64_t, float*, uint64_t);
void orc_std_uniform_f64(uint64_t, uint64_t, uint64_t, double*, uint64_t);
#define FILLS(T, S)                                                                         \
  uint64_t orc_uniform_##S(uint64_t, uint64_t, uint64_t, const T*, const T*, T*, uint64_t,  \
                           uint64_t);                                                       \
  uint64_t orc_gaussian_##S(uint64_t, uint64_t, uint64_t, const T*, const T*, T*, uint64_t, \
                            uint64_t);                                                      \
  uint64_t orc_exponential_##S(uint64_t, uint64_t, uint64_t, const T*, T*, uint64_t,         \
                               uint64_t);                                                   \
  void orc_log_uniform_##S(uint64_t, uint64_t, uint64_t, T*, uint64_t, uint64_t);           \
  uint64_t orc_laplace_##S(uint64_t, uint64_t, uint64_t, const T*, const T*, T*, uint64_t,  \
                           uint64_t);                                                       \
  uint64_t orc_weibull_##S(uint64_t, uint64_t, uint64_t, const T*, const T*, T*, uint64_t,  \
                           uint64_t);                                                       \
  uint64_t orc_gamma_##S(uint64_t, uint64_t, uint64_t, const T*, const T*, T*, uint8_t*,    \
                         uint64_t, uint64_t);                                               \
  uint64_t orc_dirichlet_##S(uint64_t, uint64_t, uint64_t, const T*, uint64_t, T*, uint8_t*, \
                             uint64_t, uint64_t, double*);
FILLS(float, f32)
FILLS(double, f64)
int orc_mt_trial(double d, double c, double u_r, double u_theta, double U, double* g,
                 double* margin, double* onepcz);
void orc_mt_consts(double alpha, double* d, double* c);
void orc_mt_trial_uniforms(uint64_t, uint64_t, uint64_t, uint64_t, uint32_t, double*, double*,
                           double*);
double orc_gamma_one(uint64_t, uint64_t, uint64_t, uint64_t, double, double, uint32_t*, int*);
uint64_t orc_gibbs_triangle(uint64_t seed, uint64_t stream_id, uint64_t base, uint64_t n_chains,
                            uint64_t n_sweeps, const double* x0, const double* y0,
                            uint64_t burn_in, double* out_x, double* out_y, double* chain_stats,
                            double* final_xy, double* totals);

static int fails = 0;
#define CHECK(c)                                                              \
  do {                                                                        \
    if (!(c)) { fprintf(stderr, "CHECK failed line %d: %s\n", __LINE__, #c); ++fails; } \
  } while (0)

static void* xmalloc(size_t n) { void* p = malloc(n ? n : 1); if (!p) abort(); return p; }

/* edge parameters: NaN, +-inf, 0, negative, subnormal, huge, ordinary */
static const double EDGE[] = {NAN, INFINITY, -INFINITY, 0.0, -1.0, 4.9e-324, 1e300, 0.05, 1.0,
                              2.5, 200.0, 1e-3, 7.0};
#define NE (sizeof(EDGE) / sizeof(EDGE[0]))

#define RUN_FILLS(T, S)                                                                      \
  do {                                                                                       \
    const uint64_t n = NE * NE;                                                              \
    T* a = xmalloc(n * sizeof(T)); T* b = xmalloc(n * sizeof(T)); T* o = xmalloc(n * sizeof(T)); \
    for (uint64_t i = 0; i < n; ++i) { a[i] = (T)EDGE[i / NE]; b[i] = (T)EDGE[i % NE]; }     \
    uint64_t bad = orc_uniform_##S(7, 1, (1ull << 32) - 3, a, b, o, 5, n);                   \
    bad += orc_gaussian_##S(7, 1, ~0ull - 100, a, b, o, 3, n);                               \
    bad += orc_exponential_##S(7, 1, 0, a, o, 1, n);                                         \
    orc_log_uniform_##S(7, 1, 0, o, 0, n);                                                   \
    bad += orc_laplace_##S(7, 1, 0, a, b, o, 2, n);                                          \
    bad += orc_weibull_##S(7, 1, 0, a, b, o, 2, n);                                          \
    CHECK(bad > 0);                                                                          \
    uint8_t* tr = xmalloc(n);                                                                \
    bad = orc_gamma_##S(11, 0, 0, a, b, o, tr, 0, n);                                        \
    CHECK(bad > 0);                                                                          \
    for (uint64_t i = 0; i < n; ++i) CHECK((tr[i] == 0) == isnan((double)o[i]));            \
    free(tr);                                                                                \
    /* Dirichlet: K = 1, a K = NE row set, and an LDA-like row */                            \
    double* scr = xmalloc(NE * sizeof(double));                                              \
    uint8_t* t2 = xmalloc(n);                                                                \
    orc_dirichlet_##S(3, 0, 0, a, 1, o, t2, 0, n, scr);                                      \
    orc_dirichlet_##S(3, 0, 0, a, NE, o, t2, 4, NE, scr);                                    \
    orc_dirichlet_##S(3, 0, 0, a, NE, o, NULL, 0, NE, scr);                                  \
    free(scr); free(t2);                                                                     \
    free(a); free(b); free(o);                                                               \
  } while (0)

int main(void) {
  uint32_t w[4], c[4] = {0xffffffffu, 0xffffffffu, 0, 0xffffffffu}, k[2] = {0xffffffffu, 1};
  orc_philox4x32_10(c, k, w);
  orc_block(~0ull, ~0ull, ~0ull, w);
  CHECK(orc_u24(0xffffffffu) < 1.0 && orc_u53(0xffffffffu, 0xffffffffu) < 1.0);
  CHECK(orc_u32d(0) == 0.0);
  for (double u = 0.0; u < 1.0; u += 1.0 / 64) {
    CHECK(fabs(orc_cos2pi(u)) <= 1.0 && fabs(orc_sin2pi(u)) <= 1.0);
    CHECK(isfinite(orc_box_muller(u, u, 0)) && isfinite(orc_box_muller(u, u, 1)));
  }
  uint32_t* r = xmalloc(13 * 4); orc_raw_u32(1, 2, ~0ull - 2, r, 13); free(r);
  float* f = xmalloc(13 * 4); orc_std_uniform_f32(1, 2, 3, f, 13); free(f);
  double* d = xmalloc(13 * 8); orc_std_uniform_f64(1, 2, 3, d, 13); free(d);
  RUN_FILLS(float, f32);
  RUN_FILLS(double, f64);
  double dd, cc, g, m, t, ur, ut, U;
  orc_mt_consts(0.05, &dd, &cc);
  orc_mt_trial_uniforms(1, 0, 0, 5, 255, &ur, &ut, &U);
  (void)orc_mt_trial(dd, cc, ur, ut, U, &g, &m, &t);
  (void)orc_mt_trial(dd, cc, 0.0, 0.5, 1.0, NULL, NULL, NULL);
  uint32_t tri; int bad;
  CHECK(isnan(orc_gamma_one(1, 0, 0, 0, -1.0, 1.0, &tri, &bad)) && bad && tri == 0);
  CHECK(isfinite(orc_gamma_one(1, 0, 0, 0, 1e-300, 1.0, &tri, &bad)));
  /* Gibbs: every optional output, burn-in, per-chain starts incl. invalid */
  const uint64_t nc = 9, ns = 17;
  double* x0 = xmalloc(nc * 8); double* y0 = xmalloc(nc * 8);
  for (uint64_t i = 0; i < nc; ++i) { x0[i] = 0.1 * (double)i; y0[i] = EDGE[i % NE]; }
  double* ox = xmalloc(nc * ns * 8); double* oy = xmalloc(nc * ns * 8);
  double* st = xmalloc(5 * nc * 8); double* fx = xmalloc(2 * nc * 8);
  double* tot = calloc(272, 8);
  uint64_t nbad = orc_gibbs_triangle(42, ~0ull - nc, 3, nc, ns, x0, y0, 4, ox, oy, st, fx, tot);
  CHECK(nbad > 0);
  nbad = orc_gibbs_triangle(42, 0, 0, nc, ns, NULL, NULL, ns - 2, NULL, NULL, NULL, NULL, tot);
  CHECK(nbad == 0);
  (void)orc_gibbs_triangle(42, 0, 0, nc, 1, NULL, NULL, 0, ox, NULL, st, NULL, NULL);
  free(x0); free(y0); free(ox); free(oy); free(st); free(fx); free(tot);
  if (fails) { fprintf(stderr, "oracle_asan: %d failures\n", fails); return 1; }
  printf("oracle_asan ok\n");
  return 0;
}
