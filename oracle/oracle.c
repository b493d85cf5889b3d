/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded, obviously-correct CPU implementation of the
 * varying-parameter random-deviate hot path of arXiv 1412.4825 ("BatchRNG"),
 * written from PAPER.md and the contract readings in DESIGN.md ("Contract").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load this library.  It shares no code, header,
 * table or constant generator with paper_1412_4825_b200/csrc (the CUDA path),
 * and never includes anything from there.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -shared -fPIC
 *        (no FMA contraction: every fma below is an explicit fma() call that
 *        the contract names; every other operation is one IEEE-754 binary64
 *        operation in source order).
 *
 * Citation keys: P:Lnn = /root/reference/PAPER.md line nn (section given);
 * S:Lnn = SPEC.md line nn; R-xx = DESIGN.md reading xx.
 *
 * Parity pins for every function are listed in DESIGN.md "Oracle pins" and
 * implemented in tests/test_oracle_*.py (-m "not gpu").
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------- */
/* 1. Base generator: Philox4x32-10 (R-01).  The paper's "core engine" that    */
/*    produces uniform random integers (§2.1 key concept 1,      */
/*    §2.2 "vectorized RNG for uniform distribution").                         */
/*    Definition (Salmon, Moraes, Dror, Shaw, SC'11): one round maps           */
/*    (c0,c1,c2,c3) -> (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1,           */
/*    lo(M0*c0)); the key is bumped by the Weyl constants between rounds.      */
/* ------------------------------------------------------------------------- */
ORC_API void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                               uint32_t out[4])
{
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += W0; k1 += W1; }
        uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Counter map (R-02): key = (lo32 seed, hi32 seed); counter = (lo32 pos,
 * hi32 pos, lo32 stream, hi32 stream); pos is a 64-bit BLOCK index. */
ORC_API void orc_block(uint64_t seed, uint64_t stream, uint64_t pos, uint32_t out[4])
{
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t ctr[4] = { (uint32_t)pos, (uint32_t)(pos >> 32),
                        (uint32_t)stream, (uint32_t)(stream >> 32) };
    orc_philox4x32_10(ctr, key, out);
}

/* ------------------------------------------------------------------------- */
/* 2. Word -> standard uniform U[0,1) (R-04; "standard uniform U[0,1)"). */
/* ------------------------------------------------------------------------- */
ORC_API double orc_u24(uint32_t w)            /* f32 uniform, exact */
{
    return (double)(w >> 8) * 0x1p-24;
}
ORC_API double orc_u53(uint32_t lo, uint32_t hi) /* f64 uniform, exact */
{
    uint64_t m = ((uint64_t)hi << 32) | (uint64_t)lo;
    return (double)(m >> 11) * 0x1p-53;
}
ORC_API double orc_u32d(uint32_t w)           /* 32-bit f64 uniform, exact */
{
    return (double)w * 0x1p-32;
}

/* ------------------------------------------------------------------------- */
/* 3. cos(2*pi*u), sin(2*pi*u) for a dyadic u in [0,1) (R-06).                */
/*    The plain definition, evaluated with exact argument reduction so the    */
/*    result is accurate to a few ulp RELATIVE even next to the zeros: every  */
/*    subtraction below is exact for dyadic arguments (Sterbenz), and the     */
/*    final libm call sees pi*r with r in [0, 1/4].                           */
/* ------------------------------------------------------------------------- */
ORC_API double orc_cos2pi(double u)
{
    const double PI = 3.14159265358979323846;
    double x = 2.0 * u;          /* exact */
    double s = 1.0;
    if (x >= 1.0) { x = x - 1.0; s = -s; }      /* cos(pi(x+1)) = -cos(pi x) */
    if (x > 0.5)  { x = 1.0 - x; s = -s; }      /* cos(pi(1-x)) = -cos(pi x) */
    if (x <= 0.25) return s * cos(PI * x);
    return s * sin(PI * (0.5 - x));             /* cos(pi x) = sin(pi(1/2-x)) */
}
ORC_API double orc_sin2pi(double u)
{
    const double PI = 3.14159265358979323846;
    double x = 2.0 * u;
    double s = 1.0;
    if (x >= 1.0) { x = x - 1.0; s = -s; }      /* sin(pi(x+1)) = -sin(pi x) */
    if (x > 0.5)  { x = 1.0 - x; }              /* sin(pi(1-x)) = sin(pi x)  */
    if (x <= 0.25) return s * sin(PI * x);
    return s * cos(PI * (0.5 - x));
}

/* Box-Muller (R-06): r = sqrt(-2 ln(1-u_r)), z = r cos / r sin. */
ORC_API double orc_box_muller(double u_r, double u_theta, int use_sin)
{
    double r = sqrt(-2.0 * log(1.0 - u_r));
    return use_sin ? r * orc_sin2pi(u_theta) : r * orc_cos2pi(u_theta);
}

/* ------------------------------------------------------------------------- */
/* 4. Raw words and standard uniforms (R-04, R-12 sample->block map).         */
/* ------------------------------------------------------------------------- */
ORC_API void orc_raw_u32(uint64_t seed, uint64_t stream, uint64_t base,
                         uint32_t *out, uint64_t n)
{
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t w[4];
        orc_block(seed, stream, base + i / 4, w);
        out[i] = w[i % 4];
    }
}
ORC_API void orc_std_uniform_f32(uint64_t seed, uint64_t stream, uint64_t base,
                                 float *out, uint64_t n)
{
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t w[4];
        orc_block(seed, stream, base + i / 4, w);
        out[i] = (float)orc_u24(w[i % 4]);
    }
}
ORC_API void orc_std_uniform_f64(uint64_t seed, uint64_t stream, uint64_t base,
                                 double *out, uint64_t n)
{
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t w[4];
        orc_block(seed, stream, base + i / 2, w);
        int j = (int)(i % 2);
        out[i] = orc_u53(w[2 * j], w[2 * j + 1]);
    }
}

/* Standard deviates consumed by sample i of an f32 / f64 fill (R-12). */
static double std_uniform_at(uint64_t seed, uint64_t stream, uint64_t base,
                             uint64_t i, int is_f64)
{
    uint32_t w[4];
    if (is_f64) {
        orc_block(seed, stream, base + i / 2, w);
        int j = (int)(i % 2);
        return orc_u53(w[2 * j], w[2 * j + 1]);
    }
    orc_block(seed, stream, base + i / 4, w);
    return orc_u24(w[i % 4]);
}
static double std_gaussian_at(uint64_t seed, uint64_t stream, uint64_t base,
                              uint64_t i, int is_f64)
{
    uint32_t w[4];
    if (is_f64) {
        orc_block(seed, stream, base + i / 2, w);
        double ur = orc_u53(w[0], w[1]), ut = orc_u53(w[2], w[3]);
        return orc_box_muller(ur, ut, (int)(i % 2));
    }
    orc_block(seed, stream, base + i / 4, w);
    int p = (int)((i % 4) / 2);
    double ur = orc_u24(w[2 * p]), ut = orc_u24(w[2 * p + 1]);
    return orc_box_muller(ur, ut, (int)(i % 2));
}

/* ------------------------------------------------------------------------- */
/* 5. Reducible distributions with per-sample parameters ("a + (b - a)  */
/*    * x"; P:L69 GetUniform/GetGaussian/GetExponential; P:L87-92 parameters   */
/*    read per sample from memory).  fp64 arithmetic, rounded once to the      */
/*    output type.  Invalid parameters -> NaN, counted (R-07, R-23).           */
/* ------------------------------------------------------------------------- */
static int finite_d(double x) { return isfinite(x); }

static double uniform_one(double a, double b, double u, int *bad)
{
    if (!(finite_d(a) && finite_d(b) && a < b)) { *bad = 1; return NAN; }
    return a + (b - a) * u;
}
static double gaussian_one(double mu, double sigma, double z, int *bad)
{
    if (!(finite_d(mu) && finite_d(sigma) && sigma >= 0.0)) { *bad = 1; return NAN; }
    return mu + sigma * z;
}
static double exponential_one(double lambda, double u, int *bad)
{
    if (!(finite_d(lambda) && lambda > 0.0)) { *bad = 1; return NAN; }
    double e = -log(1.0 - u);          /* standard exponential */
    return e / lambda;                 /* rate parameterisation (R-07)     */
}

#define DEF_FILLS(T, SFX, IS64)                                                    \
ORC_API uint64_t orc_uniform_##SFX(uint64_t seed, uint64_t stream, uint64_t base,  \
        const T *a, const T *b, T *out, uint64_t i0, uint64_t n)                   \
{                                                                                  \
    uint64_t nbad = 0;                                                             \
    for (uint64_t k = 0; k < n; ++k) {                                             \
        uint64_t i = i0 + k; int bad = 0;                                          \
        double u = std_uniform_at(seed, stream, base, i, IS64);                    \
        out[k] = (T)uniform_one((double)a[k], (double)b[k], u, &bad);              \
        nbad += (uint64_t)bad;                                                     \
    }                                                                              \
    return nbad;                                                                   \
}                                                                                  \
ORC_API uint64_t orc_gaussian_##SFX(uint64_t seed, uint64_t stream, uint64_t base, \
        const T *mu, const T *sigma, T *out, uint64_t i0, uint64_t n)              \
{                                                                                  \
    uint64_t nbad = 0;                                                             \
    for (uint64_t k = 0; k < n; ++k) {                                             \
        uint64_t i = i0 + k; int bad = 0;                                          \
        double z = std_gaussian_at(seed, stream, base, i, IS64);                   \
        out[k] = (T)gaussian_one((double)mu[k], (double)sigma[k], z, &bad);        \
        nbad += (uint64_t)bad;                                                     \
    }                                                                              \
    return nbad;                                                                   \
}                                                                                  \
ORC_API uint64_t orc_exponential_##SFX(uint64_t seed, uint64_t stream,             \
        uint64_t base, const T *lambda, T *out, uint64_t i0, uint64_t n)           \
{                                                                                  \
    uint64_t nbad = 0;                                                             \
    for (uint64_t k = 0; k < n; ++k) {                                             \
        uint64_t i = i0 + k; int bad = 0;                                          \
        double u = std_uniform_at(seed, stream, base, i, IS64);                    \
        out[k] = (T)exponential_one((double)lambda[k], u, &bad);                   \
        nbad += (uint64_t)bad;                                                     \
    }                                                                              \
    return nbad;                                                                   \
}

DEF_FILLS(float, f32, 0)
DEF_FILLS(double, f64, 1)

/* ------------------------------------------------------------------------- */
/* 5b. NEXT row N2: the paper's other irreducible getters       */
/*     GetLaplace, GetWeibull and the log-uniform buffer GetLogUniform */
/*     (P:L69).  Algorithms per SPEC S:L231-249 (paper silent, R-30):    */
/*       log-uniform  l = ln(1-u)                     (1 word, like uniform)   */
/*       Laplace      x = mu + beta * s * e,  e = -ln(1-u_a), s = -1 iff u_b<1/2 */
/*                    f32: block i/2, words (2j, 2j+1), j = i mod 2;           */
/*                    f64: block i, e from u53(w0,w1), s from u53(w2,w3)       */
/*       Weibull      x = beta * e^(1/alpha),  e = -ln(1-u)   (1 word)        */
/* ------------------------------------------------------------------------- */
static double laplace_std_at(uint64_t seed, uint64_t stream, uint64_t base, uint64_t i,
                             int is_f64)
{
    uint32_t w[4];
    double ua, ub;
    if (is_f64) {
        orc_block(seed, stream, base + i, w);
        ua = orc_u53(w[0], w[1]); ub = orc_u53(w[2], w[3]);
    } else {
        orc_block(seed, stream, base + i / 2, w);
        int j = (int)(i % 2);
        ua = orc_u24(w[2 * j]); ub = orc_u24(w[2 * j + 1]);
    }
    double e = -log(1.0 - ua);
    return ub < 0.5 ? -e : e;
}

#define DEF_NEXT(T, SFX, IS64)                                                     \
ORC_API void orc_log_uniform_##SFX(uint64_t seed, uint64_t stream, uint64_t base,  \
        T *out, uint64_t i0, uint64_t n)                                           \
{                                                                                  \
    for (uint64_t k = 0; k < n; ++k)                                               \
        out[k] = (T)log(1.0 - std_uniform_at(seed, stream, base, i0 + k, IS64));   \
}                                                                                  \
ORC_API uint64_t orc_laplace_##SFX(uint64_t seed, uint64_t stream, uint64_t base,  \
        const T *mu, const T *beta, T *out, uint64_t i0, uint64_t n)               \
{                                                                                  \
    uint64_t nbad = 0;                                                             \
    for (uint64_t k = 0; k < n; ++k) {                                             \
        double m = (double)mu[k], b = (double)beta[k];                             \
        if (!(finite_d(m) && finite_d(b) && b > 0.0)) { out[k] = (T)NAN; ++nbad; continue; } \
        out[k] = (T)(m + b * laplace_std_at(seed, stream, base, i0 + k, IS64));    \
    }                                                                              \
    return nbad;                                                                   \
}                                                                                  \
ORC_API uint64_t orc_weibull_##SFX(uint64_t seed, uint64_t stream, uint64_t base,  \
        const T *alpha, const T *beta, T *out, uint64_t i0, uint64_t n)            \
{                                                                                  \
    uint64_t nbad = 0;                                                             \
    for (uint64_t k = 0; k < n; ++k) {                                             \
        double a = (double)alpha[k], b = (double)beta[k];                          \
        if (!(finite_d(a) && finite_d(b) && a > 0.0 && b > 0.0)) {                 \
            out[k] = (T)NAN; ++nbad; continue;                                     \
        }                                                                          \
        double e = -log(1.0 - std_uniform_at(seed, stream, base, i0 + k, IS64));   \
        out[k] = (T)(b * pow(e, 1.0 / a));                                         \
    }                                                                              \
    return nbad;                                                                   \
}

DEF_NEXT(float, f32, 0)
DEF_NEXT(double, f64, 1)

/* ------------------------------------------------------------------------- */
/* 6. Gamma by Marsaglia-Tsang (R-08..R-11).  The paper withholds GetGamma     */
/*     but names it an irreducible distribution built on the Gaussian  */
/*    and log-uniform buffers; SPEC states the algorithm        */
/*    (S:L254).  No squeeze: the plain acceptance test.                        */
/* ------------------------------------------------------------------------- */
#define ORC_GAMMA_STRIDE 256u          /* blocks reserved per sample (R-11)   */
#define ORC_GAMMA_MAX_TRIAL 255u

/* One trial given its three uniforms.  Returns 1 = accept (g = d v), 0 =
 * reject.  *margin = (z^2/2 + d - d v + d ln v) - ln U (accept iff > 0) or
 * NAN when 1 + c z <= 0; *onepcz = 1 + c z. */
ORC_API int orc_mt_trial(double d, double c, double u_r, double u_theta, double U,
                         double *g, double *margin, double *onepcz)
{
    double z = sqrt(-2.0 * log(1.0 - u_r)) * orc_cos2pi(u_theta);
    double t = 1.0 + c * z;
    if (onepcz) *onepcz = t;
    if (!(t > 0.0)) { if (margin) *margin = NAN; return 0; }
    double v = t * t * t;
    double rhs = z * z / 2.0 + d - d * v + d * log(v);
    double lu = log(U);
    if (margin) *margin = rhs - lu;
    if (lu < rhs) { if (g) *g = d * v; return 1; }
    return 0;
}

/* Shape-dependent constants (R-08): alpha' = alpha<1 ? alpha+1 : alpha,
 * d = alpha' - 1/3, c = 1/sqrt(9 d). */
ORC_API void orc_mt_consts(double alpha, double *d, double *c)
{
    double ap = alpha < 1.0 ? alpha + 1.0 : alpha;
    *d = ap - 1.0 / 3.0;
    *c = 1.0 / sqrt(9.0 * *d);
}

/* Uniforms of trial t of sample i (R-09): block base + 256 i + t. */
ORC_API void orc_mt_trial_uniforms(uint64_t seed, uint64_t stream, uint64_t base,
                                   uint64_t i, uint32_t t,
                                   double *u_r, double *u_theta, double *U)
{
    uint32_t w[4];
    orc_block(seed, stream, base + (uint64_t)ORC_GAMMA_STRIDE * i + t, w);
    *u_r = orc_u53(w[0], w[1]);
    *u_theta = orc_u32d(w[2]);
    *U = 1.0 - orc_u32d(w[3]);   /* in (0, 1]: ln U finite */
}

/* Gamma(alpha, scale beta) for sample i.  Returns the value; *trial = the
 * accepting trial (1..255) or 0 when invalid / cap exhausted (NaN). */
ORC_API double orc_gamma_one(uint64_t seed, uint64_t stream, uint64_t base, uint64_t i,
                             double alpha, double beta, uint32_t *trial, int *bad)
{
    *trial = 0; *bad = 0;
    if (!(finite_d(alpha) && finite_d(beta) && alpha > 0.0 && beta > 0.0)) {
        *bad = 1; return NAN;
    }
    double d, c;
    orc_mt_consts(alpha, &d, &c);
    double g = NAN;
    uint32_t t;
    for (t = 1; t <= ORC_GAMMA_MAX_TRIAL; ++t) {
        double ur, ut, U;
        orc_mt_trial_uniforms(seed, stream, base, i, t, &ur, &ut, &U);
        if (orc_mt_trial(d, c, ur, ut, U, &g, NULL, NULL)) break;
    }
    if (t > ORC_GAMMA_MAX_TRIAL) { *bad = 1; return NAN; }
    *trial = t;
    if (alpha < 1.0) {
        /* alpha<1 boost (R-10): Gamma(alpha) = Gamma(alpha+1) * U^(1/alpha),
         * written exp(ln(1-u)/alpha) with the sample's block base+256 i. */
        uint32_t w[4];
        orc_block(seed, stream, base + (uint64_t)ORC_GAMMA_STRIDE * i, w);
        double u = orc_u53(w[0], w[1]);
        g = g * exp(log(1.0 - u) / alpha);
    }
    return g * beta;
}

#define DEF_GAMMA(T, SFX)                                                          \
ORC_API uint64_t orc_gamma_##SFX(uint64_t seed, uint64_t stream, uint64_t base,    \
        const T *alpha, const T *beta, T *out, uint8_t *trials,                    \
        uint64_t i0, uint64_t n)                                                   \
{                                                                                  \
    uint64_t nbad = 0;                                                             \
    for (uint64_t k = 0; k < n; ++k) {                                             \
        uint32_t t; int bad;                                                       \
        double g = orc_gamma_one(seed, stream, base, i0 + k, (double)alpha[k],     \
                                 (double)beta[k], &t, &bad);                       \
        out[k] = (T)g;                                                             \
        if (trials) trials[k] = (uint8_t)t;                                        \
        nbad += (uint64_t)bad;                                                     \
    }                                                                              \
    return nbad;                                                                   \
}
DEF_GAMMA(float, f32)
DEF_GAMMA(double, f64)

/* ------------------------------------------------------------------------- */
/* 7. Dirichlet from Gammas (P:L34 footnote: "draw K y_i's from               */
/*    Gamma(alpha_i,1). Next we normalize: x_i = y_i / sum_i y_i"; R-13).      */
/*    Component k of row r is Gamma sample i = r K + k with beta = 1.          */
/* ------------------------------------------------------------------------- */
#define DEF_DIRICHLET(T, SFX)                                                      \
ORC_API uint64_t orc_dirichlet_##SFX(uint64_t seed, uint64_t stream, uint64_t base,\
        const T *alpha, uint64_t k_dim, T *out, uint8_t *trials,                   \
        uint64_t row0, uint64_t n_rows, double *g_scratch)                         \
{                                                                                  \
    uint64_t nbad = 0;                                                             \
    for (uint64_t r = 0; r < n_rows; ++r) {                                        \
        uint64_t row = row0 + r;                                                   \
        double S = 0.0;                                                            \
        for (uint64_t k = 0; k < k_dim; ++k) {                                     \
            uint32_t t; int bad;                                                   \
            double y = orc_gamma_one(seed, stream, base, row * k_dim + k,          \
                                     (double)alpha[r * k_dim + k], 1.0, &t, &bad); \
            g_scratch[k] = y;                                                      \
            if (trials) trials[r * k_dim + k] = (uint8_t)t;                        \
            nbad += (uint64_t)bad;                                                 \
            S = S + y;                                                             \
        }                                                                          \
        for (uint64_t k = 0; k < k_dim; ++k)                                       \
            out[r * k_dim + k] = (T)(g_scratch[k] / S);                            \
    }                                                                              \
    return nbad;                                                                   \
}
DEF_DIRICHLET(float, f32)
DEF_DIRICHLET(double, f64)

/* ------------------------------------------------------------------------- */
/* 8. Gibbs sampling on the triangle (Eq. 1; Fig. 1):       */
/*      x ~ U(0, 1-y);  y ~ U(0, 1-x)   from (x0, y0) = (0.5, 0.5)            */
/*    Chain c uses stream stream_id + c; sweep s uses block base + s; x from  */
/*    u53(w0,w1), y from u53(w2,w3) (R-14..R-17).  Per-chain statistics and   */
/*    the 256-bin histogram of x over sweeps >= burn_in (R-18, R-19).          */
/*    out_x/out_y: [n_sweeps][n_chains] (nullable); chain_stats:              */
/*    [5][n_chains] = mean_x, var_x, mean_y, var_y, cov_xy (nullable);        */
/*    final_xy: [2][n_chains] (nullable); totals: f64[16 + 256] (nullable,    */
/*    ACCUMULATED into, layout in DESIGN.md R-18).                            */
/* ------------------------------------------------------------------------- */
#define ORC_TOTALS_HDR 16
ORC_API uint64_t orc_gibbs_triangle(uint64_t seed, uint64_t stream_id, uint64_t base,
        uint64_t n_chains, uint64_t n_sweeps, const double *x0, const double *y0,
        uint64_t burn_in, double *out_x, double *out_y, double *chain_stats,
        double *final_xy, double *totals)
{
    uint64_t nbad = 0;
    for (uint64_t c = 0; c < n_chains; ++c) {
        double x = x0 ? x0[c] : 0.5;
        double y = y0 ? y0[c] : 0.5;
        if (!(y >= 0.0 && y <= 1.0)) { x = NAN; y = NAN; ++nbad; }
        double s1x = 0.0, s2x = 0.0, s1y = 0.0, s2y = 0.0, sxy = 0.0;
        for (uint64_t s = 0; s < n_sweeps; ++s) {
            uint32_t w[4];
            orc_block(seed, stream_id + c, base + s, w);
            x = (1.0 - y) * orc_u53(w[0], w[1]);   /* x ~ U(0, 1-y) */
            y = (1.0 - x) * orc_u53(w[2], w[3]);   /* y ~ U(0, 1-x) */
            if (out_x) out_x[s * n_chains + c] = x;
            if (out_y) out_y[s * n_chains + c] = y;
            if (s >= burn_in) {
                s1x = s1x + x; s2x = fma(x, x, s2x);
                s1y = s1y + y; s2y = fma(y, y, s2y);
                sxy = fma(x, y, sxy);
                if (totals && x >= 0.0 && x < 1.0) {
                    int bin = (int)floor(x * 256.0);
                    totals[ORC_TOTALS_HDR + bin] += 1.0;
                }
            }
        }
        double n = (double)(n_sweeps - burn_in);
        double mx = s1x / n, my = s1y / n;
        double vx = (s2x - s1x * mx) / (n - 1.0);
        double vy = (s2y - s1y * my) / (n - 1.0);
        double cxy = (sxy - s1x * my) / (n - 1.0);
        if (chain_stats) {
            chain_stats[0 * n_chains + c] = mx;
            chain_stats[1 * n_chains + c] = vx;
            chain_stats[2 * n_chains + c] = my;
            chain_stats[3 * n_chains + c] = vy;
            chain_stats[4 * n_chains + c] = cxy;
        }
        if (final_xy) { final_xy[c] = x; final_xy[n_chains + c] = y; }
        if (totals) {
            totals[0] += mx; totals[1] += vx; totals[2] += mx * mx;
            totals[3] += my; totals[4] += vy; totals[5] += my * my;
            totals[6] += cxy; totals[7] += mx * my;
            totals[8] += 1.0; totals[9] += n;
        }
    }
    return nbad;
}
