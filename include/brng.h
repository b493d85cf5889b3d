/*
 * brng.h -- C ABI of libbrng: varying-parameter random deviates on NVIDIA B200
 * (sm_100a), the data-parallel hot path of arXiv 1412.4825 ("BatchRNG").
 *
 * Citation keys: P:Lnn = PAPER.md line nn (/root/reference, section given);
 * R-nn = the numbered readings in DESIGN.md ("Contract") that fix what the
 * paper leaves open.  The counter map and every per-sample formula below are
 * the contract that the CPU oracle (oracle/) implements independently.
 *
 * ---------------------------------------------------------------------------
 * Conventions common to every entry point
 * ---------------------------------------------------------------------------
 *  Handle.   A brng_t is the GPU recast of the paper's BatchRNG object
 *            (P:L54-66): the engine state is (seed, stream_id, block cursor)
 *            instead of VSL stream state + buffers + buffer counters.  It also
 *            owns a little device scratch (an invalid-sample counter, the
 *            Gamma/Dirichlet work counter, Gibbs reduction partials) shared
 *            by its calls.  One handle = one consumer at a time; distinct
 *            handles may be used concurrently on distinct streams.
 *  Counter map (R-01, R-02).  Every random word is a word of a Philox4x32-10
 *            block with key = (lo32 seed, hi32 seed) and counter = (lo32 pos,
 *            hi32 pos, lo32 stream, hi32 stream); pos is a 64-bit BLOCK index.
 *  Cursor (R-12).  A call uses blocks [cursor, cursor + span) of stream
 *            stream_id (Gibbs: of streams stream_id + c) and advances the
 *            cursor by span AT ENQUEUE TIME on the host, so results never
 *            depend on execution timing, grid shape or GPU count.
 *            span = ceil(n/4) for f32 fills and raw words, ceil(n/2) for f64
 *            fills (Laplace: ceil(n/2) f32, n f64), 256*n for Gamma, 256*n_rows*k for Dirichlet, n_sweeps for
 *            Gibbs.  Sample i of a call is a pure function of (seed, stream,
 *            cursor at enqueue, i, the i-th parameters).
 *  Pointers. Arrays are caller-owned, contiguous, any alignment (16-byte
 *            aligned arrays take the vectorised path).  DEVICE pointers (on
 *            the handle's device) are used in place and the call is
 *            asynchronous on the handle's CUDA stream: inputs must stay valid
 *            and unmodified, outputs untouched, until the stream passes the
 *            call.  HOST pointers (pinned or pageable) are staged through
 *            device memory by the library (host->device copy, kernel,
 *            device->host copy on the handle's stream); such a call returns
 *            only after its outputs are in host memory.
 *  Errors.   Every entry point returns BRNG_OK (0) or a negative brng_status.
 *            Host-detectable problems (null handle or required pointer, size
 *            overflow, cursor overflow past 2^64, k == 0, burn_in > n_sweeps)
 *            return synchronously with NO launch and NO cursor change.
 *            n == 0 is a no-op returning BRNG_OK with the cursor unchanged.
 *            Invalid PER-SAMPLE parameters (below) make that output NaN and
 *            increment the handle's device counter, read by
 *            brng_device_errors().  CUDA launch/runtime failures return
 *            BRNG_ERR_CUDA (cursor unchanged).
 *  Precision. f32 entry points read/write binary32 and compute the reducible
 *            transforms in binary32; Gamma/Dirichlet compute in binary64
 *            internally for every output type (R-28); Gibbs is binary64
 *            with IEEE sub/mul/fma only (bit-exact).  No fast-math; denormals
 *            preserved.  Transcendentals: binary32 libm (logf, sqrtf) plus a
 *            table sincos for the f32 fills; binary64 fills and the Gamma
 *            trial/boost use the library's table-driven ln/cos/exp and a
 *            Newton rsqrt (1-2 ulp, include/brng_device.cuh),
 *            well inside the 2e-6 / 1e-12 parity tolerances.
 */
#ifndef BRNG_H
#define BRNG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define BRNG_API __attribute__((visibility("default")))
#else
#define BRNG_API
#endif

#define BRNG_VERSION 1
#define BRNG_GAMMA_STRIDE 256u   /* Philox blocks reserved per Gamma sample (R-11) */
#define BRNG_GAMMA_MAX_TRIAL 255u
#define BRNG_TOTALS_HDR 16u      /* Gibbs totals: 16 moment slots + 256 bins (R-18) */
#define BRNG_TOTALS_LEN (BRNG_TOTALS_HDR + 256u)

typedef struct brng_handle_s* brng_t;

typedef enum brng_status {
    BRNG_OK = 0,
    BRNG_ERR_NULL = -1,      /* null handle or required pointer            */
    BRNG_ERR_SIZE = -2,      /* size overflow / k == 0 / burn_in > sweeps  */
    BRNG_ERR_CUDA = -3,      /* CUDA runtime error (launch, copy, alloc)   */
    BRNG_ERR_PARAM = -4,     /* invalid scalar argument                    */
    BRNG_ERR_OVERFLOW = -5,  /* cursor + span would pass 2^64              */
    BRNG_ERR_STATE = -6      /* the handle's device cannot be made current */
} brng_status;

/* ---- lifecycle (the paper's constructor / destructor) ---------- */

/* Create a handle bound to the CURRENT CUDA device, cursor 0, default stream.
 * Every later call runs on that device whatever device is current in the
 * calling thread, and leaves the caller's current device unchanged.
 * seed: Philox key (any value, including 0).  stream_id: Philox stream (upper
 * counter half) used by every fill/Gamma/Dirichlet call; Gibbs chain c uses
 * stream stream_id + c.  *out receives the handle.  Allocates 16 B of device
 * counters (the Gibbs partials, ~0.6 MB, on the first Gibbs call; a binary32
 * Dirichlet call with K > 1024 grows a scratch of one row of K doubles per
 * resident warp, at most 2 GB). */
BRNG_API int brng_create(uint64_t seed, uint64_t stream_id, brng_t* out);
/* Synchronise the handle's stream and free the handle and its scratch. */
BRNG_API int brng_destroy(brng_t h);
/* Enqueue subsequent calls on this cudaStream_t (e.g. torch's current stream;
 * NULL = legacy default stream).  Not owned by the handle.  Switching streams
 * makes the new stream wait for the work already enqueued on the old one
 * (the handle's device scratch is shared by its calls). */
BRNG_API int brng_set_cuda_stream(brng_t h, void* cuda_stream);
BRNG_API int brng_get_offset(brng_t h, uint64_t* block_cursor);
/* Reposition the cursor (resume a checkpoint, or shard: rank r of a data-
 * parallel job sets cursor = base + r * span_per_rank, R-20). */
BRNG_API int brng_set_offset(brng_t h, uint64_t block_cursor);
BRNG_API int brng_get_key(brng_t h, uint64_t* seed, uint64_t* stream_id);
/* Number of invalid-parameter / trial-cap samples seen since the last reset.
 * Synchronises the handle's stream. */
BRNG_API int brng_device_errors(brng_t h, uint64_t* n_invalid);
BRNG_API int brng_reset_device_errors(brng_t h);
/* cudaStreamSynchronize on the handle's stream. */
BRNG_API int brng_synchronize(brng_t h);
BRNG_API const char* brng_status_string(int status);
BRNG_API int brng_version(void);

/* ---- base generator and standard deviates (R-01..R-04) ----- */

/* out[i] = word (i mod 4) of block cursor + floor(i/4).  u32[n]. */
BRNG_API int brng_raw_u32(brng_t h, uint32_t* out, uint64_t n);
/* out[i] = u24(w) = (w >> 8) * 2^-24 in [0, 1-2^-24], w as for raw_u32. */
BRNG_API int brng_std_uniform_f32(brng_t h, float* out, uint64_t n);
/* out[i] = u53(w[2j], w[2j+1]) = ((w[2j+1]*2^32 + w[2j]) >> 11) * 2^-53 with
 * j = i mod 2 of block cursor + floor(i/2); in [0, 1-2^-53]. */
BRNG_API int brng_std_uniform_f64(brng_t h, double* out, uint64_t n);

/* ---- reducible distributions, per-sample parameters -------
 * The paper's GetUniform/GetGaussian/GetExponential called once per sample
 * with parameters read from memory, as one fused pass:
 * Philox -> standard deviate -> per-sample transform -> store.
 *   uniform:     out[i] = a[i] + (b[i]-a[i]) * u_i           valid iff a<b, finite
 *   gaussian:    out[i] = mu[i] + sigma[i] * z_i              valid iff sigma>=0, finite
 *   exponential: out[i] = -ln(1-u_i) / lambda[i]  (rate, R-07) valid iff lambda>0, finite
 * u_i: the standard uniform of std_uniform_{f32,f64} at the same i.
 * z_i (Box-Muller, R-06): f32 -- block cursor+floor(i/4), pair p=(i mod 4)/2:
 *   r = sqrt(-2 ln(1-u24(w[2p]))), theta = 2 pi u24(w[2p+1]); even i -> r cos
 *   theta, odd i -> r sin theta.  f64 -- block cursor+floor(i/2): r from
 *   u53(w0,w1), theta from u53(w2,w3); even i -> cos, odd -> sin.
 * All arrays length n. */
BRNG_API int brng_uniform_f32(brng_t h, const float* a, const float* b, float* out, uint64_t n);
BRNG_API int brng_uniform_f64(brng_t h, const double* a, const double* b, double* out, uint64_t n);
BRNG_API int brng_gaussian_f32(brng_t h, const float* mu, const float* sigma, float* out, uint64_t n);
BRNG_API int brng_gaussian_f64(brng_t h, const double* mu, const double* sigma, double* out, uint64_t n);
BRNG_API int brng_exponential_f32(brng_t h, const float* lambda, float* out, uint64_t n);
BRNG_API int brng_exponential_f64(brng_t h, const double* lambda, double* out, uint64_t n);

/* ---- NEXT row N2: the paper's other getters (P:L69 GetLogUniform; P:L70
 * GetLaplace, GetWeibull; algorithms R-30 / SPEC S:L221-249) ----------------
 *   log-uniform: out[i] = ln(1 - u_i)            (u_i as std_uniform; <= 0)
 *   Laplace:     out[i] = mu[i] + beta[i] * s * e, e = -ln(1-u_a), s = -1 iff
 *                u_b < 1/2; valid iff beta > 0, finite.  Two uniforms per
 *                sample: f32 -- block cursor+floor(i/2), (u_a,u_b) = u24 of
 *                words (2j, 2j+1), j = i mod 2 (span ceil(n/2)); f64 -- block
 *                cursor+i, u_a = u53(w0,w1), u_b = u53(w2,w3) (span n).
 *   Weibull:     out[i] = beta[i] * e^(1/alpha[i]), e = -ln(1-u_i) (shape
 *                alpha, scale beta); valid iff alpha > 0, beta > 0, finite.
 * All arrays length n. */
BRNG_API int brng_log_uniform_f32(brng_t h, float* out, uint64_t n);
BRNG_API int brng_log_uniform_f64(brng_t h, double* out, uint64_t n);
BRNG_API int brng_laplace_f32(brng_t h, const float* mu, const float* beta, float* out, uint64_t n);
BRNG_API int brng_laplace_f64(brng_t h, const double* mu, const double* beta, double* out,
                              uint64_t n);
BRNG_API int brng_weibull_f32(brng_t h, const float* alpha, const float* beta, float* out,
                              uint64_t n);
BRNG_API int brng_weibull_f64(brng_t h, const double* alpha, const double* beta, double* out,
                              uint64_t n);

/* ---- fixed-parameter batch fill (NEXT row N1: the paper's "VSL-Batch"
 * column) --------------------------------
 * Every sample i uses the same parameters (p0, p1) -- no parameter arrays,
 * 4 (f32) / 8 (f64) bytes per sample.  dist: BRNG_DIST_UNIFORM (a, b),
 * _GAUSSIAN (mu, sigma), _EXPONENTIAL (lambda, unused), _LAPLACE (mu, beta),
 * _WEIBULL (alpha, beta); dtype: BRNG_DTYPE_F32 / _F64.  Same counters, span
 * and values as the per-sample call with constant parameter arrays.  An
 * unknown dist/dtype returns BRNG_ERR_PARAM; invalid p0/p1 make every output
 * NaN and are counted per sample. */
#define BRNG_DIST_UNIFORM 2
#define BRNG_DIST_GAUSSIAN 3
#define BRNG_DIST_EXPONENTIAL 4
#define BRNG_DIST_LAPLACE 6
#define BRNG_DIST_WEIBULL 7
#define BRNG_DTYPE_F32 0
#define BRNG_DTYPE_F64 1
BRNG_API int brng_batch_fill(brng_t h, int dist, int dtype, double p0, double p1, void* out,
                             uint64_t n);

/* ---- Gamma (Marsaglia-Tsang, R-08..R-11) -----------
 * out[i] ~ Gamma(shape alpha[i], scale beta[i]); valid iff alpha>0, beta>0,
 * finite.  alpha' = alpha<1 ? alpha+1 : alpha; d = alpha' - 1/3;
 * c = 1/sqrt(9d).  Trial t = 1..255 uses block cursor + 256 i + t:
 * z = sqrt(-2 ln(1-u53(w0,w1))) cos(2 pi u32d(w2)), U = 1 - u32d(w3);
 * reject if 1+cz <= 0, else v = (1+cz)^3, accept iff
 * ln U < z^2/2 + d - d v + d ln v; g = d v.  alpha<1: g *= exp(ln(1-u)/alpha)
 * with u = u53(w0,w1) of block cursor + 256 i (the U^(1/alpha) boost).
 * out[i] = g * beta[i].  No acceptance by t = 255 -> NaN, counted.
 * trials (nullable, u8[n]): accepting trial index, 0 for NaN outputs. */
BRNG_API int brng_gamma_f32(brng_t h, const float* alpha, const float* beta, float* out, uint64_t n,
                   uint8_t* trials);
BRNG_API int brng_gamma_f64(brng_t h, const double* alpha, const double* beta, double* out, uint64_t n,
                   uint8_t* trials);

/* ---- Dirichlet (P:L34 footnote: x_i = y_i / sum y_i, y_i ~ Gamma(alpha_i,1))
 * alpha, out: row-major [n_rows][k].  Component (r, j) is Gamma sample
 * i = r*k + j of the contract above with beta = 1; S_r = sum_j y_rj (binary64,
 * any order); out[r][j] = y_rj / S_r rounded to the output type.  An invalid
 * component makes its whole row NaN.  trials: nullable u8[n_rows][k].
 * 1 <= k < 2^24 (BRNG_ERR_SIZE otherwise).
 * Arithmetic: the kernels form fl(1/S_r) once per row and output
 * y_rj * fl(1/S_r) (binary64) rounded to the output type; this is within one
 * binary64 ulp of y_rj / S_r before that rounding, inside the parity
 * tolerance (the oracle divides, as the definition states).  The sum is
 * taken lane-strided then by a fixed shuffle tree: deterministic for given
 * (alpha, k). */
BRNG_API int brng_dirichlet_f32(brng_t h, const float* alpha, uint64_t n_rows, uint64_t k, float* out,
                       uint8_t* trials);
BRNG_API int brng_dirichlet_f64(brng_t h, const double* alpha, uint64_t n_rows, uint64_t k, double* out,
                       uint8_t* trials);

/* ---- Gibbs sampling on the triangle (Eq. 1 and Fig. 1) ---------
 * n_chains independent chains; chain c uses Philox stream stream_id + c and
 * sweep s uses block cursor + s:  x = (1-y) u53(w0,w1);  y = (1-x) u53(w2,w3)
 * (x ~ U(0,1-y) then y ~ U(0,1-x), R-15/R-16), starting from (x0[c], y0[c])
 * (nullable: 0.5 each, Fig. 1).  Cursor advances by n_sweeps, so a run split
 * into calls that pass the previous final_xy as x0/y0 is bit-identical.
 *   out_x, out_y  (nullable) f64[n_sweeps][n_chains]: every sample.
 *   chain_stats   (nullable) f64[5][n_chains]: mean_x, var_x, mean_y, var_y,
 *                 cov_xy over sweeps s >= burn_in (n-1 divisor; R-18).
 *   final_xy      (nullable) f64[2][n_chains].
 *   totals        (nullable) f64[272], OVERWRITTEN: [0] sum_c mean_x, [1] sum
 *                 var_x, [2] sum mean_x^2, [3] sum mean_y, [4] sum var_y,
 *                 [5] sum mean_y^2, [6] sum cov_xy, [7] sum mean_x*mean_y,
 *                 [8] n_chains, [9] n_chains*(n_sweeps-burn_in), [10..15] 0,
 *                 [16+b] count of x samples with floor(256 x) = b (R-19).
 *                 Summation order is fixed for a given launch shape
 *                 (deterministic run to run); a call chunked differently
 *                 (host buffers) or sharded over ranks gives the same
 *                 histogram and per-chain values but moment totals equal
 *                 only to rounding (~1e-15 relative).
 * A chain with y0 outside [0,1] (or NaN) yields NaN and is counted.
 * Limits: n_sweeps < 2^22 (BRNG_ERR_SIZE otherwise: the per-CTA histogram
 * counters are 32-bit, and a CTA round holds at most 768 chains, so a bin
 * stays below 768 * 2^22 < 2^32 by construction); burn_in <= n_sweeps;
 * stream_id + n_chains must not pass 2^64 (BRNG_ERR_OVERFLOW).
 * Graph capture: the first call of a given chain count allocates the
 * handle's partial-sum scratch and must run eagerly; inside a capture a call
 * that would need a larger scratch returns BRNG_ERR_STATE. */
BRNG_API int brng_gibbs_triangle(brng_t h, uint64_t n_chains, uint64_t n_sweeps, const double* x0,
                        const double* y0, uint64_t burn_in, double* out_x, double* out_y,
                        double* chain_stats, double* final_xy, double* totals);

/* ---- NEXT row N4: LDA fold-in Gibbs consumer (R-33) -------
 * The paper's motivating use: Gibbs sampling of LDA, which draws a Dirichlet
 * deviate whose parameters change every iteration.  Fold-in: the
 * topic-word matrix phi is FIXED (inference of new documents' topics).
 * Corpus (device pointers only, else BRNG_ERR_PARAM): n_docs documents in CSR
 * form, doc_off u64[n_docs + 1] (doc_off[0] = 0, non-decreasing,
 * doc_off[n_docs] = n_tokens), words u32[n_tokens] (< v), phi f64[v][k]
 * (row w = phi[w, 0..k-1], >= 0), alpha f64[k] (> 0), z u16[n_tokens]
 * (topics < k; IN: the current state, OUT: the state after n_iter
 * iterations), theta (nullable) f64[n_docs][k]: theta of the last iteration.
 * Iteration t at cursor c_t = cursor + t * span, span = 256 n_docs k +
 * ceil(n_tokens / 2) blocks (the cursor advances by n_iter * span):
 *   n_dk    = #{tokens j of document d with z_j = k};
 *   theta_d = Dirichlet(alpha + n_d.) drawn exactly as brng_dirichlet_f64 at
 *             cursor c_t would (component (d, k) = Gamma sample d k + k);
 *   u_j     = brng_std_uniform_f64 sample j at cursor c_t + 256 n_docs k;
 *   z_j     = the first k with fl(u_j C_j) < c_jk, where p_jk =
 *             fl(theta_dk phi[w_j, k]), c_jk = fl(c_j,k-1 + p_jk) in k order,
 *             C_j = c_j,k-1 (binary64, no FMA); else the last k with p_jk > 0.
 * mode: BRNG_LDA_INLINE (the consumer kernel calls the device API getters),
 * BRNG_LDA_RING (asynchronous service: a producer kernel on a side stream
 * fills a two-slot ring with iteration t+1's parameter-free standard
 * deviates -- trial-1 normals, boost log-uniforms, token uniforms -- while the
 * consumer runs iteration t), BRNG_LDA_BULK (per iteration: counts, the
 * library's Dirichlet and uniform-fill kernels into scratch, then the
 * consumer).  All three give the same bits.  A component whose alpha_k + n_dk
 * is not positive and finite makes the document's theta NaN (counted once
 * per such component) and its tokens' z = 0.  A document range that
 * decreases or passes n_tokens is counted and treated as empty; a token with
 * words[j] >= v is counted and keeps its z (no out-of-range access either
 * way); topics z >= k count as topic k-1.  k <= BRNG_LDA_MAX_K.  RING/BULK use handle-owned scratch
 * (two slots of 20 n_docs k + 8 n_tokens bytes / 16 n_docs k + 8 n_tokens),
 * grown on the first call of a size (not inside a graph capture:
 * BRNG_ERR_STATE).  Asynchronous on the handle's stream. */
#define BRNG_LDA_INLINE 0
#define BRNG_LDA_RING 1
#define BRNG_LDA_BULK 2
#define BRNG_LDA_MAX_K 1024u
BRNG_API int brng_lda_gibbs(brng_t h, uint64_t n_docs, uint32_t k, uint32_t v, uint64_t n_tokens,
                            const uint64_t* doc_off, const uint32_t* words, const double* phi,
                            const double* alpha, uint16_t* z, double* theta, uint32_t n_iter,
                            int mode);

#ifdef __cplusplus
}
#endif
#endif /* BRNG_H */
