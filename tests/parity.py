"""Parity criteria between the CUDA path and the CPU oracle (DESIGN.md
"Parity criteria"), shared by the -m gpu tests and __graft_entry__.smoke().

- bit-exact: raw words, standard uniforms, Gibbs samples/stats/histograms;
- tolerance: |x - x_ref| <= tau * scale + eps_min, tau = 1e-12 (f64) /
  2e-6 (f32) (BASELINE.json north_star), eps_min = smallest subnormal;
  scale = |mu| + |sigma z_ref| (Gaussian), |a| + |b - a| u (uniform),
  |x_ref| otherwise;
- Gamma/Dirichlet decisions: the accepting trial must agree; a disagreement
  is a boundary TIE iff the oracle's margin at the first disagreeing trial is
  within 1e-10 max(1, d) (or |1 + c z| <= 1e-10), else a FAIL.  Ties must
  stay below 1e-6 of the samples.
"""
from __future__ import annotations

import numpy as np

import oracle

TAU = {np.dtype(np.float32): 2e-6, np.dtype(np.float64): 1e-12}
# absolute floor: tau times the smallest NORMAL number (a subnormal result
# carries fewer significant bits; 2e-6 x 1.2e-38 and 1e-12 x 2.2e-308), but
# never below one subnormal ulp
EPS_MIN = {dt: max(float(np.finfo(dt).smallest_subnormal), TAU[dt] * float(np.finfo(dt).tiny))
           for dt in (np.dtype(np.float32), np.dtype(np.float64))}
TIE_BAND = 1e-10
TIE_RATE_MAX = 1e-6


def _np(x):
    if hasattr(x, "detach"):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def fill_reference(dist, seed, stream, base, params, i0, dtype):
    """Oracle values and error scale for samples i0 .. i0+len-1."""
    dtype = np.dtype(dtype)
    if dist == "uniform":
        a, b = params
        ref, _ = oracle.uniform(seed, stream, base, a, b, i0=i0, dtype=dtype)
        u = _std_at(seed, stream, base, i0, len(a), dtype)
        scale = np.abs(a.astype(np.float64)) + np.abs(b.astype(np.float64) - a) * u
    elif dist == "gaussian":
        mu, sigma = params
        ref, _ = oracle.gaussian(seed, stream, base, mu, sigma, i0=i0, dtype=dtype)
        # standard normal at the same positions (f32 path: its rounded value,
        # which changes the scale by < 1e-7 relative)
        z, _ = oracle.gaussian(seed, stream, base, np.zeros(len(mu), dtype),
                               np.ones(len(mu), dtype), i0=i0, dtype=dtype)
        scale = np.abs(mu.astype(np.float64)) + np.abs(sigma.astype(np.float64) * z.astype(np.float64))
    elif dist == "exponential":
        (lam,) = params
        ref, _ = oracle.exponential(seed, stream, base, lam, i0=i0, dtype=dtype)
        scale = np.abs(ref.astype(np.float64))
    elif dist == "log_uniform":
        (n,) = params
        ref = oracle.log_uniform(seed, stream, base, n, i0=i0, dtype=dtype)
        scale = np.abs(ref.astype(np.float64))
    elif dist == "laplace":
        mu, beta = params
        ref, _ = oracle.laplace(seed, stream, base, mu, beta, i0=i0, dtype=dtype)
        s, _ = oracle.laplace(seed, stream, base, np.zeros(len(mu), dtype), np.ones(len(mu), dtype),
                              i0=i0, dtype=dtype)
        scale = np.abs(mu.astype(np.float64)) + np.abs(beta.astype(np.float64) * s.astype(np.float64))
    elif dist == "weibull":
        alpha, beta = params
        ref, _ = oracle.weibull(seed, stream, base, alpha, beta, i0=i0, dtype=dtype)
        # x = beta e^(1/alpha): a relative error in e (or in ln e) is amplified
        # by 1/alpha (and |ln e| / alpha), so the scale carries that condition
        e, _ = oracle.exponential(seed, stream, base, np.ones(len(alpha), dtype), i0=i0,
                                  dtype=dtype)
        with np.errstate(divide="ignore"):
            lne = np.abs(np.log(e.astype(np.float64)))
        lne[~np.isfinite(lne)] = 0.0
        cond = np.maximum(1.0, (1.0 + lne) / alpha.astype(np.float64))
        scale = np.abs(ref.astype(np.float64)) * cond
    else:
        raise ValueError(dist)
    return ref, scale


def _std_at(seed, stream, base, i0, n, dtype):
    per = 2 if dtype == np.float64 else 4
    blk0 = i0 // per
    off = i0 - blk0 * per
    u = oracle.std_uniform(seed, stream, base + blk0, off + n, dtype)
    return u[off:].astype(np.float64)


def check_close(got, ref, scale, dtype, what=""):
    """Max of |got-ref| / (tau*scale + eps_min); asserts <= 1.  NaN must match NaN."""
    dtype = np.dtype(dtype)
    got = _np(got).astype(np.float64)
    ref = np.asarray(ref).astype(np.float64)
    nan_g, nan_r = np.isnan(got), np.isnan(ref)
    assert np.array_equal(nan_g, nan_r), f"{what}: NaN pattern differs ({nan_g.sum()} vs {nan_r.sum()})"
    m = ~nan_r
    bound = TAU[dtype] * np.asarray(scale)[m] + EPS_MIN[dtype]
    err = np.abs(got[m] - ref[m])
    ratio = float(np.max(err / bound)) if err.size else 0.0
    if ratio > 1.0:
        k = int(np.argmax(err / bound))
        idx = np.flatnonzero(m)[k]
        raise AssertionError(f"{what}: error ratio {ratio:.3g} at {idx}: got {got[idx]!r} "
                             f"ref {ref[idx]!r} scale {np.asarray(scale)[idx]!r}")
    return ratio


def gamma_compare(got, trials, alpha, beta, seed, stream, base, i0=0, dtype=np.float64,
                  index=None):
    """Compare GPU Gamma outputs for samples `index` (default i0..i0+n-1).
    Returns dict(n, n_tie, n_fail, ratio)."""
    dtype = np.dtype(dtype)
    got = _np(got); trials = _np(trials)
    alpha = np.asarray(alpha); beta = np.asarray(beta)
    n = len(got)
    idx = np.arange(i0, i0 + n) if index is None else np.asarray(index)
    ref = np.empty(n, dtype); tref = np.zeros(n, np.uint8)
    if index is None:
        ref, tref, _ = oracle.gamma(seed, stream, base, alpha, beta, i0=i0, dtype=dtype)
    else:
        for k, i in enumerate(idx):
            r, t, _ = oracle.gamma(seed, stream, base, alpha[k:k + 1], beta[k:k + 1], i0=int(i),
                                   dtype=dtype)
            ref[k] = r[0]; tref[k] = t[0]
    return _decide(got, trials, ref, tref, alpha, seed, stream, base, idx, dtype)


def value_check(got, ref, scale, dtype, cond_at=None, what="values"):
    """The value criterion with its relaxations made auditable.

    Bound = tau * scale * cond + EPS_MIN, where cond = cond_at(k) (the
    Marsaglia-Tsang condition number, Gamma/Dirichlet) is applied only where
    the plain bound tau * scale + EPS_MIN fails.  Returns dict(ratio = max
    error / bound (must be <= 1), n_values = values compared, worst_plain_rel = max
    |x - x_ref| / |x_ref| over x_ref != 0, n_plain_fail = samples outside the
    literal SURVEY 8c.5 bound tau |x_ref| + one subnormal, n_floor = those
    rescued by the tau * smallest-normal floor alone, n_cond = those that
    needed the condition factor)."""
    dtype = np.dtype(dtype)
    got = _np(got).astype(np.float64)
    ref = np.asarray(ref).astype(np.float64)
    scale = np.array(scale, dtype=np.float64, copy=True)
    nan_g, nan_r = np.isnan(got), np.isnan(ref)
    assert np.array_equal(nan_g, nan_r), f"{what}: NaN pattern differs"
    m = ~nan_r
    got, ref, scale = got[m], ref[m], scale[m]
    err = np.abs(got - ref)
    tau, sub = TAU[dtype], float(np.finfo(dtype).smallest_subnormal)
    nz = ref != 0
    worst_plain = float(np.max(err[nz] / np.abs(ref[nz]))) if nz.any() else 0.0
    plain_fail = ~(err <= tau * np.abs(ref) + sub)
    loose = ~(err <= tau * scale + EPS_MIN[dtype])
    n_floor = int(np.count_nonzero(plain_fail & ~loose & (err <= tau * np.abs(ref) + EPS_MIN[dtype])))
    if cond_at is not None:
        ks = np.flatnonzero(m)
        for k in np.flatnonzero(loose):
            scale[k] *= max(1.0, cond_at(int(ks[k])))
    bound = tau * scale + EPS_MIN[dtype]
    ratio = float(np.max(err / bound)) if err.size else 0.0
    if ratio > 1.0:
        k = int(np.argmax(err / bound))
        raise AssertionError(f"{what}: error ratio {ratio:.3g}: got {got[k]!r} ref {ref[k]!r}")
    return dict(ratio=ratio, n_values=int(err.size), worst_plain_rel=worst_plain,
                n_plain_fail=int(np.count_nonzero(plain_fail)), n_floor=n_floor,
                n_cond=int(np.count_nonzero(loose)))


def _decide(got, trials, ref, tref, alpha, seed, stream, base, idx, dtype):
    same = trials == tref
    n_tie = n_fail = 0
    fails = []
    for k in np.flatnonzero(~same):
        t_star = int(min(trials[k], tref[k]))
        if t_star == 0:
            n_fail += 1; fails.append(int(idx[k])); continue
        m, onepcz, d = oracle.gamma_tie_margin(seed, stream, base, int(idx[k]), float(alpha[k]),
                                               t_star)
        if (np.isfinite(m) and abs(m) <= TIE_BAND * max(1.0, d)) or abs(onepcz) <= TIE_BAND:
            n_tie += 1
        else:
            n_fail += 1; fails.append(int(idx[k]))
    # conditioning: g = d (1 + c z)^3 has condition 3|c z / (1 + c z)| in z, so
    # any 1-ulp difference in z (log, sqrt, cos) is amplified near 1 + cz -> 0;
    # the scale carries that factor where the plain bound fails
    ks = np.flatnonzero(same)
    vc = value_check(got[same], ref[same], np.abs(ref[same].astype(np.float64)), dtype,
                     lambda j: gamma_condition(seed, stream, base, int(idx[ks[j]]),
                                               float(alpha[ks[j]]), int(tref[ks[j]])),
                     "gamma values") if same.any() else dict(ratio=0.0)
    return dict(n=len(got), n_tie=n_tie, n_fail=n_fail, fails=fails[:10], **vc)


def gamma_condition(seed, stream, base, i, alpha, t):
    """3 |c z / (1 + c z)| at the accepting trial t of sample i (oracle values)."""
    d, c = oracle.mt_consts(alpha)
    ur, ut, U = oracle.mt_trial_uniforms(seed, stream, base, i, t)
    _, _, _, onepcz = oracle.mt_trial(d, c, ur, ut, U)
    return 3.0 * abs((onepcz - 1.0) / onepcz)


def dirichlet_compare(got, trials, alpha, seed, stream, base, row0=0, dtype=np.float32):
    """Rows row0.. of a Dirichlet call.  Rows containing a decision tie are
    excluded from the value comparison (and counted)."""
    dtype = np.dtype(dtype)
    got = _np(got); trials = _np(trials); alpha = np.asarray(alpha)
    ref, tref, _ = oracle.dirichlet(seed, stream, base, alpha, row0=row0, dtype=dtype)
    rows, k = alpha.shape
    n_tie = n_fail = 0
    tie_rows = np.zeros(rows, bool)
    for r, c in zip(*np.nonzero(trials != tref)):
        t_star = int(min(trials[r, c], tref[r, c]))
        i = (row0 + r) * k + c
        if t_star == 0:
            n_fail += 1; continue
        m, onepcz, d = oracle.gamma_tie_margin(seed, stream, base, int(i), float(alpha[r, c]),
                                               t_star)
        if (np.isfinite(m) and abs(m) <= TIE_BAND * max(1.0, d)) or abs(onepcz) <= TIE_BAND:
            n_tie += 1; tie_rows[r] = True
        else:
            n_fail += 1
    ok = ~tie_rows
    rr, cc = np.nonzero(np.broadcast_to(ok[:, None], got.shape))
    # x_k = g_k / S: the row sum is well conditioned; g_k carries its own
    # Marsaglia-Tsang conditioning (see gamma_compare)
    vc = value_check(got[ok].reshape(-1), ref[ok].reshape(-1),
                     np.abs(ref[ok].reshape(-1).astype(np.float64)), dtype,
                     lambda j: gamma_condition(seed, stream, base, (row0 + int(rr[j])) * k + int(cc[j]),
                                               float(alpha[rr[j], cc[j]]), int(tref[rr[j], cc[j]])),
                     "dirichlet")
    return dict(n=got.size, n_tie=n_tie, n_fail=n_fail, **vc)


def windows(n, n_windows=32, width=256, seed=0):
    """Sampled parity at full size: head, tail and random interior windows
    of contiguous indices [(lo, hi), ...]."""
    rng = np.random.default_rng(seed)
    w = [(0, min(width, n)), (max(0, n - width), n)]
    if n > 2 * width:
        for lo in rng.integers(width, n - 2 * width, n_windows):
            w.append((int(lo), int(lo) + width))
    return w
