"""Power of the oracle pins ("injected bug ... at least one check
fails"): plausible mistakes in the method, applied to the SAME draws the
oracle uses, must fail the closed-form / statistical pins that the correct
oracle passes.  Each mutant is written out here in numpy; none of this feeds
a parity expectation."""
import math

import numpy as np
from scipy import stats

import oracle
from tests.stats_util import mt_acceptance, pit_gamma, pit_uniform

KS = 1.63  # S:L89 1% critical constant


def _ks_fails(u):
    return stats.kstest(np.asarray(u, np.float64), "uniform").pvalue < 0.01


def test_uniform_transform_mutant_fails_pit():
    n = 1 << 16
    rng = np.random.default_rng(1)
    a = rng.uniform(-1, 0, n); b = a + np.exp(rng.uniform(math.log(1e-3), math.log(1e3), n))
    u = oracle.std_uniform(7, 0, 0, n, np.float64)
    good, _ = oracle.uniform(7, 0, 0, a, b)
    assert not _ks_fails(pit_uniform(good, a, b))
    mutant = a + b * u                                 # forgot the "- a"
    assert _ks_fails(pit_uniform(mutant, a, b))


def test_gamma_acceptance_mutants_break_closed_form():
    # the trial uniforms of the oracle, decisions by the correct test and by
    # two mutants: a dropped d*ln(v) term and a sign error on d*v
    alpha, n = 2.1, 1 << 14
    d, c = oracle.mt_consts(alpha)
    acc = np.zeros(3)
    for i in range(n):
        ur, ut, U = oracle.mt_trial_uniforms(13, 0, 0, i, 1)
        z = math.sqrt(-2 * math.log(1 - ur)) * oracle.cos2pi(ut)
        t = 1 + c * z
        if t <= 0:
            continue
        v = t ** 3
        lu = math.log(U)
        acc[0] += lu < z * z / 2 + d - d * v + d * math.log(v)
        acc[1] += lu < z * z / 2 + d - d * v                   # dropped d ln v
        acc[2] += lu < z * z / 2 + d + d * v + d * math.log(v)  # sign of d v
    P = mt_acceptance(alpha)
    band = 5 * math.sqrt(P * (1 - P) / n)
    assert abs(acc[0] / n - P) < band
    assert abs(acc[1] / n - P) > band and abs(acc[2] / n - P) > band


def test_gamma_boost_mutant_fails_pit():
    n = 1 << 15
    alpha = np.full(n, 0.3)
    g, tr, _ = oracle.gamma(17, 0, 0, alpha, np.ones(n))
    assert not _ks_fails(pit_gamma(g, alpha, 1.0))
    # mutant: boost with exponent alpha instead of 1/alpha (U^alpha)
    bu = np.array([oracle.u53(*[int(x) for x in oracle.block(17, 0, 256 * i)[:2]])
                   for i in range(n)])
    unboosted = g / np.exp(np.log1p(-bu) / alpha)
    mutant = unboosted * np.exp(np.log1p(-bu) * alpha)
    assert _ks_fails(pit_gamma(mutant, alpha, 1.0))


def test_gibbs_order_mutant_breaks_transient_means():
    # y updated before x (Fig. 1 draws x first) changes E[mean_x over 3 sweeps]
    n_chains, n = 1 << 16, 3
    w = oracle.raw_u32(5, 0, 0, 4 * n_chains * n).reshape(n_chains, n, 4).astype(np.uint64)
    u1 = ((w[..., 1] << 32 | w[..., 0]) >> 11).astype(np.float64) * 2.0**-53
    u2 = ((w[..., 3] << 32 | w[..., 2]) >> 11).astype(np.float64) * 2.0**-53
    x = np.full(n_chains, 0.5); y = np.full(n_chains, 0.5)
    sx = np.zeros(n_chains)
    for s in range(n):
        y = (1 - x) * u2[:, s]
        x = (1 - y) * u1[:, s]
        sx += x
    ex = 1 / 3 - (1 - 4.0**-n) / (9 * n)
    sd = math.sqrt(1 / 18 / n_chains)
    assert abs(sx.mean() / n - ex) > 5 * sd
    r = oracle.gibbs_triangle(5, 0, 0, 4096, n, want_samples=False)
    assert abs(r["chain_stats"][0].mean() - ex) < 5 * math.sqrt(1 / 18 / 4096)


def test_histogram_pin_detects_uniform_marginal():
    # a sampler of the unit square (forgetting the triangle constraint) has
    # flat bins, not p_b = (511 - 2b)/65536
    rng = np.random.default_rng(9)
    x = rng.random(1 << 20)
    hist = np.bincount((x * 256).astype(int), minlength=256)
    p = (511 - 2 * np.arange(256)) / 65536.0
    chi2 = np.sum((hist - hist.sum() * p) ** 2 / (hist.sum() * p))
    assert stats.chi2.sf(chi2, 255) < 1e-6
