"""Pins for the oracle's Marsaglia-Tsang Gamma and alpha<1 boost (R-08..R-11).

- S:L257 forced acceptance at z = 0 (g = d = alpha - 1/3);
- the CLOSED-FORM acceptance probability of the (squeeze-free) test,
  P(a') = e^d Gamma(a') sqrt(d) / (sqrt(2 pi) d^a'),
  against the trial counts: a dropped/mis-signed term in the test moves it;
- Gamma(1,1) == Exp(1) by KS;
- PIT via the regularised incomplete gamma for varying (alpha, beta),
  including the boosted alpha < 1 branch; mean alpha*beta, var alpha*beta^2.
"""
import math

import numpy as np
import pytest

import oracle
from tests.stats_util import (assert_ks_uniform, mean_band, mt_acceptance, pit_exponential,
                              pit_gamma)


def test_golden_z0_forced_acceptance(golden):
    for alpha in golden["gamma_z0"]["alpha"]:
        d, c = oracle.mt_consts(alpha)
        assert d == alpha - 1.0 / 3.0 and c == 1.0 / math.sqrt(9.0 * d)
        for U in (1e-300, 0.5, 1.0 - 2**-32):
            acc, g, margin, t = oracle.mt_trial(d, c, 0.0, 0.123, U)   # u_r = 0 -> z = 0
            assert acc and g == d and t == 1.0
            assert margin == pytest.approx(-math.log(U), abs=1e-15)
        acc, _, margin, _ = oracle.mt_trial(d, c, 0.0, 0.123, 1.0)     # ln 1 = 0 is not < 0
        assert not acc and margin == 0.0


def test_negative_one_plus_cz_rejects():
    d, c = oracle.mt_consts(1.0)
    # z = -r with r large: u_theta = 1/2 gives cos = -1; 1 - u_r tiny -> r ~ 8.5
    acc, g, margin, t = oracle.mt_trial(d, c, 1 - 2**-53, 0.5, 0.5)
    assert t < 0 and not acc and math.isnan(margin)


def test_trial_uniform_counter_map():
    for i, t in ((0, 1), (7, 1), (7, 255), (123456, 3)):
        ur, ut, U = oracle.mt_trial_uniforms(9, 2, 1000, i, t)
        w = oracle.block(9, 2, 1000 + 256 * i + t)
        assert ur == oracle.u53(int(w[0]), int(w[1]))
        assert ut == oracle.u32d(int(w[2]))
        assert U == 1.0 - oracle.u32d(int(w[3]))


@pytest.mark.parametrize("alpha", [1.0, 2.1, 10.0, 0.3, 200.0])
def test_acceptance_rate_closed_form(alpha):
    n = 1 << 16
    _, trials, bad = oracle.gamma(31, 0, 0, np.full(n, alpha), np.ones(n))
    assert bad == 0 and trials.min() >= 1
    P = mt_acceptance(alpha + 1.0 if alpha < 1 else alpha)
    first = float(np.mean(trials == 1))
    assert abs(first - P) <= 5 * math.sqrt(P * (1 - P) / n), (first, P)
    mt = float(np.mean(trials))
    assert abs(mt - 1 / P) <= 5 * math.sqrt((1 - P) / P**2 / n), (mt, 1 / P)


def test_acceptance_closed_form_values():
    # the closed form itself against the simulated values quoted in SURVEY 8c.4
    assert mt_acceptance(1.0) == pytest.approx(0.9515, abs=5e-4)
    assert mt_acceptance(2.1) == pytest.approx(0.9827, abs=5e-4)
    assert mt_acceptance(10.0) == pytest.approx(0.9970, abs=5e-4)


def test_gamma1_is_exponential():
    n = 1 << 17
    x, _, bad = oracle.gamma(41, 0, 0, np.ones(n), np.ones(n))
    assert bad == 0
    assert_ks_uniform(pit_exponential(x, 1.0), "Gamma(1) vs Exp(1)")


def test_pit_varying_alpha_beta():
    n = 1 << 17
    rng = np.random.default_rng(11)
    alpha = np.exp(rng.uniform(np.log(0.05), np.log(200), n))
    beta = np.exp(rng.uniform(np.log(0.1), np.log(10), n))
    x, tr, bad = oracle.gamma(11, 0, 0, alpha, beta)
    assert bad == 0 and np.all(x > 0) and np.all(tr >= 1)
    assert_ks_uniform(pit_gamma(x, alpha, beta), "gamma PIT")
    # boosted and unboosted halves separately
    lo = alpha < 1
    assert_ks_uniform(pit_gamma(x[lo], alpha[lo], beta[lo]), "gamma PIT alpha<1")
    assert_ks_uniform(pit_gamma(x[~lo], alpha[~lo], beta[~lo]), "gamma PIT alpha>=1")


def test_golden_moments(golden):
    n = 1 << 17
    for k, (alpha, beta) in enumerate(golden["gamma_moments"]["cases"]):
        x, _, _ = oracle.gamma(100 + k, 0, 0, np.full(n, alpha), np.full(n, beta))
        ok, m = mean_band(x, alpha * beta, alpha * beta * beta)
        assert ok, (alpha, beta, m)
        # variance: E[(x - ab)^2] = a b^2 with Var((x-m)^2) = b^4 (mu4 - a^2),
        # mu4 = 3a^2 + 6a for Gamma(a,1)
        ok, v = mean_band((x - alpha * beta) ** 2, alpha * beta**2,
                          beta**4 * (3 * alpha**2 + 6 * alpha - alpha**2))
        assert ok, (alpha, beta, v)


def test_boost_uses_block_zero():
    alpha = 0.4
    g_all, t, bad = oracle.gamma_one(3, 0, 0, 17, alpha, 1.0)
    assert not bad and t >= 1
    d, c = oracle.mt_consts(alpha)
    ur, ut, U = oracle.mt_trial_uniforms(3, 0, 0, 17, t)
    _, g, _, _ = oracle.mt_trial(d, c, ur, ut, U)
    w = oracle.block(3, 0, 256 * 17)
    u = oracle.u53(int(w[0]), int(w[1]))
    assert g_all == g * math.exp(math.log(1 - u) / alpha)


def test_invalid_and_offsets():
    a = np.array([1.0, 0.0, -1.0, np.nan, 2.0, 1.0])
    b = np.array([1.0, 1.0, 1.0, 1.0, 0.0, np.inf])
    x, tr, bad = oracle.gamma(1, 0, 0, a, b)
    assert bad == 5 and x[0] > 0 and np.all(np.isnan(x[1:])) and np.all(tr[1:] == 0)
    alpha = np.linspace(0.1, 20, 100); beta = np.ones(100)
    whole, tw, _ = oracle.gamma(2, 0, 0, alpha, beta)
    part, tp, _ = oracle.gamma(2, 0, 0, alpha[37:], beta[37:], i0=37)
    assert np.array_equal(whole[37:], part) and np.array_equal(tw[37:], tp)
    # next call at cursor + 256 * n continues (R-12)
    tail, _, _ = oracle.gamma(2, 0, 256 * 37, alpha[37:], beta[37:])
    assert np.array_equal(tail, part)
    f32, t32, _ = oracle.gamma(2, 0, 0, alpha.astype(np.float32), beta.astype(np.float32))
    ref, tr32, _ = oracle.gamma(2, 0, 0, alpha.astype(np.float32).astype(np.float64), beta)
    assert np.array_equal(f32, ref.astype(np.float32)) and np.array_equal(t32, tr32)
