"""Pins for the oracle's NEXT-row N2 functions: log-uniform,
Laplace and Weibull (algorithms; R-30).

- SPEC worked examples S:L81 (ln identity), S:L237-238 (Laplace sign rule),
  S:L246-247 (Weibull(1) = exponential; 4^(1/2) = 2);
- log-uniform = -exponential at the same positions;
- Laplace variance 2 beta^2 and KS vs the Laplace CDF; Weibull KS vs
  1 - exp(-(x/beta)^alpha), varying parameters by PIT.
"""
import math

import numpy as np

import oracle
from tests.stats_util import assert_ks_uniform, mean_band


def test_log_uniform_is_negated_exponential():
    for dt in (np.float32, np.float64):
        lu = oracle.log_uniform(5, 1, 9, 1000, dtype=dt)
        e, _ = oracle.exponential(5, 1, 9, np.ones(1000, dt))
        assert np.array_equal(lu, -e) and np.all(lu <= 0)
    assert math.log(1.0 - (1.0 - math.exp(-1.0))) == -1.0 or \
        abs(math.log(math.exp(-1.0)) + 1.0) < 1e-16


def test_laplace_sign_rule_and_pairing():
    # e = 1, u = 0.7 -> +2; u = 0.3 -> -2 with (a, beta) = (0, 2):
    # check the rule on the oracle's own draws: x / beta = +-e, sign from u_b
    n = 64
    x, bad = oracle.laplace(3, 2, 11, np.zeros(n), np.full(n, 2.0))
    assert bad == 0
    for i in range(n):
        w = oracle.block(3, 2, 11 + i)
        e = -math.log(1 - oracle.u53(int(w[0]), int(w[1])))
        s = -1.0 if oracle.u53(int(w[2]), int(w[3])) < 0.5 else 1.0
        assert x[i] == 2.0 * s * e
    x32, _ = oracle.laplace(3, 2, 11, np.zeros(n, np.float32), np.ones(n, np.float32))
    for i in range(n):
        w = oracle.block(3, 2, 11 + i // 2)
        j = i % 2
        e = -math.log(1 - oracle.u24(int(w[2 * j])))
        s = -1.0 if oracle.u24(int(w[2 * j + 1])) < 0.5 else 1.0
        assert x32[i] == np.float32(s * e)


def test_laplace_moments_and_ks():
    n = 1 << 18
    x, _ = oracle.laplace(7, 0, 0, np.zeros(n), np.ones(n))
    ok, v = mean_band(x * x, 2.0, 24.0 - 4.0); assert ok, v               # E x^4 = 24
    ok, m = mean_band(x, 0.0, 2.0); assert ok, m
    rng = np.random.default_rng(1)
    mu = rng.uniform(-10, 10, n); b = np.exp(rng.uniform(math.log(1e-3), math.log(1e3), n))
    y, bad = oracle.laplace(7, 0, 1 << 20, mu, b)
    assert bad == 0
    z = (y - mu) / b
    pit = np.where(z < 0, 0.5 * np.exp(z), 1 - 0.5 * np.exp(-z))
    assert_ks_uniform(pit, "Laplace PIT")


def test_weibull_examples_moments_ks():
    n = 4096
    w1, _ = oracle.weibull(9, 0, 5, np.ones(n), np.full(n, 3.0))
    e, _ = oracle.exponential(9, 0, 5, np.full(n, 1.0 / 3.0))
    np.testing.assert_allclose(w1, e, rtol=1e-15)
    assert 1.0 * 4.0 ** (1 / 2) == 2.0
    n = 1 << 18
    rng = np.random.default_rng(2)
    a = np.exp(rng.uniform(math.log(0.5), math.log(5), n))
    b = np.exp(rng.uniform(math.log(0.1), math.log(10), n))
    x, bad = oracle.weibull(9, 0, 0, a, b)
    assert bad == 0 and np.all(x >= 0)
    assert_ks_uniform(-np.expm1(-(x / b) ** a), "Weibull PIT")
    x2, _ = oracle.weibull(10, 0, 0, np.full(n, 2.0), np.ones(n))
    ok, m = mean_band(x2, math.gamma(1.5), 1 - math.gamma(1.5) ** 2); assert ok, m


def test_invalid_next_parameters():
    x, bad = oracle.laplace(1, 0, 0, np.array([0.0, np.nan, 0.0]), np.array([1.0, 1.0, 0.0]))
    assert bad == 2 and not np.isnan(x[0]) and np.isnan(x[1:]).all()
    x, bad = oracle.weibull(1, 0, 0, np.array([1.0, 0.0, 1.0]), np.array([1.0, 1.0, -1.0]))
    assert bad == 2 and not np.isnan(x[0]) and np.isnan(x[1:]).all()
