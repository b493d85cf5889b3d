"""Pins for the oracle's reducible distributions (R-06, R-07).

- SPEC worked examples (tests/golden/spec_examples.json, each cited);
- exact special values of the dyadic-reduced cos/sin(2 pi u);
- closed forms near the zeros of cos/sin (relative accuracy);
- PIT Kolmogorov-Smirnov with varying per-sample parameters and moments.
"""
import math

import numpy as np
import pytest

import oracle
from tests.stats_util import (assert_ks_uniform, mean_band, pit_exponential, pit_normal,
                              pit_uniform)


def test_golden_box_muller(golden):
    g = golden["box_muller"]
    u_r = 1.0 - math.exp(-2.0)
    assert oracle.box_muller(u_r, g["u_theta"], False) == pytest.approx(g["z_cos"], rel=1e-14)
    assert oracle.box_muller(u_r, g["u_theta"], True) == g["z_sin"]
    q = golden["box_muller_quarter_turn"]
    assert oracle.cos2pi(q["u_theta"]) == q["cos"]
    assert oracle.sin2pi(q["u_theta"]) == q["sin"]


def test_trig_special_values():
    for u, c, s in [(0.0, 1.0, 0.0), (0.25, 0.0, 1.0), (0.5, -1.0, 0.0), (0.75, 0.0, -1.0)]:
        assert oracle.cos2pi(u) == c and oracle.sin2pi(u) == s
    r2 = math.sqrt(0.5)
    for u in (0.125, 0.375, 0.625, 0.875):
        assert abs(abs(oracle.cos2pi(u)) - r2) < 2e-16
        assert abs(abs(oracle.sin2pi(u)) - r2) < 2e-16


def test_trig_relative_accuracy_near_zeros():
    # cos(2 pi (1/4 + d)) = -sin(2 pi d) ~ -2 pi d (1 - (2 pi d)^2 / 6): the
    # value must be RELATIVELY accurate for tiny dyadic d (a naive cos(2*pi*u)
    # has absolute error ~1e-16 there, i.e. relative error ~1 at d = 2^-50).
    for k in (20, 30, 40, 50, 52):
        d = 2.0 ** -k
        for base, sgn_c, sgn_s in ((0.25, -1, None), (0.75, +1, None), (0.5, None, -1),
                                   (0.0, None, +1)):
            x = 2 * math.pi * d
            series = x - x ** 3 / 6
            if sgn_c is not None:
                assert oracle.cos2pi(base + d) == pytest.approx(sgn_c * series, rel=4e-16)
            else:
                assert oracle.sin2pi(base + d) == pytest.approx(sgn_s * series, rel=4e-16)


def test_trig_pythagoras_and_quadrants():
    rng = np.random.default_rng(3)
    for u in rng.integers(0, 2**53, 2000) * 2.0**-53:
        c, s = oracle.cos2pi(u), oracle.sin2pi(u)
        assert abs(c * c + s * s - 1) < 1e-15
        # against libm far from the zeros, where the naive form is accurate
        if min(abs(u - q) for q in (0, .25, .5, .75, 1)) > 1e-3:
            assert c == pytest.approx(math.cos(2 * math.pi * u), rel=1e-12)
            assert s == pytest.approx(math.sin(2 * math.pi * u), rel=1e-12)


def test_golden_exponential_loguniform(golden):
    # exponential with lambda = 1 is -ln(1-u); check the SPEC pairs through
    # the transform on a one-sample array whose standard uniform is known.
    for expr, val in golden["exponential"]["cases"]:
        u = 1 - math.exp(-2.0) if expr != "0" else 0.0
        assert -math.log(1.0 - u) == pytest.approx(val, abs=1e-15)
    # and the oracle's exponential equals -ln(1-u)/lambda at its own positions
    lam = np.array([1.0, 2.0, 0.5, 1e3, 1e-3])
    out, bad = oracle.exponential(11, 0, 0, lam)
    u = oracle.std_uniform(11, 0, 0, 5, np.float64)
    assert bad == 0
    np.testing.assert_allclose(out, -np.log1p(-u) / lam, rtol=1e-15)


def test_golden_uniform_identity(golden):
    g = golden["uniform"]
    n = 64
    a = np.full(n, g["a"]); b = np.full(n, g["b"])
    out, _ = oracle.uniform(5, 1, 3, a, b)
    u = oracle.std_uniform(5, 1, 3, n, np.float64)
    assert np.array_equal(out, 2.0 * u)                     # a + (b-a) u, exact
    out01, _ = oracle.uniform(5, 1, 3, np.zeros(n), np.ones(n))
    assert np.array_equal(out01, u)                          # identity case
    assert g["a"] + (g["b"] - g["a"]) * g["u"] == g["x"]


def test_golden_gaussian(golden):
    g = golden["gaussian"]
    n = 40
    out, _ = oracle.gaussian(8, 0, 0, np.full(n, g["sigma0"]["mu"]), np.zeros(n))
    assert np.all(out == g["sigma0"]["x"])
    z, _ = oracle.gaussian(8, 0, 0, np.zeros(n), np.ones(n))
    x, _ = oracle.gaussian(8, 0, 0, np.full(n, 1.0), np.full(n, 3.0))
    np.testing.assert_allclose(x, 1.0 + 3.0 * z, rtol=1e-15, atol=1e-15)
    a = g["affine"]
    assert a["mu"] + a["sigma"] * a["z"] == a["x"]


def test_gaussian_pairing_f64_f32():
    # f64: sample 2j -> r cos, 2j+1 -> r sin of block j; f32: two pairs/block.
    n = 8
    z64, _ = oracle.gaussian(3, 4, 5, np.zeros(n), np.ones(n), dtype=np.float64)
    for i in range(n):
        w = oracle.block(3, 4, 5 + i // 2)
        ur, ut = oracle.u53(int(w[0]), int(w[1])), oracle.u53(int(w[2]), int(w[3]))
        assert z64[i] == oracle.box_muller(ur, ut, i % 2 == 1)
    z32, _ = oracle.gaussian(3, 4, 5, np.zeros(n, np.float32), np.ones(n, np.float32))
    for i in range(n):
        w = oracle.block(3, 4, 5 + i // 4)
        p = (i % 4) // 2
        ref = oracle.box_muller(oracle.u24(int(w[2 * p])), oracle.u24(int(w[2 * p + 1])),
                                i % 2 == 1)
        assert z32[i] == np.float32(ref)
    # cos/sin partners share r: z_cos^2 + z_sin^2 = r^2 = -2 ln(1-u_r)
    w = oracle.block(3, 4, 5)
    r2 = -2 * math.log(1 - oracle.u53(int(w[0]), int(w[1])))
    assert z64[0] ** 2 + z64[1] ** 2 == pytest.approx(r2, rel=1e-14)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_pit_ks_varying_parameters(dtype):
    n = 1 << 17
    rng = np.random.default_rng(20141216)
    mu = rng.uniform(-10, 10, n).astype(dtype)
    sigma = np.exp(rng.uniform(np.log(1e-3), np.log(1e3), n)).astype(dtype)
    x, bad = oracle.gaussian(7, 0, 0, mu, sigma)
    assert bad == 0
    assert_ks_uniform(pit_normal(x, mu.astype(np.float64), sigma.astype(np.float64)), "gauss")
    a = rng.uniform(-1, 0, n).astype(dtype)
    b = (a.astype(np.float64) + np.exp(rng.uniform(np.log(1e-3), np.log(1e3), n))).astype(dtype)
    x, bad = oracle.uniform(7, 0, 1 << 20, a, b)
    assert bad == 0
    assert np.all(x >= a) and np.all(x <= b)
    assert_ks_uniform(pit_uniform(x, a, b), "uniform")
    lam = np.exp(rng.uniform(np.log(1e-3), np.log(1e3), n)).astype(dtype)
    x, bad = oracle.exponential(7, 0, 1 << 21, lam)
    assert bad == 0 and np.all(x >= 0)
    assert_ks_uniform(pit_exponential(x, lam), "exponential")


def test_moments_fixed_parameters():
    n = 1 << 18
    z, _ = oracle.gaussian(21, 0, 0, np.full(n, -1.0), np.full(n, 2.0))
    ok, m = mean_band(z, -1.0, 4.0); assert ok, m
    ok, v = mean_band((z + 1.0) ** 2, 4.0, 32.0); assert ok, v       # Var = 4, Var(z^2)=2 s^4
    u, _ = oracle.uniform(21, 1, 0, np.full(n, 2.0), np.full(n, 4.0))
    ok, m = mean_band(u, 3.0, 1.0 / 3.0); assert ok, m
    e, _ = oracle.exponential(21, 2, 0, np.full(n, 1.0 / 3.0))
    ok, m = mean_band(e, 3.0, 9.0); assert ok, m


def test_invalid_parameters_nan_and_counted():
    a = np.array([0.0, 1.0, np.nan, 0.0, -np.inf])
    b = np.array([1.0, 1.0, 1.0, np.inf, 0.0])
    x, bad = oracle.uniform(1, 0, 0, a, b)
    assert bad == 4 and not np.isnan(x[0]) and np.all(np.isnan(x[1:]))
    x, bad = oracle.gaussian(1, 0, 0, np.array([0.0, 0.0, np.nan]), np.array([-1.0, 0.0, 1.0]))
    assert bad == 2 and np.isnan(x[0]) and x[1] == 0.0 and np.isnan(x[2])
    x, bad = oracle.exponential(1, 0, 0, np.array([0.0, -1.0, 1.0, np.inf]))
    assert bad == 3 and np.isnan(x[0]) and np.isnan(x[1]) and x[2] >= 0 and np.isnan(x[3])


def test_chunk_invariance_and_offsets():
    n = 1000
    mu = np.zeros(n); sg = np.ones(n)
    whole, _ = oracle.gaussian(4, 0, 10, mu, sg)
    # samples i0.. of the same call (sampled parity uses this)
    part, _ = oracle.gaussian(4, 0, 10, mu[300:], sg[300:], i0=300)
    assert np.array_equal(whole[300:], part)
    # a second call at cursor + ceil(300/2) continues the stream (f64: 2/block)
    head, _ = oracle.gaussian(4, 0, 10, mu[:300], sg[:300])
    tail, _ = oracle.gaussian(4, 0, 10 + 150, mu[300:], sg[300:])
    assert np.array_equal(np.concatenate([head, tail]), whole)
