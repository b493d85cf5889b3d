"""Pins for the oracle's Gibbs sampler on the triangle (R-14..R-19).

- support X >= 0, Y >= 0, X + Y <= 1 exactly (Eq. 1);
- TRANSIENT-EXACT means from (0.5, 0.5): E[mean_x over n sweeps] =
  1/3 - (1 - 4^-n)/(9n), E[mean_y] = 1/3 + (1 - 4^-n)/(18n) (derived in
  DESIGN.md; a dropped (1-y) or swapped update order fails it);
- stationary Var 1/18, Cov -1/36;
- histogram bin probabilities p_b = (511 - 2b)/65536 of the marginal 2(1-x);
- brute-force rejection sampling of the triangle, two-sample KS;
- chunk invariance (R-12) and the cfg1 output count (BASELINE configs[0]).
"""
import math
from fractions import Fraction

import numpy as np
from scipy import stats

import oracle


def test_support_exact():
    r = oracle.gibbs_triangle(42, 0, 0, 64, 500)
    x, y = r["out_x"], r["out_y"]
    assert np.all(x >= 0) and np.all(y >= 0) and np.all(x + y < 1)
    for xi, yi in zip(x.reshape(-1)[::97], y.reshape(-1)[::97]):
        assert Fraction(float(xi)) + Fraction(float(yi)) < 1


def test_golden_cfg1_shape(golden):
    r = oracle.gibbs_triangle(42, 0, 0, 1024, 1000)
    assert r["out_x"].size + r["out_y"].size == golden["gibbs_triangle"]["cfg1_output_doubles"]
    assert r["n_invalid"] == 0


def test_transient_exact_means():
    n_chains, n = 1 << 18, 3
    r = oracle.gibbs_triangle(7, 0, 0, n_chains, n, want_samples=False)
    st = r["chain_stats"]
    ex = 1 / 3 - (1 - 4.0**-n) / (9 * n)
    ey = 1 / 3 + (1 - 4.0**-n) / (18 * n)
    # per-chain mean over 3 sweeps has variance <= Var(X) = 1/18
    sd = math.sqrt(1 / 18 / n_chains)
    assert abs(st[0].mean() - ex) < 5 * sd, (st[0].mean(), ex)
    assert abs(st[2].mean() - ey) < 5 * sd, (st[2].mean(), ey)
    # first sweep exactly: x1 = 0.5 u ~ U(0, 0.5): E = 1/4
    r1 = oracle.gibbs_triangle(8, 0, 0, n_chains, 1)
    assert abs(r1["out_x"].mean() - 0.25) < 5 * math.sqrt(1 / 48 / n_chains)
    assert abs(r1["out_y"].mean() - 0.375) < 5 * math.sqrt(0.07 / n_chains)


def test_stationary_moments(golden):
    g = golden["gibbs_triangle"]
    r = oracle.gibbs_triangle(42, 0, 0, 1024, 1000, burn_in=32)
    x = r["out_x"][32:].reshape(-1); y = r["out_y"][32:].reshape(-1)
    assert abs(x.mean() - g["mean"]) < 0.002 and abs(y.mean() - g["mean"]) < 0.002
    assert abs(x.var() - g["var"]) < 0.001 and abs(y.var() - g["var"]) < 0.001
    assert abs(np.mean((x - x.mean()) * (y - y.mean())) - g["cov"]) < 0.001
    st = r["chain_stats"]
    assert abs(st[1].mean() - g["var"]) < 0.002 and abs(st[4].mean() - g["cov"]) < 0.002


def test_histogram_chi2_closed_form():
    n_chains, n_sweeps, burn = 4096, 288, 32
    r = oracle.gibbs_triangle(3, 0, 0, n_chains, n_sweeps, burn_in=burn, want_samples=False)
    hist = r["totals"][oracle.TOTALS_HDR:]
    N = n_chains * (n_sweeps - burn)
    assert hist.sum() == N and np.all(hist == np.round(hist))
    p = (511 - 2 * np.arange(256)) / 65536.0
    assert abs(p.sum() - 1) < 1e-15
    # consecutive sweeps are correlated (rho = 1/4 per lag): thin by using a
    # variance-inflated chi^2 -- chi2 / (5/3) ~ chi2_255 approximately
    chi2 = np.sum((hist - N * p) ** 2 / (N * p)) / (5.0 / 3.0)
    assert stats.chi2.sf(chi2, 255) > 1e-3, chi2


def test_rejection_sampling_brute_force():
    # triangle points by brute-force rejection from the unit square
    rng = np.random.default_rng(503)
    pts = rng.random((400_000, 2))
    ref_x = pts[pts.sum(axis=1) < 1][:, 0]
    r = oracle.gibbs_triangle(42, 0, 0, 1024, 1000)
    gx = r["out_x"][32::8].reshape(-1)          # thinned, after burn-in
    p = stats.ks_2samp(gx, ref_x).pvalue
    assert p > 0.01, p


def test_chunk_invariance_and_totals():
    n_chains = 50
    a = oracle.gibbs_triangle(9, 100, 0, n_chains, 1000)
    b1 = oracle.gibbs_triangle(9, 100, 0, n_chains, 500)
    f = b1["final_xy"]
    b2 = oracle.gibbs_triangle(9, 100, 500, n_chains, 500, x0=f[0], y0=f[1])
    assert np.array_equal(a["out_x"], np.concatenate([b1["out_x"], b2["out_x"]]))
    assert np.array_equal(a["final_xy"], b2["final_xy"])
    # chain c uses stream stream_id + c
    c7 = oracle.gibbs_triangle(9, 107, 0, 1, 1000)
    assert np.array_equal(c7["out_x"][:, 0], a["out_x"][:, 7])
    t = a["totals"]; st = a["chain_stats"]
    assert t[8] == n_chains and t[9] == n_chains * 1000
    np.testing.assert_allclose(t[[0, 1, 3, 4, 6]], st[[0, 1, 2, 3, 4]].sum(axis=1), rtol=1e-13)
    assert t[oracle.TOTALS_HDR:].sum() == n_chains * 1000


def test_invalid_start():
    r = oracle.gibbs_triangle(1, 0, 0, 3, 10, y0=np.array([0.5, 1.5, np.nan]))
    assert r["n_invalid"] == 2
    assert not np.isnan(r["final_xy"][0, 0]) and np.all(np.isnan(r["final_xy"][:, 1:]))
