"""Pins for the oracle's between-chain moment totals of the Gibbs sampler
(totals[2] = sum_c mean_x^2, totals[5] = sum_c mean_y^2, totals[7] =
sum_c mean_x mean_y; R-18, BASELINE configs[4] "NCCL reduce of
per-chain mean/variance"), against EXACT expectations derived from the law of
the chain itself (Fig. 1: x ~ U(0, 1-y), then y ~ U(0, 1-x), from
(0.5, 0.5)) -- not from the oracle's code.

Derivation (all exact rationals).  One sweep, from y = y_{s-1}:
  E[x_s] = (1 - E y)/2,  E[x_s^2] = E[(1-y)^2]/3,
  E[y_s] = (1 - E x_s)/2, E[y_s^2] = E[(1-x_s)^2]/3, E[x_s y_s] = E[x_s(1-x_s)]/2.
Given the state after sweep s, only y_s matters for the future, and the
conditional means are affine in y_s:
  E[y_{s+k} | y_s] = 1/3 + (y_s - 1/3) 4^-k,
  E[x_{s+k} | y_s] = 1/3 - (y_s - 1/3) / (2 4^(k-1))      (k >= 1),
so every cross moment E[x_s x_t], E[y_s y_t], E[x_s y_t], E[y_s x_t] follows
from the one-sweep moments at the earlier sweep.  The means over the sweeps
s >= burn_in are then E[mean_x^2] = m^-2 sum_{s,t} E[x_s x_t], etc.

A plausible slip in the oracle (totals[7] += mx*mx, a swapped accumulator, a
missing square) moves a total by tens of standard errors: the mutant cases
below check that the pin catches each of them.
"""
import math
from fractions import Fraction as F

import numpy as np
import pytest

import oracle


def exact_moments(n_sweeps, burn_in, exact=True):
    """E[mean_x^2], E[mean_y^2], E[mean_x mean_y], E[mean_x], E[mean_y] over
    sweeps burn_in .. n_sweeps-1 (0-based, as the oracle counts them).
    exact=False evaluates the same sums in binary64 (large n)."""
    one = F(1) if exact else 1.0
    ey, ey2 = one / 2, one / 4                     # y_0 = 0.5 (deterministic)
    mom = []                                       # per sweep: Ex, Ey, Ex2, Ey2, Exy
    for _ in range(n_sweeps):
        ex = (1 - ey) / 2
        ex2 = (1 - 2 * ey + ey2) / 3
        ey_n = (1 - ex) / 2
        ey2_n = (1 - 2 * ex + ex2) / 3
        exy = (ex - ex2) / 2
        mom.append((ex, ey_n, ex2, ey2_n, exy))
        ey, ey2 = ey_n, ey2_n
    S = range(burn_in, n_sweeps)
    m = len(S)
    third = one / 3
    sxx = syy = sxy = 0 * one
    for s in S:
        ex, ey, ex2, ey2, exy = mom[s]
        sxx += ex2
        syy += ey2
        sxy += exy
        # the K later sweeps t = s + k, k = 1..K: sum_k 4^-k = (1 - 4^-K)/3 and
        # sum_k 1/(2 4^(k-1)) = 2 (1 - 4^-K)/3
        K = n_sweeps - 1 - s
        g1 = (1 - (one / 4) ** K) / 3
        sxx += 2 * (K * ex * third - (exy - ex * third) * 2 * g1)      # E[x_s x_t]
        syy += 2 * (K * ey * third + (ey2 - ey * third) * g1)          # E[y_s y_t]
        sxy += K * ex * third + (exy - ex * third) * g1                # E[x_s y_t]
        sxy += K * ey * third - (ey2 - ey * third) * 2 * g1            # E[y_s x_t]
    mx = sum(mom[s][0] for s in S) / m
    my = sum(mom[s][1] for s in S) / m
    return dict(mx2=sxx / m**2, my2=syy / m**2, mxmy=sxy / m**2, mx=mx, my=my)


def exact_moments_pairwise(n_sweeps, burn_in):
    """The same expectations by the explicit double sum over sweep pairs
    (cross-checks the geometric-series closed form above)."""
    ey, ey2 = F(1, 2), F(1, 4)
    mom = []
    for _ in range(n_sweeps):
        ex = (1 - ey) / 2
        ex2 = (1 - 2 * ey + ey2) / 3
        ey_n = (1 - ex) / 2
        ey2_n = (1 - 2 * ex + ex2) / 3
        mom.append((ex, ey_n, ex2, ey2_n, (ex - ex2) / 2))
        ey, ey2 = ey_n, ey2_n
    S = range(burn_in, n_sweeps)
    third = F(1, 3)
    sxx = syy = sxy = F(0)
    for s in S:
        ex, ey, ex2, ey2, exy = mom[s]
        sxx += ex2; syy += ey2; sxy += exy
        for t in S:
            if t <= s:
                continue
            k = t - s
            sxx += 2 * (ex * third - (exy - ex * third) / (2 * F(4) ** (k - 1)))
            syy += 2 * (ey * third + (ey2 - ey * third) / F(4) ** k)
            sxy += ex * third + (exy - ex * third) / F(4) ** k
            sxy += ey * third - (ey2 - ey * third) / (2 * F(4) ** (k - 1))
    m = len(S)
    return dict(mx2=sxx / m**2, my2=syy / m**2, mxmy=sxy / m**2)


def pin_failures(totals, chain_stats, n_sweeps, burn_in, n_sd=5.0):
    """Names of the totals that miss their exact expectation by > n_sd
    standard errors (SE from the per-chain values themselves)."""
    e = exact_moments(n_sweeps, burn_in, exact=n_sweeps <= 256)
    C = chain_stats.shape[1]
    mx, my = chain_stats[0], chain_stats[2]
    bad = []
    for name, idx, per_chain in (("mean_x^2", 2, mx * mx), ("mean_y^2", 5, my * my),
                                 ("mean_x*mean_y", 7, mx * my), ("mean_x", 0, mx),
                                 ("mean_y", 3, my)):
        want = float(e[{0: "mx", 3: "my", 2: "mx2", 5: "my2", 7: "mxmy"}[idx]])
        se = per_chain.std() / math.sqrt(C)
        if abs(totals[idx] / C - want) > n_sd * se:
            bad.append(name)
    return bad


def test_closed_form_matches_pairwise_sum():
    for n, b in ((1, 0), (2, 0), (5, 1), (17, 4)):
        a, p = exact_moments(n, b), exact_moments_pairwise(n, b)
        assert (a["mx2"], a["my2"], a["mxmy"]) == (p["mx2"], p["my2"], p["mxmy"])
    f, e = exact_moments(40, 5, exact=False), exact_moments(40, 5)
    for k in ("mx2", "my2", "mxmy"):
        assert abs(f[k] - float(e[k])) < 1e-15


def test_closed_form_limits():
    # transient-exact first moments (independently derived)
    for n in (1, 3, 10):
        e = exact_moments(n, 0)
        assert e["mx"] == F(1, 3) - (1 - F(4) ** -n) / (9 * n)
        assert e["my"] == F(1, 3) + (1 - F(4) ** -n) / (18 * n)
    # one sweep: x_1 ~ U(0, 1/2): E x^2 = 1/12; y_1 = (1-x)V: E y^2 = E(1-x)^2/3
    e1 = exact_moments(1, 0)
    assert e1["mx2"] == F(1, 12)
    assert e1["my2"] == (1 - 2 * F(1, 4) + F(1, 12)) / 3
    # stationary limit: Var(mean over m) * m -> (1/18)(1 + 2 sum_k 4^-k) = (5/3)(1/18)
    m, b = 200, 60
    e = exact_moments(b + m, b)
    var_m = float(e["mx2"] - e["mx"] ** 2) * m
    assert abs(var_m - (5 / 3) / 18) < 0.01 * (5 / 3) / 18 + 2.0 / m


@pytest.mark.parametrize("n_sweeps,burn_in,n_chains", [(4, 0, 1 << 17), (24, 6, 1 << 15)])
def test_between_chain_totals(n_sweeps, burn_in, n_chains):
    r = oracle.gibbs_triangle(1234, 0, 0, n_chains, n_sweeps, burn_in=burn_in,
                              want_samples=False)
    t, st = r["totals"], r["chain_stats"]
    assert pin_failures(t, st, n_sweeps, burn_in) == []
    assert t[8] == n_chains and t[9] == n_chains * (n_sweeps - burn_in)


def test_mutants_are_caught():
    n_sweeps, burn_in, C = 4, 0, 1 << 17
    r = oracle.gibbs_triangle(1234, 0, 0, C, n_sweeps, burn_in=burn_in, want_samples=False)
    t, st = r["totals"], r["chain_stats"]
    mx, my = st[0], st[2]
    mutants = {
        "totals[7] += mx*mx": (7, (mx * mx).sum()),
        "totals[7] += my*my": (7, (my * my).sum()),
        "totals[5] += mx*my": (5, (mx * my).sum()),
        "totals[2] += mx (no square)": (2, mx.sum()),
        "totals[2] += my*my": (2, (my * my).sum()),
        "totals[0] += my": (0, my.sum()),
    }
    for name, (idx, val) in mutants.items():
        tm = t.copy()
        tm[idx] = val
        assert pin_failures(tm, st, n_sweeps, burn_in) != [], name


def test_derivation_vs_independent_simulation():
    """The closed forms themselves against a numpy simulation of Fig. 1's loop
    with numpy's own generator (no oracle code involved)."""
    n, b, C = 24, 6, 1 << 20
    e = exact_moments(n, b)
    rng = np.random.default_rng(20141215)
    y = np.full(C, 0.5)
    sx = np.zeros(C)
    sy = np.zeros(C)
    for s in range(n):
        x = (1 - y) * rng.random(C)
        y = (1 - x) * rng.random(C)
        if s >= b:
            sx += x
            sy += y
    mx, my = sx / (n - b), sy / (n - b)
    for name, v in (("mx2", mx * mx), ("my2", my * my), ("mxmy", mx * my),
                    ("mx", mx), ("my", my)):
        assert abs(v.mean() - float(e[name])) < 5 * v.std() / math.sqrt(C), name
