"""Statistical helpers shared by the oracle pins and the GPU statistical tests.

KS p-values use scipy.stats.kstest (asymptotic Kolmogorov); the 1% critical
value 1.63/sqrt(n) of S:L89 / S:L317 is asserted alongside.  Seeds and sample
sizes are fixed in advance and never re-rolled.
"""
import math

import numpy as np
from scipy import special, stats

KS_P_MIN = 0.01


def ks_uniform(u):
    """PIT values u ~ U(0,1)?  Returns (D, p)."""
    r = stats.kstest(np.asarray(u, np.float64), "uniform")
    return r.statistic, r.pvalue


def assert_ks_uniform(u, what=""):
    D, p = ks_uniform(u)
    n = len(u)
    assert p > KS_P_MIN and D < 1.63 / math.sqrt(n), f"{what}: KS D={D:.3g} p={p:.3g} n={n}"
    return D, p


def pit_normal(x, mu, sigma):
    return special.ndtr((np.asarray(x, np.float64) - mu) / sigma)


def pit_uniform(x, a, b):
    return (np.asarray(x, np.float64) - a) / (np.asarray(b, np.float64) - np.asarray(a, np.float64))


def pit_exponential(x, lam):
    return -np.expm1(-np.asarray(lam, np.float64) * np.asarray(x, np.float64))


def pit_gamma(x, alpha, beta):
    return special.gammainc(np.asarray(alpha, np.float64), np.asarray(x, np.float64) / beta)


def pit_beta(x, a, b):
    return special.betainc(a, b, np.asarray(x, np.float64))


def mean_band(values, mean, var, z=5.0):
    """|sample mean - mean| <= z * sqrt(var / n)."""
    n = len(values)
    m = float(np.mean(values))
    return abs(m - mean) <= z * math.sqrt(var / n), m


def mt_acceptance(alpha_prime):
    """Closed-form Marsaglia-Tsang acceptance probability (no squeeze), derived
    in DESIGN.md "Oracle pins": P = e^d Gamma(a') sqrt(d) / (sqrt(2 pi) d^a'),
    d = a' - 1/3."""
    a = alpha_prime
    d = a - 1.0 / 3.0
    return math.exp(d + math.lgamma(a) + 0.5 * math.log(d) - 0.5 * math.log(2 * math.pi)
                    - a * math.log(d))
