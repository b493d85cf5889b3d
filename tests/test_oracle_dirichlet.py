"""Pins for the oracle's Dirichlet-from-Gamma (P:L34 footnote; R-13).

- rows sum to 1 within K ulps;
- Dirichlet(1,1) first component ~ U(0,1);
- component means alpha_i / sum(alpha) and variances;
- Beta(alpha_k, A - alpha_k) marginal PIT on LDA-shaped synthetic alpha.
"""
import numpy as np

import oracle
import workloads
from tests.stats_util import assert_ks_uniform, mean_band, pit_beta


def test_rows_sum_to_one_and_counter_map():
    alpha = workloads.cfg4_params(64, 256, seed=5).double().numpy()
    x, tr, bad = oracle.dirichlet(3, 0, 0, alpha)
    assert bad == 0 and np.all(tr >= 1) and np.all(x >= 0)
    assert np.all(np.abs(x.sum(axis=1) - 1.0) <= 256 * 2.0**-52)
    # component k of row r is Gamma sample r*K + k with beta = 1 (R-13)
    g, tg, _ = oracle.gamma(3, 0, 0, alpha.reshape(-1), np.ones(alpha.size))
    g = g.reshape(alpha.shape)
    assert np.array_equal(tg.reshape(alpha.shape), tr)
    S = np.zeros(alpha.shape[0])
    for k in range(alpha.shape[1]):          # the oracle's sequential order
        S = S + g[:, k]
    assert np.array_equal(x, g / S[:, None])


def test_golden_uniform_marginal(golden):
    a = golden["dirichlet"]["alpha_uniform_marginal"]
    n = 100_000
    x, _, bad = oracle.dirichlet(17, 0, 0, np.tile(np.array(a), (n, 1)))
    assert bad == 0
    assert_ks_uniform(x[:, 0], "Dirichlet(1,1) marginal")


def test_golden_moments(golden):
    a = np.array(golden["dirichlet"]["alpha_moments"])
    A = a.sum()
    n = 200_000
    x, _, _ = oracle.dirichlet(19, 0, 0, np.tile(a, (n, 1)))
    for i in range(3):
        var = a[i] * (A - a[i]) / (A * A * (A + 1))
        ok, m = mean_band(x[:, i], a[i] / A, var)
        assert ok, (i, m)


def test_beta_marginal_pit_lda_shaped():
    alpha = workloads.cfg4_params(2000, 256, seed=3).double().numpy()
    x, _, bad = oracle.dirichlet(3, 0, 0, alpha)
    assert bad == 0
    A = alpha.sum(axis=1, keepdims=True)
    u = pit_beta(x, alpha, A - alpha).reshape(-1)
    assert_ks_uniform(u, "Dirichlet Beta-marginal PIT")


def test_f32_rounds_f64_and_row_offsets():
    alpha = workloads.cfg4_params(20, 16, seed=8)
    x32, t32, _ = oracle.dirichlet(4, 1, 99, alpha.numpy())
    x64, t64, _ = oracle.dirichlet(4, 1, 99, alpha.double().numpy())
    assert np.array_equal(x32, x64.astype(np.float32)) and np.array_equal(t32, t64)
    part, _, _ = oracle.dirichlet(4, 1, 99, alpha.double().numpy()[7:], row0=7)
    assert np.array_equal(part, x64[7:])


def test_invalid_component_poisons_row():
    alpha = np.ones((3, 4)); alpha[1, 2] = -1.0
    x, tr, bad = oracle.dirichlet(1, 0, 0, alpha)
    assert bad == 1 and np.all(np.isnan(x[1])) and not np.any(np.isnan(x[[0, 2]]))
