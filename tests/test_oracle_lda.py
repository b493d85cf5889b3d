"""Pins for the oracle's LDA fold-in Gibbs iteration (NEXT row N4; PAPER.md
P:L34 "sample from a Dirichlet distribution whose parameters are updated
during each iteration", footnote: normalised Gammas; reading R-33).

The Dirichlet step is oracle.dirichlet (pinned in test_oracle_dirichlet.py);
these pin the rest against what the model fixes:
- the categorical step's frequencies equal p_k / sum p (exact on a fine grid);
- one-hot topic-word rows force the topic; K = 1 forces theta = 1, z = 0;
- the chain's stationary law: for a tiny document, the long-run frequency of
  every topic configuration equals the exact collapsed posterior
  p(z | w) ~ prod_k Gamma(alpha_k + n_k) prod_n phi[w_n, z_n], enumerated;
- counts and the cursor span (256 D K + ceil(T/2) blocks per iteration).
"""
import itertools
import math

import numpy as np
from scipy import stats

import oracle


def test_categorical_frequencies_exact_on_grid():
    theta = np.array([0.1, 0.0, 0.35, 0.05, 0.5])
    phi_w = np.array([0.3, 0.9, 0.2, 0.6, 0.1])
    p = theta * phi_w
    M = 200_000
    counts = np.zeros(5)
    for m in range(M):
        z, _, _ = oracle.lda_categorical(theta, phi_w, (m + 0.5) / M)
        counts[z] += 1
    np.testing.assert_allclose(counts / M, p / p.sum(), atol=2.0 / M)
    assert counts[1] == 0                                    # theta_1 = 0: never chosen


def test_forced_topics_and_single_topic():
    # word 0 only in topic 2, word 1 only in topic 0 (one-hot phi rows)
    phi = np.array([[0.0, 0.0, 1.0], [1.0, 0.0, 0.0]])
    doc_off = np.array([0, 3, 5])
    words = np.array([0, 1, 0, 1, 1])
    r = oracle.lda_iteration(9, 0, 0, doc_off, words, phi, np.full(3, 0.5),
                             np.zeros(5, np.int64))
    assert list(r["z"]) == [2, 0, 2, 0, 0]
    np.testing.assert_allclose(r["theta"].sum(axis=1), 1.0, rtol=1e-15)
    r1 = oracle.lda_iteration(9, 0, 0, doc_off, words, np.ones((2, 1)), np.ones(1),
                              np.zeros(5, np.int64))
    assert np.all(r1["z"] == 0) and np.all(r1["theta"] == 1.0)


def test_counts_and_span():
    doc_off = np.array([0, 2, 2, 7])
    z = np.array([1, 1, 0, 3, 3, 3, 2])
    n = oracle.lda_counts(doc_off, z, 4)
    assert n.tolist() == [[0, 2, 0, 0], [0, 0, 0, 0], [1, 0, 1, 3]]
    assert oracle.lda_span(3, 4, 7) == 256 * 12 + 4


def test_stationary_law_equals_exact_posterior():
    """Many independent copies of one 3-token document (K = 3), each chain run
    for 12 iterations from z = 0: the empirical law of z equals the exact
    posterior p(z | w) ~ prod_k Gamma(alpha_k + n_k(z)) prod_n phi[w_n, z_n]
    (theta integrated out), enumerated over all 27 configurations."""
    K, words1 = 3, np.array([0, 1, 1])
    phi = np.array([[0.6, 0.3, 0.1], [0.2, 0.2, 0.6]])          # [V = 2][K]
    alpha = np.array([0.4, 1.3, 0.7])
    D = 20_000
    doc_off = np.arange(D + 1) * 3
    words = np.tile(words1, D)
    z = np.zeros(3 * D, np.int64)
    base = 0
    for _ in range(12):
        z = oracle.lda_iteration(2024, 5, base, doc_off, words, phi, alpha, z)["z"]
        base += oracle.lda_span(D, K, 3 * D)
    configs = list(itertools.product(range(K), repeat=3))
    w_post = []
    for c in configs:
        n = np.bincount(c, minlength=K)
        lw = sum(math.lgamma(alpha[k] + n[k]) for k in range(K))
        lw += sum(math.log(phi[words1[i], c[i]]) for i in range(3))
        w_post.append(math.exp(lw))
    post = np.array(w_post) / sum(w_post)
    zz = z.reshape(D, 3)
    idx = zz[:, 0] * 9 + zz[:, 1] * 3 + zz[:, 2]
    obs = np.bincount(idx, minlength=27)
    chi2 = np.sum((obs - D * post) ** 2 / (D * post))
    assert stats.chi2.sf(chi2, 26) > 1e-3, (chi2, obs, D * post)
