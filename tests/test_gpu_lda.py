"""NEXT row N4 on the GPU: the LDA fold-in Gibbs consumer (brng_lda_gibbs,
include/brng.h; reading R-33).

- chained one-iteration parity against the oracle-side loop built from
  oracle.dirichlet (oracle.lda_iteration): from the same state z, theta within
  the Dirichlet parity tolerance and every token's topic equal, except
  rounding ties of the categorical step (x within 1e-9 C of the boundary),
  which are counted;
- the three deviate sources (inline device API, asynchronous producer ring,
  synchronous bulk calls) give the same bits over several iterations, and
  the cursor advances by n_iter * (256 D K + ceil(T/2));
- the inline theta equals brng_dirichlet_f64 at the same cursor bit for bit;
- argument errors.
"""
import numpy as np
import pytest
import torch

import oracle
import workloads
from tests import parity
from tests.gpu_util import dev, handle

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
import paper_1412_4825_b200 as B  # noqa: E402


def _corpus(D=300, K=16, V=64, L=30, seed=5):
    c = workloads.lda_corpus(D, K, V, L, seed=seed)
    alpha = torch.linspace(0.05, 1.5, K, dtype=torch.float64)     # boosted and not
    return c, alpha


def _run(c, alpha, z, n_iter, mode, seed=77, stream=3, cursor=0, theta=True):
    D, K = len(c["doc_off"]) - 1, c["phi"].shape[1]
    V, T = c["phi"].shape[0], c["n_tokens"]
    zd = z.to(dev()).clone()
    th = torch.empty(D, K, dtype=torch.float64, device=dev()) if theta else None
    with handle(seed, stream, cursor) as h:
        B.brng_lda_gibbs(h, D, K, V, T, c["doc_off"].to(dev()), c["words"].to(dev()),
                         c["phi"].to(dev()), alpha.to(dev()), zd, th, n_iter, mode)
        end = B.brng_get_offset(h)
        errs = B.brng_device_errors(h)
    return zd.cpu().numpy().astype(np.int64), (th.cpu().numpy() if theta else None), end, errs


def test_chained_iterations_match_oracle():
    c, alpha = _corpus()
    D, K, T = len(c["doc_off"]) - 1, c["phi"].shape[1], c["n_tokens"]
    doc_off, words = c["doc_off"].numpy(), c["words"].numpy()
    phi, al = c["phi"].numpy(), alpha.numpy()
    z = c["z0"]
    cursor = (1 << 32) - 5000                       # the iterations cross a 2^32 block boundary
    span = oracle.lda_span(D, K, T)
    n_tie = 0
    for it in range(4):
        zg, thg, end, errs = _run(c, alpha, z, 1, B.LDA_INLINE, cursor=cursor)
        assert end == cursor + span and errs == 0
        r = oracle.lda_iteration(77, 3, cursor, doc_off, words, phi, al,
                                 z.numpy().astype(np.int64))
        # theta: the Dirichlet criterion (tests/parity.py), rows as in brng_dirichlet_f64
        dr = parity.value_check(thg.reshape(-1), r["theta"].reshape(-1),
                                np.abs(r["theta"].reshape(-1)), np.float64,
                                lambda j: parity.gamma_condition(77, 3, cursor, j,
                                                                 float(r["rows"].reshape(-1)[j]),
                                                                 int(r["trials"].reshape(-1)[j])),
                                f"theta it{it}")
        assert dr["ratio"] <= 1.0
        for j in np.flatnonzero(zg != r["z"]):
            # a disagreement must be a rounding tie of x against a running sum
            cum, x = np.array(r["cum"][j]), r["x"][j]
            kk = min(int(zg[j]), int(r["z"][j]))
            assert abs(x - cum[kk]) <= 1e-9 * cum[-1], (it, j, zg[j], r["z"][j])
            n_tie += 1
        z = torch.from_numpy(zg.astype(np.int16))   # continue from the GPU's state
        cursor += span
    assert n_tie <= 2


def test_three_sources_bit_identical():
    c, alpha = _corpus(D=517, K=40, V=200, L=45, seed=9)
    D, K, T = len(c["doc_off"]) - 1, c["phi"].shape[1], c["n_tokens"]
    res = [_run(c, alpha, c["z0"], 3, m, cursor=123) for m in (B.LDA_INLINE, B.LDA_RING,
                                                               B.LDA_BULK)]
    for zg, th, end, errs in res[1:]:
        assert np.array_equal(zg, res[0][0]) and np.array_equal(th, res[0][1])
        assert end == res[0][2] == 123 + 3 * oracle.lda_span(D, K, T) and errs == 0
    # the state moved (the sampler is not a no-op) and stays in range
    assert (res[0][0] != c["z0"].numpy()).mean() > 0.3 and res[0][0].max() < K


def test_inline_theta_equals_bulk_dirichlet_call():
    c, alpha = _corpus(D=200, K=24, V=50, L=20, seed=11)
    D, K = len(c["doc_off"]) - 1, c["phi"].shape[1]
    zg, th, _, _ = _run(c, alpha, c["z0"], 1, B.LDA_INLINE, cursor=999)
    rows = torch.from_numpy(alpha.numpy()[None, :] +
                            oracle.lda_counts(c["doc_off"].numpy(), c["z0"].numpy().astype(np.int64),
                                              K)).to(dev())
    out = torch.empty(D, K, dtype=torch.float64, device=dev())
    with handle(77, 3, 999) as h:
        B.brng_dirichlet_f64(h, rows, D, K, out, None)
    assert np.array_equal(out.cpu().numpy(), th)


def test_lda_argument_errors():
    c, alpha = _corpus(D=8, K=4, V=8, L=5)
    D, K, V, T = 8, 4, 8, c["n_tokens"]
    d = {k: v.to(dev()) for k, v in c.items() if k != "n_tokens"}
    with handle(1) as h:
        raw = lambda *a: B.brng._lib.brng_lda_gibbs(h, *a)  # noqa: E731
        args = [D, K, V, T, d["doc_off"].data_ptr(), d["words"].data_ptr(), d["phi"].data_ptr(),
                alpha.to(dev()).data_ptr(), d["z0"].data_ptr(), None, 1]
        assert raw(*args[:1], 0, *args[2:], 0) == -2                 # k == 0
        assert raw(*args, 7) == -4                                   # unknown mode
        host_z = c["z0"].clone()
        a2 = list(args); a2[8] = host_z.data_ptr()
        assert raw(*a2, 0) == -4                                     # host pointer
        assert B.brng_get_offset(h) == 0
        assert raw(*args[:-1], 0, 0) == 0 and B.brng_get_offset(h) == 0   # n_iter == 0


def test_lda_edge_cases():
    """Empty documents, K = 1, the maximum K, an invalid alpha component."""
    # empty documents between non-empty ones; K = 3
    doc_off = torch.tensor([0, 0, 4, 4, 4, 9, 9], dtype=torch.int64)
    words = torch.tensor([0, 1, 2, 1, 0, 2, 2, 1, 0], dtype=torch.int32)
    phi = torch.tensor([[0.5, 0.3, 0.2], [0.1, 0.1, 0.8], [0.3, 0.3, 0.4]], dtype=torch.float64)
    alpha = torch.tensor([0.2, 1.0, 3.0], dtype=torch.float64)
    z0 = torch.tensor([0, 1, 2, 0, 1, 2, 0, 1, 2], dtype=torch.int16)
    c = dict(doc_off=doc_off, words=words, phi=phi, z0=z0, n_tokens=9)
    zg, th, end, errs = _run(c, alpha, z0, 1, B.LDA_INLINE, cursor=77)
    r = oracle.lda_iteration(77, 3, 77, doc_off.numpy(), words.numpy(), phi.numpy(),
                             alpha.numpy(), z0.numpy().astype(np.int64))
    assert np.array_equal(zg, r["z"]) and errs == 0
    np.testing.assert_allclose(th, r["theta"], rtol=1e-11, atol=0)   # empty docs: Dirichlet(alpha)
    assert end == 77 + oracle.lda_span(6, 3, 9)
    # K = 1: theta = g fl(1/g) (within an ulp of 1; R-13), z = 0
    c1 = dict(doc_off=doc_off, words=words, phi=torch.ones(3, 1, dtype=torch.float64),
              z0=torch.zeros(9, dtype=torch.int16), n_tokens=9)
    zg, th, _, _ = _run(c1, torch.ones(1, dtype=torch.float64), c1["z0"], 2, B.LDA_RING)
    assert np.all(zg == 0) and np.all(np.abs(th - 1.0) <= 2.0**-52)
    # a component with alpha_k + n_dk not positive-finite (here alpha_1 = NaN):
    # every document's theta NaN, one error per document, its tokens z = 0
    bad = alpha.clone(); bad[1] = float("nan")
    for mode in (B.LDA_INLINE, B.LDA_RING, B.LDA_BULK):
        zg, th, _, errs = _run(c, bad, z0, 1, mode)
        assert np.all(np.isnan(th)) and errs == 6 and np.all(zg == 0), mode


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_lda_max_k(mode):
    """K = 1024 (BRNG_LDA_MAX_K: 12 KB of shared memory per warp): the three
    sources agree with each other and the oracle on one iteration."""
    c, _ = _corpus(D=24, K=1024, V=40, L=60, seed=21)
    alpha = torch.full((1024,), 0.05, dtype=torch.float64)
    zg, th, _, errs = _run(c, alpha, c["z0"], 1, mode, cursor=5)
    r = oracle.lda_iteration(77, 3, 5, c["doc_off"].numpy(), c["words"].numpy(), c["phi"].numpy(),
                             alpha.numpy(), c["z0"].numpy().astype(np.int64))
    assert errs == 0
    mism = np.flatnonzero(zg != r["z"])
    for j in mism:                                      # only rounding ties may differ
        cum, x = np.array(r["cum"][j]), r["x"][j]
        assert abs(x - cum[min(int(zg[j]), int(r["z"][j]))]) <= 1e-9 * cum[-1]
    assert len(mism) <= 1
    np.testing.assert_allclose(th, r["theta"], rtol=1e-9, atol=0)


def test_lda_malformed_inputs_are_counted_not_followed():
    """A decreasing / out-of-range document range and out-of-range word ids
    are counted in the device error counter and skipped (no out-of-bounds
    access); the other documents are unaffected."""
    c, alpha = _corpus(D=6, K=4, V=8, L=5, seed=3)
    good = _run(c, alpha, c["z0"], 1, B.LDA_INLINE, cursor=9)
    bad = dict(c)
    off = c["doc_off"].clone()
    off[3] = off[4] + 1000                     # doc 2 ends past doc 3's end (decreasing next)
    bad["doc_off"] = off
    zg, _, _, errs = _run(bad, alpha, c["z0"], 1, B.LDA_INLINE, cursor=9)
    assert errs >= 2                           # docs 2 and 3 malformed
    keep = np.r_[int(off[0]):int(off[2]), int(c["doc_off"][4]):c["n_tokens"]]
    assert np.array_equal(zg[keep], good[0][keep])
    w = c["words"].clone()
    w[0] = 8                                   # == v: out of range
    bad2 = dict(c, words=w)
    zg2, _, _, errs2 = _run(bad2, alpha, c["z0"], 1, B.LDA_BULK, cursor=9)
    assert errs2 == 1 and zg2[0] == int(c["z0"][0])
    assert np.array_equal(zg2[1:], good[0][1:])


def _phi_at(phi, byte_off):
    """phi's values in device memory starting byte_off bytes past a 256-byte
    boundary (the consumer reads rows with 256-bit loads only when phi is
    32-byte aligned and K % 4 == 0)."""
    n = phi.numel()
    buf = torch.empty(n + 64, dtype=torch.float64, device=dev())
    v = buf[byte_off // 8: byte_off // 8 + n].view(phi.shape)
    v.copy_(phi.to(dev()))
    return v


@pytest.mark.parametrize("K", [64, 40, 7])
def test_categorical_load_paths_agree(K):
    """The 256-bit-load search (K % 4 == 0, phi 32-byte aligned) and the
    scalar search (phi 8 bytes off) give the same topics bit for bit, and
    both match the oracle's plain sequential search up to rounding ties of
    theta."""
    c, alpha = _corpus(D=400, K=K, V=120, L=40, seed=31 + K)
    D, T = len(c["doc_off"]) - 1, c["n_tokens"]
    res = []
    for off in (0, 8):
        zd = c["z0"].to(dev()).clone()
        th = torch.empty(D, K, dtype=torch.float64, device=dev())
        with handle(77, 3, 11) as h:
            B.brng_lda_gibbs(h, D, K, c["phi"].shape[0], T, c["doc_off"].to(dev()),
                             c["words"].to(dev()), _phi_at(c["phi"], off), alpha.to(dev()), zd, th,
                             1, B.LDA_INLINE)
            assert B.brng_device_errors(h) == 0
        res.append((zd.cpu().numpy().astype(np.int64), th.cpu().numpy()))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    r = oracle.lda_iteration(77, 3, 11, c["doc_off"].numpy(), c["words"].numpy(),
                             c["phi"].numpy(), alpha.numpy(), c["z0"].numpy().astype(np.int64))
    mism = np.flatnonzero(res[0][0] != r["z"])
    for j in mism:
        cum, x = np.array(r["cum"][j]), r["x"][j]
        assert abs(x - cum[min(int(res[0][0][j]), int(r["z"][j]))]) <= 1e-9 * cum[-1]
    assert len(mism) <= 2


def test_categorical_negative_weights_take_the_plain_search():
    """phi entries with a set sign bit (negative values, -0.0) make the running
    sums non-monotone; the consumer then runs the plain sequential search, so
    the topics still equal the oracle's first k with x < c_k (given theta)."""
    c, alpha = _corpus(D=300, K=32, V=50, L=30, seed=5)
    phi = c["phi"].clone()
    phi[::3, 5] *= -1.0                       # every third word: a negative weight
    phi[1::7, 9] = -0.0
    c2 = dict(c, phi=phi)
    zg, th, _, errs = _run(c2, alpha, c["z0"], 1, B.LDA_BULK, cursor=21)
    assert errs == 0
    r = oracle.lda_iteration(77, 3, 21, c["doc_off"].numpy(), c["words"].numpy(), phi.numpy(),
                             alpha.numpy(), c["z0"].numpy().astype(np.int64))
    # recompute the oracle's search from the GPU's own theta: exact equality
    words, doc_off = c["words"].numpy(), c["doc_off"].numpy()
    u = oracle.std_uniform(77, 3, 21 + oracle.GAMMA_STRIDE * th.size, c["n_tokens"], np.float64)
    for d in range(len(doc_off) - 1):
        for j in range(doc_off[d], doc_off[d + 1]):
            zj, _, _ = oracle.lda_categorical(th[d], phi.numpy()[words[j]], u[j])
            assert zg[j] == zj, (d, j)
    assert (zg != r["z"]).mean() < 0.01
