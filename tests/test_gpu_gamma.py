"""GPU parity of K3 (Gamma) and K4 (Dirichlet) against the CPU oracle.

Decisions (the accepting trial index) must agree except boundary ties
(< 1e-6 of samples); values within 1e-12 (f64) / 2e-6 (f32).  Full cfg3 and
cfg4 sizes are checked on sampled windows / rows in the bench's launch
configuration, plus PIT-KS on a 2^20 subsample.
"""
import numpy as np
import pytest
import torch

import oracle
import workloads
from tests import parity
from tests.gpu_util import dev, empty, handle, to_dev

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
import paper_1412_4825_b200 as B  # noqa: E402


def _assert_decisions(r, what):
    assert r["n_fail"] == 0, f"{what}: {r}"
    assert r["n_tie"] <= max(1, r["n"] * parity.TIE_RATE_MAX), f"{what}: ties {r}"


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("n", [1, 31, 33, 1025, 70_001])
def test_gamma_parity(dtype, n):
    td = torch.float64 if dtype == np.float64 else torch.float32
    p = workloads.cfg3_params(n, seed=11, dtype=td)
    for off in (0, 1):
        with handle(11, 3, 12345) as h:
            out = empty(n, td, off)
            tr = empty(n, torch.uint8, off)
            B.brng_gamma_f64(h, to_dev(p["alpha"], off), to_dev(p["beta"], off), out, n, tr) \
                if dtype == np.float64 else \
                B.brng_gamma_f32(h, to_dev(p["alpha"], off), to_dev(p["beta"], off), out, n, tr)
            assert B.brng_get_offset(h) == 12345 + 256 * n
            assert B.brng_device_errors(h) == 0
        r = parity.gamma_compare(out, tr, p["alpha"].numpy(), p["beta"].numpy(), 11, 3, 12345,
                                 dtype=dtype)
        _assert_decisions(r, f"gamma {dtype.__name__} n={n}")


def test_gamma_special_shapes_and_invalid():
    alpha = torch.tensor([1.0, 1e-3, 0.999999, 1.0 + 1e-12, 1e6, 0.0, -1.0, float("nan"),
                          2.0, 3.0], dtype=torch.float64)
    beta = torch.tensor([1.0, 1.0, 2.0, 0.5, 1e-3, 1.0, 1.0, 1.0, 0.0, float("inf")],
                        dtype=torch.float64)
    n = len(alpha)
    with handle(2) as h:
        out = torch.empty(n, dtype=torch.float64, device=dev())
        tr = torch.empty(n, dtype=torch.uint8, device=dev())
        B.brng_gamma_f64(h, alpha.to(dev()), beta.to(dev()), out, n, tr)
        assert B.brng_device_errors(h) == 5
    r = parity.gamma_compare(out, tr, alpha.numpy(), beta.numpy(), 2, 0, 0)
    _assert_decisions(r, "special shapes")
    assert (tr.cpu().numpy()[5:] == 0).all()


def test_gamma_trials_optional_and_host_buffers():
    n = 5000
    p = workloads.cfg3_params(n, seed=4)
    with handle(4) as h:
        o1 = torch.empty(n, dtype=torch.float64, device=dev())
        B.brng_gamma_f64(h, p["alpha"].to(dev()), p["beta"].to(dev()), o1, n, None)
    with handle(4) as h:
        o2 = np.empty(n)
        t2 = np.empty(n, np.uint8)
        B.brng_gamma_f64(h, p["alpha"].numpy(), p["beta"].numpy(), o2, n, t2)
    assert np.array_equal(o1.cpu().numpy(), o2)


def test_gamma_statistics_closed_form():
    from tests.stats_util import assert_ks_uniform, mt_acceptance, pit_exponential
    n = 1 << 20
    with handle(41) as h:
        a = torch.ones(n, dtype=torch.float64, device=dev())
        out = torch.empty(n, dtype=torch.float64, device=dev())
        tr = torch.empty(n, dtype=torch.uint8, device=dev())
        B.brng_gamma_f64(h, a, a, out, n, tr)
    assert_ks_uniform(pit_exponential(out.cpu().numpy(), 1.0), "GPU Gamma(1) vs Exp(1)")
    P = mt_acceptance(1.0)
    first = (tr == 1).double().mean().item()
    assert abs(first - P) < 5 * np.sqrt(P * (1 - P) / n)


@pytest.mark.slow
def test_cfg3_full_size_sampled():
    cfg = workloads.CFG3
    n = cfg["n"]
    p = workloads.cfg3_params(n, seed=cfg["seed"], device=dev())
    out = torch.empty(n, dtype=torch.float64, device=dev())
    tr = torch.empty(n, dtype=torch.uint8, device=dev())
    with handle(cfg["seed"]) as h:
        B.brng_gamma_f64(h, p["alpha"], p["beta"], out, n, tr)
        assert B.brng_device_errors(h) == 0
    tot = dict(n=0, n_tie=0, n_fail=0)
    for lo, hi in parity.windows(n, 48, 1024, seed=3):
        r = parity.gamma_compare(out[lo:hi], tr[lo:hi], p["alpha"][lo:hi].cpu().numpy(),
                                 p["beta"][lo:hi].cpu().numpy(), cfg["seed"], 0, 0, i0=lo)
        for k in tot:
            tot[k] += r[k]
    _assert_decisions(tot, "cfg3 sampled")
    assert (tr > 0).all().item()
    from tests.stats_util import assert_ks_uniform, pit_gamma
    idx = torch.arange(0, n, n >> 20, device=dev())
    assert_ks_uniform(pit_gamma(out[idx].cpu().numpy(), p["alpha"][idx].cpu().numpy(),
                                p["beta"][idx].cpu().numpy()), "cfg3 gamma PIT")


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("rows,k", [(1, 1), (3, 2), (257, 256), (64, 37), (33, 300),
                                    (9, 700), (5, 2049), (2, 5000)])
def test_dirichlet_parity(dtype, rows, k):
    td = torch.float64 if dtype == np.float64 else torch.float32
    alpha = workloads.cfg4_params(rows, k, seed=3, dtype=td)
    with handle(3, 0, 77) as h:
        out = torch.empty(rows, k, dtype=td, device=dev())
        tr = torch.empty(rows, k, dtype=torch.uint8, device=dev())
        fn = B.brng_dirichlet_f64 if dtype == np.float64 else B.brng_dirichlet_f32
        fn(h, alpha.to(dev()), rows, k, out, tr)
        assert B.brng_get_offset(h) == 77 + 256 * rows * k
        assert B.brng_device_errors(h) == 0
    r = parity.dirichlet_compare(out, tr, alpha.numpy(), 3, 0, 77, dtype=dtype)
    _assert_decisions(r, f"dirichlet {rows}x{k}")
    s = out.double().sum(dim=1).cpu().numpy()
    assert np.all(np.abs(s - 1) <= k * (2e-6 if dtype == np.float32 else 1e-15))


def test_dirichlet_equals_normalised_gamma_counters():
    rows, k = 40, 256
    alpha = workloads.cfg4_params(rows, k, seed=9, dtype=torch.float64)
    with handle(9) as h:
        out = torch.empty(rows, k, dtype=torch.float64, device=dev())
        B.brng_dirichlet_f64(h, alpha.to(dev()), rows, k, out, None)
    with handle(9) as h:
        g = torch.empty(rows * k, dtype=torch.float64, device=dev())
        B.brng_gamma_f64(h, alpha.reshape(-1).to(dev()), torch.ones(rows * k, dtype=torch.float64,
                         device=dev()), g, rows * k, None)
    g = g.view(rows, k)
    np.testing.assert_allclose(out.cpu().numpy(), (g / g.sum(dim=1, keepdim=True)).cpu().numpy(),
                               rtol=1e-14, atol=1e-300)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("k", [37, 256, 1500])
def test_dirichlet_trials_array_does_not_change_values(dtype, k):
    """The kernels are specialised on whether a trials array was passed (no
    per-sample null test without one); both forms give the same bits."""
    rows = 300
    al = workloads.cfg4_params(rows, k, seed=8).numpy().astype(dtype)
    td = torch.float32 if dtype == np.float32 else torch.float64
    fn = B.brng_dirichlet_f32 if dtype == np.float32 else B.brng_dirichlet_f64
    outs = []
    for with_trials in (False, True):
        x = torch.empty(rows, k, dtype=td, device=dev())
        tr = torch.empty(rows, k, dtype=torch.uint8, device=dev()) if with_trials else None
        with handle(9, 2, 77) as h:
            fn(h, torch.from_numpy(al).to(dev()), rows, k, x, tr)
            assert B.brng_device_errors(h) == 0
        outs.append(x.cpu().numpy())
    assert np.array_equal(outs[0].view(np.uint8), outs[1].view(np.uint8))


def test_dirichlet_invalid_row():
    alpha = torch.ones(3, 4, dtype=torch.float64)
    alpha[1, 2] = -1.0
    with handle(1) as h:
        out = torch.empty(3, 4, dtype=torch.float64, device=dev())
        B.brng_dirichlet_f64(h, alpha.to(dev()), 3, 4, out, None)
        assert B.brng_device_errors(h) == 1
    o = out.cpu().numpy()
    assert np.isnan(o[1]).all() and not np.isnan(o[[0, 2]]).any()


@pytest.mark.slow
def test_cfg4_full_size_sampled():
    cfg = workloads.CFG4
    D, K = cfg["n_docs"], cfg["k"]
    alpha = workloads.cfg4_params(D, K, seed=cfg["seed"], device=dev())
    out = torch.empty(D, K, device=dev())
    tr = torch.empty(D, K, dtype=torch.uint8, device=dev())
    with handle(cfg["seed"]) as h:
        B.brng_dirichlet_f32(h, alpha, D, K, out, tr)
        assert B.brng_device_errors(h) == 0
    tot = dict(n=0, n_tie=0, n_fail=0)
    for lo, hi in parity.windows(D, 24, 16, seed=4):
        r = parity.dirichlet_compare(out[lo:hi], tr[lo:hi], alpha[lo:hi].cpu().numpy(),
                                     cfg["seed"], 0, 0, row0=lo, dtype=np.float32)
        for k in tot:
            tot[k] += r[k]
    _assert_decisions(tot, "cfg4 sampled")
    s = out.double().sum(dim=1)
    assert (s - 1).abs().max().item() < K * 2e-6
    from tests.stats_util import assert_ks_uniform, pit_beta
    rows = torch.arange(0, D, D // 4096, device=dev())
    x = out[rows].double().cpu().numpy()
    a = alpha[rows].double().cpu().numpy()
    A = a.sum(axis=1, keepdims=True)
    assert_ks_uniform(pit_beta(x, a, A - a).reshape(-1), "cfg4 Beta-marginal PIT")


def test_host_pipeline_multi_chunk_gamma_dirichlet():
    n = 10_000_001                                    # 80 MB per f64 array -> 2 chunks
    p = workloads.cfg3_params(n, seed=21)
    oh = np.empty(n); th = np.empty(n, np.uint8)
    with handle(21) as h:
        B.brng_gamma_f64(h, p["alpha"].numpy(), p["beta"].numpy(), oh, n, th)
    with handle(21) as h:
        od = torch.empty(n, dtype=torch.float64, device=dev())
        td = torch.empty(n, dtype=torch.uint8, device=dev())
        B.brng_gamma_f64(h, p["alpha"].to(dev()), p["beta"].to(dev()), od, n, td)
    assert np.array_equal(oh, od.cpu().numpy()) and np.array_equal(th, td.cpu().numpy())
    D, K = 100_003, 256                               # 102 MB f32 -> 2 chunks
    al = workloads.cfg4_params(D, K, seed=22)
    xh = np.empty((D, K), np.float32)
    with handle(22) as h:
        B.brng_dirichlet_f32(h, al.numpy(), D, K, xh, None)
    with handle(22) as h:
        xd = torch.empty(D, K, device=dev())
        B.brng_dirichlet_f32(h, al.to(dev()), D, K, xd, None)
    assert np.array_equal(xh, xd.cpu().numpy())
    # long rows (the scratch / in-place paths), both output types, 2+ chunks
    for dt, npt, fn in ((torch.float32, np.float32, B.brng_dirichlet_f32),
                        (torch.float64, np.float64, B.brng_dirichlet_f64)):
        D, K = 9_001, 3_000
        al = workloads.cfg4_params(D, K, seed=23, dtype=dt)
        xh = np.empty((D, K), npt)
        with handle(23) as h:
            fn(h, al.numpy(), D, K, xh, None)
        with handle(23) as h:
            xd = torch.empty(D, K, dtype=dt, device=dev())
            fn(h, al.to(dev()), D, K, xd, None)
        assert np.array_equal(xh, xd.cpu().numpy()), dt


@pytest.mark.slow
def test_dirichlet_beyond_2_31_components():
    """64-bit indexing: D*K = 2^31 + 129 components (f32, 8.6 GB each way);
    sampled rows, including the last one, match the oracle."""
    K = 129
    D = (1 << 31) // K + 2
    assert D * K > (1 << 31)
    alpha = torch.full((D, K), 0.5, dtype=torch.float32, device=dev())
    out = torch.empty(D, K, device=dev())
    tr = torch.empty(D, K, dtype=torch.uint8, device=dev())
    with handle(5, 3, 11) as h:
        B.brng_dirichlet_f32(h, alpha, D, K, out, tr)
        assert B.brng_device_errors(h) == 0
        assert B.brng_get_offset(h) == 11 + 256 * D * K
    tot = dict(n=0, n_tie=0, n_fail=0)
    wins = list(parity.windows(D, 6, 4, seed=9)) + [(D - 4, D)]
    for lo, hi in wins:
        r = parity.dirichlet_compare(out[lo:hi], tr[lo:hi], alpha[lo:hi].cpu().numpy(), 5, 3, 11,
                                     row0=lo, dtype=np.float32)
        for k in tot:
            tot[k] += r[k]
    _assert_decisions(tot, "dirichlet > 2^31")
    del alpha, out, tr
    torch.cuda.empty_cache()


def test_gamma_extreme_shapes():
    """Shapes at the ends of binary64: tiny and subnormal alpha (the boost
    underflows to 0 unless ln(1-u) = 0), huge alpha, infinite alpha
    (invalid); each matches the oracle's decisions and values."""
    alpha = torch.tensor([1e-300, 5e-324, 1e-20, 1e-8, 1e15, 1e300, float("inf"), 0.5],
                         dtype=torch.float64)
    beta = torch.tensor([1.0, 1.0, 3.0, 1.0, 1e-10, 1.0, 1.0, 1e100], dtype=torch.float64)
    alpha = alpha.repeat(64)                      # several trials/boost blocks per shape
    beta = beta.repeat(64)
    n = len(alpha)
    with handle(17, 3, 5) as h:
        out = torch.empty(n, dtype=torch.float64, device=dev())
        tr = torch.empty(n, dtype=torch.uint8, device=dev())
        B.brng_gamma_f64(h, alpha.to(dev()), beta.to(dev()), out, n, tr)
        assert B.brng_device_errors(h) == 64       # alpha = inf
    r = parity.gamma_compare(out, tr, alpha.numpy(), beta.numpy(), 17, 3, 5)
    _assert_decisions(r, "extreme shapes")
    o = out.cpu().numpy().reshape(64, 8)
    assert np.isnan(o[:, 6]).all()
    assert np.all(o[:, [0, 1, 2]] >= 0) and np.all(np.isfinite(o[:, [0, 1, 2, 3, 4, 5, 7]]))
