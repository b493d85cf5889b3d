"""GPU parity of K1/K2 (raw words, standard uniforms, per-sample uniform /
Gaussian / exponential fills) against the CPU oracle, through the C ABI.

Bit-exact: raw words and standard uniforms.  Tolerance: 2e-6 (f32) / 1e-12
(f64) relative to the scale of tests/parity.py.  Sizes span many CTAs and a
ragged tail; misaligned (non-16-byte) pointers take the scalar path; cursors
cross the 2^32 block boundary; full cfg2 size is checked on sampled windows.
"""
import numpy as np
import pytest
import torch

import oracle
import workloads
from tests import parity
from tests.gpu_util import dev, empty, handle, to_dev

pytestmark = pytest.mark.gpu

B = pytest.importorskip("paper_1412_4825_b200") if torch.cuda.is_available() else None
if B is None:
    pytest.skip("no CUDA device", allow_module_level=True)

SIZES = [1, 3, 4, 5, 7, 1023, 4099, 100_003]
CURSORS = [0, 17, (1 << 32) - 5, (1 << 64) - (1 << 20)]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("cursor", CURSORS)
def test_raw_u32_bit_exact(n, cursor):
    for off in (0, 1):
        with handle(0xDEADBEEF12345678, 0xABCDEF, cursor) as h:
            out = empty(n, torch.int32, off)
            B.brng_raw_u32(h, out, n)
            got = out.cpu().numpy().view(np.uint32)
            ref = oracle.raw_u32(0xDEADBEEF12345678, 0xABCDEF, cursor, n)
            assert np.array_equal(got, ref)
            assert B.brng_get_offset(h) == cursor + (n + 3) // 4


@pytest.mark.parametrize("n", SIZES)
def test_std_uniform_bit_exact(n):
    for off in (0, 1):
        with handle(99, 5, (1 << 32) - 3) as h:
            o32 = empty(n, torch.float32, off)
            B.brng_std_uniform_f32(h, o32, n)
            o64 = empty(n, torch.float64, off)
            B.brng_std_uniform_f64(h, o64, n)
            c2 = (1 << 32) - 3 + (n + 3) // 4
            assert np.array_equal(o32.cpu().numpy(),
                                  oracle.std_uniform(99, 5, (1 << 32) - 3, n, np.float32))
            assert np.array_equal(o64.cpu().numpy(), oracle.std_uniform(99, 5, c2, n, np.float64))
            assert B.brng_get_offset(h) == c2 + (n + 1) // 2


def _params(dist, n, dtype, seed=7):
    p = workloads.cfg2_params(n, seed=seed)
    td = torch.float32 if dtype == np.float32 else torch.float64
    if dist == "uniform":
        return [p["a"].to(td), p["b"].to(td)]
    if dist == "gaussian":
        return [p["mu"].to(td), p["sigma"].to(td)]
    return [workloads.exp_params(n, seed=seed, dtype=td)]


def _call(h, dist, dtype, params, out, n):
    sfx = "f32" if dtype == np.float32 else "f64"
    getattr(B, f"brng_{dist}_{sfx}")(h, *params, out, n)


@pytest.mark.parametrize("dist", ["uniform", "gaussian", "exponential"])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [1, 5, 4099, 100_003])
def test_fill_parity(dist, dtype, n):
    td = torch.float32 if dtype == np.float32 else torch.float64
    for off in (0, 1):
        params = _params(dist, n, dtype)
        with handle(7, 0, 1000) as h:
            dparams = [to_dev(p, off) for p in params]
            out = empty(n, td, off)
            _call(h, dist, dtype, dparams, out, n)
            ref, scale = parity.fill_reference(dist, 7, 0, 1000, [p.numpy() for p in params], 0,
                                               dtype)
            parity.check_close(out, ref, scale, dtype, f"{dist} {dtype.__name__} n={n} off={off}")
            assert B.brng_device_errors(h) == 0
            per = 2 if dtype == np.float64 else 4
            assert B.brng_get_offset(h) == 1000 + (n + per - 1) // per


def test_chunk_invariance_fills():
    n = 4096
    params = _params("gaussian", n, np.float32)
    d = [p.to(dev()) for p in params]
    with handle(3) as h:
        whole = torch.empty(n, device=dev())
        B.brng_gaussian_f32(h, d[0], d[1], whole, n)
    with handle(3) as h:
        a = torch.empty(n, device=dev())
        B.brng_gaussian_f32(h, d[0][:1000], d[1][:1000], a[:1000], 1000)   # 1000 % 4 == 0
        B.brng_gaussian_f32(h, d[0][1000:], d[1][1000:], a[1000:], n - 1000)
    assert torch.equal(whole, a)


def test_invalid_parameters_nan_and_counted():
    a = torch.tensor([0.0, 1.0, float("nan"), 0.0, -float("inf"), 0.0, 0.5], device=dev())
    b = torch.tensor([1.0, 1.0, 1.0, float("inf"), 0.0, 1.0, 0.25], device=dev())
    out = torch.empty(7, device=dev())
    with handle(1) as h:
        B.brng_uniform_f32(h, a, b, out, 7)
        assert B.brng_device_errors(h) == 5
        o = out.cpu().numpy()
        assert not np.isnan(o[0]) and not np.isnan(o[5])
        assert np.isnan(o[[1, 2, 3, 4, 6]]).all()
        B.brng_reset_device_errors(h)
        mu = torch.zeros(4, dtype=torch.float64, device=dev())
        sg = torch.tensor([-1.0, 0.0, float("nan"), 2.0], dtype=torch.float64, device=dev())
        o2 = torch.empty(4, dtype=torch.float64, device=dev())
        B.brng_gaussian_f64(h, mu, sg, o2, 4)
        assert B.brng_device_errors(h) == 2
        assert o2[1].item() == 0.0
        lam = torch.tensor([0.0, -1.0, 3.0], device=dev())
        o3 = torch.empty(3, device=dev())
        B.brng_exponential_f32(h, lam, o3, 3)
        assert B.brng_device_errors(h) == 4


def test_host_buffers_match_device():
    n = 10_001
    params = _params("gaussian", n, np.float64)
    with handle(11) as h:
        out_h = np.empty(n)
        B.brng_gaussian_f64(h, params[0].numpy(), params[1].numpy(), out_h, n)
        c_after = B.brng_get_offset(h)
    with handle(11) as h:
        out_d = torch.empty(n, dtype=torch.float64, device=dev())
        B.brng_gaussian_f64(h, params[0].to(dev()), params[1].to(dev()), out_d, n)
        assert B.brng_get_offset(h) == c_after
    assert np.array_equal(out_h, out_d.cpu().numpy())


def test_shard_concatenation_equals_whole():
    # rank r of G processes samples [rN/G, (r+1)N/G) at cursor base + blocks
    n, G = 1 << 16, 4
    params = _params("uniform", n, np.float32)
    d = [p.to(dev()) for p in params]
    with handle(5) as h:
        whole = torch.empty(n, device=dev())
        B.brng_uniform_f32(h, d[0], d[1], whole, n)
    parts = []
    for r in range(G):
        lo, hi = r * n // G, (r + 1) * n // G
        with handle(5, 0, lo // 4) as h:
            o = torch.empty(hi - lo, device=dev())
            B.brng_uniform_f32(h, d[0][lo:hi], d[1][lo:hi], o, hi - lo)
            parts.append(o)
    assert torch.equal(torch.cat(parts), whole)


@pytest.mark.slow
def test_cfg2_full_size_sampled():
    cfg = workloads.CFG2
    n = cfg["n"]
    p = workloads.cfg2_params(n, seed=cfg["seed"], device=dev())
    out_g = torch.empty(n, device=dev())
    out_u = torch.empty(n, device=dev())
    with handle(cfg["seed"]) as h:
        B.brng_gaussian_f32(h, p["mu"], p["sigma"], out_g, n)
        base_u = B.brng_get_offset(h)
        B.brng_uniform_f32(h, p["a"], p["b"], out_u, n)
        assert B.brng_device_errors(h) == 0
    for lo, hi in parity.windows(n, 48, 512, seed=2):
        mu, sg = p["mu"][lo:hi].cpu().numpy(), p["sigma"][lo:hi].cpu().numpy()
        ref, sc = parity.fill_reference("gaussian", cfg["seed"], 0, 0, [mu, sg], lo, np.float32)
        parity.check_close(out_g[lo:hi], ref, sc, np.float32, f"cfg2 gaussian [{lo},{hi})")
        a, b = p["a"][lo:hi].cpu().numpy(), p["b"][lo:hi].cpu().numpy()
        ref, sc = parity.fill_reference("uniform", cfg["seed"], 0, base_u, [a, b], lo, np.float32)
        parity.check_close(out_u[lo:hi], ref, sc, np.float32, f"cfg2 uniform [{lo},{hi})")
    # statistics on a deterministic stride subsample of 2^20 (KS, PIT)
    from tests.stats_util import assert_ks_uniform, pit_normal, pit_uniform
    idx = torch.arange(0, n, n >> 20, device=dev())
    assert_ks_uniform(pit_normal(out_g[idx].double().cpu().numpy(),
                                 p["mu"][idx].double().cpu().numpy(),
                                 p["sigma"][idx].double().cpu().numpy()), "cfg2 gaussian PIT")
    a, b = p["a"][idx].cpu().numpy(), p["b"][idx].cpu().numpy()
    x = out_u[idx].cpu().numpy()
    assert np.all(x >= a) and np.all(x <= b)
    assert_ks_uniform(pit_uniform(x, a, b), "cfg2 uniform PIT")


@pytest.mark.slow
def test_exponential_full_size_sampled():
    """SURVEY.md §8(d) extra on-path check: exponential f32 at N = 2^28,
    lambda ~ logU(1e-3, 1e3) (seed 7), deviates on stream 5."""
    n = 1 << 28
    lam = workloads.exp_params(n, seed=7, device=dev())
    out = torch.empty(n, device=dev())
    with handle(7, 5) as h:
        B.brng_exponential_f32(h, lam, out, n)
        assert B.brng_device_errors(h) == 0
        assert B.brng_get_offset(h) == n // 4
    for lo, hi in parity.windows(n, 48, 512, seed=3):
        ref, sc = parity.fill_reference("exponential", 7, 5, 0, [lam[lo:hi].cpu().numpy()],
                                        lo, np.float32)
        parity.check_close(out[lo:hi], ref, sc, np.float32, f"exp 2^28 [{lo},{hi})")
    from tests.stats_util import assert_ks_uniform, pit_exponential
    idx = torch.arange(0, n, n >> 20, device=dev())
    x = out[idx].double().cpu().numpy()
    assert np.all(x >= 0) and np.all(np.isfinite(x))
    assert_ks_uniform(pit_exponential(x, lam[idx].double().cpu().numpy()), "exp 2^28 PIT")


def test_host_pipeline_multi_chunk_equals_device():
    # > 64 MB per array: the host path runs as several pipelined chunks
    n = 40_000_003
    p = workloads.cfg2_params(n, seed=12)
    mu, sg = p["mu"].numpy(), p["sigma"].numpy()
    out_h = np.empty(n, np.float32)
    with handle(12, 0, 5) as h:
        B.brng_gaussian_f32(h, mu, sg, out_h, n)
        c_after = B.brng_get_offset(h)
    with handle(12, 0, 5) as h:
        out_d = torch.empty(n, device=dev())
        B.brng_gaussian_f32(h, p["mu"].to(dev()), p["sigma"].to(dev()), out_d, n)
        assert B.brng_get_offset(h) == c_after
    assert np.array_equal(out_h, out_d.cpu().numpy())
    # mixed: device inputs, host output
    with handle(12, 0, 5) as h:
        out_m = np.empty(n, np.float32)
        B.brng_gaussian_f32(h, p["mu"].to(dev()), p["sigma"].to(dev()), out_m, n)
    assert np.array_equal(out_m, out_h)


# ---- NEXT row N2: log-uniform, Laplace, Weibull ---------------
def _next_params(dist, n, dtype, seed=13):
    import math
    g = torch.Generator().manual_seed(seed)
    td = torch.float32 if dtype == np.float32 else torch.float64
    u = lambda lo, hi: (lo + (hi - lo) * torch.rand(n, generator=g, dtype=torch.float64))  # noqa
    lu = lambda lo, hi: torch.exp(math.log(lo) + u(0, 1) * (math.log(hi) - math.log(lo)))  # noqa
    if dist == "laplace":
        return [u(-10, 10).to(td), lu(1e-3, 1e3).to(td)]
    return [lu(0.2, 5).to(td), lu(0.1, 10).to(td)]          # weibull alpha, beta


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [1, 3, 4099, 100_003])
def test_next_row_n2_parity(dtype, n):
    td = torch.float32 if dtype == np.float32 else torch.float64
    sfx = "f32" if dtype == np.float32 else "f64"
    for off in (0, 1):
        with handle(13, 2, 77) as h:
            out = empty(n, td, off)
            getattr(B, f"brng_log_uniform_{sfx}")(h, out, n)
            ref, sc = parity.fill_reference("log_uniform", 13, 2, 77, [n], 0, dtype)
            parity.check_close(out, ref, sc, dtype, f"log_uniform {sfx} n={n}")
            per = 2 if dtype == np.float64 else 4
            assert B.brng_get_offset(h) == 77 + (n + per - 1) // per
        for dist in ("laplace", "weibull"):
            params = _next_params(dist, n, dtype)
            with handle(13, 2, 77) as h:
                out = empty(n, td, off)
                getattr(B, f"brng_{dist}_{sfx}")(h, *[to_dev(p, off) for p in params], out, n)
                assert B.brng_device_errors(h) == 0
                pd = {"laplace": 1 if dtype == np.float64 else 2}.get(dist, per)
                assert B.brng_get_offset(h) == 77 + (n + pd - 1) // pd
            ref, sc = parity.fill_reference(dist, 13, 2, 77, [p.numpy() for p in params], 0, dtype)
            parity.check_close(out, ref, sc, dtype, f"{dist} {sfx} n={n} off={off}")


def test_next_row_n2_statistics_and_invalid():
    from tests.stats_util import assert_ks_uniform
    n = 1 << 20
    mu, b = _next_params("laplace", n, np.float32)
    al, be = _next_params("weibull", n, np.float32, seed=14)
    with handle(21) as h:
        x = torch.empty(n, device=dev())
        B.brng_laplace_f32(h, mu.to(dev()), b.to(dev()), x, n)
        w = torch.empty(n, device=dev())
        B.brng_weibull_f32(h, al.to(dev()), be.to(dev()), w, n)
        bad = torch.tensor([0.0, -1.0, float("nan"), 2.0], device=dev())
        o = torch.empty(4, device=dev())
        B.brng_weibull_f32(h, bad, torch.ones(4, device=dev()), o, 4)
        assert B.brng_device_errors(h) == 3
        assert torch.isnan(o[:3]).all().item() and not torch.isnan(o[3])
    z = (x.double().cpu().numpy() - mu.double().numpy()) / b.double().numpy()
    assert_ks_uniform(np.where(z < 0, 0.5 * np.exp(z), 1 - 0.5 * np.exp(-z)), "GPU Laplace PIT")
    wv = w.double().cpu().numpy()
    assert_ks_uniform(-np.expm1(-(wv / be.double().numpy()) ** al.double().numpy()),
                      "GPU Weibull PIT")


def test_batch_fill_equals_constant_arrays():
    # the fixed-parameter batch fill (N1, VSL-Batch analogue) draws the same
    # counters and applies the same transform as the per-sample call
    n = 100_003
    for dist, (p0, p1) in {"uniform": (-1.0, 2.5), "gaussian": (1.0, 3.0),
                           "exponential": (0.5, 0.0), "laplace": (2.0, 0.25),
                           "weibull": (1.5, 2.0)}.items():
        for dt, td, code in ((np.float32, torch.float32, 0), (np.float64, torch.float64, 1)):
            with handle(31, 4, 9) as h:
                ob = torch.empty(n, dtype=td, device=dev())
                B.brng_batch_fill(h, B.DIST[dist], code, p0, p1, ob, n)
                cb = B.brng_get_offset(h)
            with handle(31, 4, 9) as h:
                oa = torch.empty(n, dtype=td, device=dev())
                arrs = [torch.full((n,), p0, dtype=td, device=dev())]
                if dist != "exponential":
                    arrs.append(torch.full((n,), p1, dtype=td, device=dev()))
                sfx = "f32" if dt == np.float32 else "f64"
                getattr(B, f"brng_{dist}_{sfx}")(h, *arrs, oa, n)
                assert B.brng_get_offset(h) == cb
            assert torch.equal(oa, ob), (dist, sfx)
    with handle(1) as h:
        with pytest.raises(B.brng.BrngError):
            B.brng_batch_fill(h, 5, 0, 0.0, 1.0, torch.empty(4, device=dev()), 4)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_batch_fill_vs_oracle(dt):
    """N1 (the VSL-Batch column; P:L7 vdRngUniform(method, stream, n,
    r, a, b)): the fixed-parameter batch fill against the ORACLE fed constant
    parameter arrays, element by element (ragged n, a cursor crossing 2^32
    blocks, a nonzero stream), under the fills' parity tolerance."""
    n = 40_009
    base = (1 << 32) - 7000
    code = 0 if dt == np.float32 else 1
    td = torch.float32 if dt == np.float32 else torch.float64
    for dist, (p0, p1) in {"uniform": (-1.0, 2.5), "gaussian": (1.0, 3.0),
                           "exponential": (0.5, 0.0), "laplace": (2.0, 0.25),
                           "weibull": (1.5, 2.0)}.items():
        with handle(31, 4, base) as h:
            ob = torch.empty(n, dtype=td, device=dev())
            B.brng_batch_fill(h, B.DIST[dist], code, p0, p1, ob, n)
        params = [np.full(n, p0, dt)] + ([] if dist == "exponential" else [np.full(n, p1, dt)])
        ref, scale = parity.fill_reference(dist, 31, 4, base, params, 0, dt)
        parity.check_close(ob, ref, scale, dt, f"batch {dist} {np.dtype(dt).name}")


@pytest.mark.slow
def test_fill_beyond_2_31_samples():
    """64-bit indexing: n = 2^31 + 7 f32 uniforms (8.6 GB per array); sampled
    windows and the ragged tail match the oracle."""
    n = (1 << 31) + 7
    a = torch.zeros(n, device=dev())
    b = torch.full((n,), 2.0, device=dev())
    out = torch.empty(n, device=dev())
    with handle(21, 4, 3) as h:
        B.brng_uniform_f32(h, a, b, out, n)
        assert B.brng_get_offset(h) == 3 + (n + 3) // 4
    for lo, hi in list(parity.windows(n, 16, 256, seed=5)) + [(n - 9, n)]:
        ref, sc = parity.fill_reference("uniform", 21, 4, 3, [a[lo:hi].cpu().numpy(),
                                                               b[lo:hi].cpu().numpy()],
                                        lo, np.float32)
        parity.check_close(out[lo:hi], ref, sc, np.float32, f"2^31+ [{lo},{hi})")
    del a, b, out
    torch.cuda.empty_cache()
