"""The public device API (include/brng_device.cuh): a user kernel drawing
one sample at a time through brng_dev:: getters must reproduce the bulk C-ABI
calls BIT-FOR-BIT (same counters, same arithmetic), and its Fig. 1 Gibbs loop
the oracle's chains.  The user kernel (tests/cuda/device_api_kernels.cu) is
compiled here with nvcc for sm_100a."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest
import torch

import oracle
import workloads
from tests.gpu_util import dev, handle

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
import paper_1412_4825_b200 as B  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def user_lib(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("devapi") / "libdevapi.so")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-gencode",
                           "arch=compute_100a,code=sm_100a", "-std=c++17", "-shared",
                           "-Xcompiler", "-fPIC", "-cudart", "shared", "-I",
                           os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cuda", "device_api_kernels.cu"),
                           "-o", out])
    L = C.CDLL(out)
    u64, vp, i = C.c_uint64, C.c_void_p, C.c_int
    L.dev_fill.argtypes = [i, u64, u64, u64, vp, vp, vp, u64, vp]
    L.dev_fill32.argtypes = [i, u64, u64, u64, vp, vp, vp, u64, vp]
    L.dev_gamma.argtypes = [u64, u64, u64, vp, vp, vp, vp, u64, vp]
    L.dev_gibbs.argtypes = [u64, u64, u64, u64, u64, vp, vp, vp]
    return L


def _s():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("dist", ["uniform", "gaussian", "exponential", "log_uniform", "laplace",
                                  "weibull"])
def test_fill_getters_bit_exact(user_lib, dist):
    n = 10_007
    g = torch.Generator().manual_seed(5)
    p0c = torch.rand(n, generator=g, dtype=torch.float64) * 3 + 0.1
    p1 = (p0c + torch.rand(n, generator=g, dtype=torch.float64) * 5 + 0.1).to(dev())
    p0 = p0c.to(dev())
    out_dev = torch.empty(n, dtype=torch.float64, device=dev())
    code = {"uniform": 2, "gaussian": 3, "exponential": 4, "log_uniform": 5, "laplace": 6,
            "weibull": 7}[dist]
    assert user_lib.dev_fill(code, 77, 3, 1000, p0.data_ptr(), p1.data_ptr(), out_dev.data_ptr(),
                             n, _s()) == 0
    with handle(77, 3, 1000) as h:
        out = torch.empty(n, dtype=torch.float64, device=dev())
        if dist == "log_uniform":
            B.brng_log_uniform_f64(h, out, n)
        elif dist == "exponential":
            B.brng_exponential_f64(h, p0, out, n)
        else:
            getattr(B, f"brng_{dist}_f64")(h, p0, p1, out, n)
    assert torch.equal(out_dev, out)


@pytest.mark.parametrize("dist", ["uniform", "gaussian", "exponential"])
def test_fill_getters_f32_bit_exact(user_lib, dist):
    n = 10_007
    p = workloads.cfg2_params(n, seed=3)
    a, b = (p["a"], p["b"]) if dist == "uniform" else (p["mu"], p["sigma"])
    if dist == "exponential":
        a = workloads.exp_params(n, seed=3)
    a, b = a.to(dev()), b.to(dev())
    code = {"uniform": 2, "gaussian": 3, "exponential": 4}[dist]
    o1 = torch.empty(n, device=dev())
    assert user_lib.dev_fill32(code, 7, 0, 9, a.data_ptr(), b.data_ptr(), o1.data_ptr(), n,
                               _s()) == 0
    with handle(7, 0, 9) as h:
        o2 = torch.empty(n, device=dev())
        if dist == "exponential":
            B.brng_exponential_f32(h, a, o2, n)
        else:
            getattr(B, f"brng_{dist}_f32")(h, a, b, o2, n)
    assert torch.equal(o1, o2)


def test_gamma_getter_bit_exact(user_lib):
    n = 50_001
    p = workloads.cfg3_params(n, seed=11, device=dev())
    o1 = torch.empty(n, dtype=torch.float64, device=dev())
    t1 = torch.empty(n, dtype=torch.uint8, device=dev())
    assert user_lib.dev_gamma(11, 0, 256, p["alpha"].data_ptr(), p["beta"].data_ptr(),
                              o1.data_ptr(), t1.data_ptr(), n, _s()) == 0
    with handle(11, 0, 256) as h:
        o2 = torch.empty(n, dtype=torch.float64, device=dev())
        t2 = torch.empty(n, dtype=torch.uint8, device=dev())
        B.brng_gamma_f64(h, p["alpha"], p["beta"], o2, n, t2)
    assert torch.equal(t1, t2) and torch.equal(o1, o2)


def test_split_trial_producer_consumer_bit_exact(user_lib):
    """mt_normal / mt_accept_z / mt_boost_log / mt_boost_from_log (the
    producer/consumer split of a trial, N4 R-33) composed in a user kernel
    equal the bulk Gamma call bit for bit, decisions included; invalid
    parameters give NaN with trial 0 (the bulk call also counts them)."""
    n = 40_003
    p = workloads.cfg3_params(n, seed=13, device=dev())
    p["alpha"][7] = -1.0
    p["beta"][9] = float("nan")
    o1 = torch.empty(n, dtype=torch.float64, device=dev())
    t1 = torch.empty(n, dtype=torch.uint8, device=dev())
    user_lib.dev_gamma_split.argtypes = user_lib.dev_gamma.argtypes
    assert user_lib.dev_gamma_split(13, 2, 512, p["alpha"].data_ptr(), p["beta"].data_ptr(),
                                    o1.data_ptr(), t1.data_ptr(), n, _s()) == 0
    with handle(13, 2, 512) as h:
        o2 = torch.empty(n, dtype=torch.float64, device=dev())
        t2 = torch.empty(n, dtype=torch.uint8, device=dev())
        B.brng_gamma_f64(h, p["alpha"], p["beta"], o2, n, t2)
    assert torch.equal(t1, t2)
    assert torch.equal(torch.nan_to_num(o1, nan=-7.0), torch.nan_to_num(o2, nan=-7.0))
    assert (t1 > 1).any()                               # later trials exercised


def test_fig1_user_gibbs_loop_matches_oracle_and_bulk(user_lib):
    nc, ns = 1024, 200
    ox = torch.empty(ns, nc, dtype=torch.float64, device=dev())
    oy = torch.empty_like(ox)
    assert user_lib.dev_gibbs(42, 0, 0, nc, ns, ox.data_ptr(), oy.data_ptr(), _s()) == 0
    r = oracle.gibbs_triangle(42, 0, 0, nc, ns)
    assert np.array_equal(ox.cpu().numpy(), r["out_x"])
    assert np.array_equal(oy.cpu().numpy(), r["out_y"])


# ---- table-driven binary64 math of the Gamma path (brng_dev::dm) -----------------
def _math(user_lib, fn, x=None, w=None, n=None):
    n = n if n is not None else len(x) if x is not None else len(w)
    xd = torch.tensor(x if x is not None else [0.0], dtype=torch.float64, device=dev())
    wd = torch.tensor(np.asarray(w if w is not None else [0], dtype=np.uint32).view(np.int32),
                      device=dev())
    out = torch.empty(n, dtype=torch.float64, device=dev())
    L = user_lib
    L.dev_math.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                           C.c_void_p]
    assert L.dev_math(fn, xd.data_ptr(), wd.data_ptr(), out.data_ptr(), n, _s()) == 0
    return out.cpu().numpy()


def _ulp_err(got, exact):
    import math
    return [abs(float(g) - float(e)) / math.ulp(float(e)) if e != 0 else abs(float(g))
            for g, e in zip(got, exact)]


def test_dm_ln_pos_accuracy(user_lib):
    """ln(1 - u53) over the trial's whole argument range [2^-53, 1] (and any
    positive normal) within 2.5 ulp of the mpmath value; exactly 0 at 1 and
    relative-accurate next to 1."""
    import mpmath as mp
    mp.mp.dps = 40
    rng = np.random.default_rng(1)
    k = np.concatenate([[0, 1, 2, 3, 2**52, 2**52 - 1, 2**53 - 1, 2**53 - 2],
                        rng.integers(0, 2**53, 3000, dtype=np.int64),
                        rng.integers(0, 2**20, 500, dtype=np.int64),
                        (2**53 - rng.integers(1, 2**20, 500, dtype=np.int64))])
    x = [(2**53 - int(v)) * 2.0**-53 for v in k]
    x += list(np.exp(rng.uniform(-690, 690, 1000)))
    x += [float(np.sqrt(0.5)), float(np.nextafter(np.sqrt(0.5), 0)), float(np.sqrt(2.0)),
          1.0 + 1.0 / 256, 1.0 - 1.0 / 256, 2.0**-1022]
    got = _math(user_lib, 0, x=x)
    exact = [mp.log(mp.mpf(v)) for v in x]
    err = _ulp_err(got, exact)
    assert got[0] == 0.0
    assert max(err) <= 2.5, (max(err), x[int(np.argmax(err))])


def test_dm_cos2pi_u32_accuracy(user_lib):
    """cos(2 pi w / 2^32) for 32-bit w (the trial's angle): absolute error
    <= 2^-53 everywhere, exact values at the quarter turns and relative
    accuracy next to the zeros of cos."""
    import mpmath as mp
    mp.mp.dps = 40
    rng = np.random.default_rng(2)
    special = [0, 1 << 30, 1 << 31, 3 << 30, (1 << 30) + 1, (1 << 30) - 1, (3 << 30) + 7,
               (1 << 23) - 1, 1 << 23, (1 << 23) + 1, 0xFFFFFFFF, 0xFF800000, 0x7FFFFFFF]
    w = special + list(rng.integers(0, 2**32, 5000, dtype=np.uint64))
    got = _math(user_lib, 1, w=w)
    exact = [mp.cos(2 * mp.pi * int(v) / mp.mpf(2) ** 32) for v in w]
    abs_err = [abs(float(g) - float(e)) for g, e in zip(got, exact)]
    assert max(abs_err) <= 2.0**-53, max(abs_err)
    assert list(got[:4]) == [1.0, 0.0, -1.0, 0.0]
    for idx in (4, 5, 6):       # next to a zero: relative accuracy
        assert abs(float(got[idx]) - float(exact[idx])) <= 2 * abs(float(exact[idx])) * 2.0**-52


def test_dm_exp_nonpos_accuracy(user_lib):
    """e^y for y <= 0 (the boost's ln(1-u)/alpha) within 2 ulp in the normal
    range, exact at 0, and through libdevice below -700 (subnormal results)."""
    import mpmath as mp
    mp.mp.dps = 40
    rng = np.random.default_rng(3)
    y = [0.0, -0.0, -1e-300, -2.0**-60, -1e-10, -0.5, -1.0, -700.0, -700.0 - 2**-40, -708.5,
         -745.0, -800.0, float(np.log(0.5))]
    y += list(-rng.exponential(20.0, 3000)) + list(-rng.uniform(0, 0.01, 500))
    got = _math(user_lib, 2, x=y)
    exact = [mp.exp(mp.mpf(v)) for v in y]
    assert got[0] == 1.0 and got[1] == 1.0
    import math
    for g, e, v in zip(got, exact, y):
        e = float(e)
        if e >= 2.0**-1022:
            assert abs(float(g) - e) <= 2 * math.ulp(e), (v, g, e)
        else:
            assert abs(float(g) - e) <= math.ulp(0.0) * 2, (v, g, e)


def test_dm_one_minus_u53_exact(user_lib):
    """1 - u53 built from the word bits equals fl(1 - u53(lo, hi)) exactly
    (no rounding happens in either), including k = 0, 1, 2^52, 2^53 - 1."""
    rng = np.random.default_rng(4)
    pairs = [(0, 0), (0x800, 0), (0, 0x80000000), (0xFFFFFFFF, 0xFFFFFFFF), (0x7FF, 0),
             (0xFFFFF800, 0x7FFFFFFF), (0, 0x00100000)]
    pairs += [tuple(int(v) for v in rng.integers(0, 2**32, 2, dtype=np.uint64))
              for _ in range(5000)]
    w = [v for p in pairs for v in p]
    got = _math(user_lib, 3, w=w, n=len(pairs))
    for (lo, hi), g in zip(pairs, got):
        k = ((hi << 32) | lo) >> 11
        assert float(g) == (2**53 - k) / 2**53, (lo, hi)


def test_dm_ln1m_u53_two_paths_and_accuracy(user_lib):
    """ln(1 - u53) as the kernels compute it (1 - u53 = (2^53 - k) 2^-53 by
    I2F, 53 taken off the exponent) equals ln_pos(one_minus_u53(...)) bit for
    bit, is exactly 0 at k = 0, and is within 2.5 ulp of mpmath."""
    import mpmath as mp
    mp.mp.dps = 40
    rng = np.random.default_rng(14)
    pairs = [(0, 0), (0x800, 0), (0, 0x80000000), (0xFFFFFFFF, 0xFFFFFFFF), (0x7FF, 0),
             (0xFFFFF800, 0x7FFFFFFF), (0, 0x00100000), (0xFFFFF800, 0xFFFFFFFF)]
    pairs += [tuple(int(v) for v in rng.integers(0, 2**32, 2, dtype=np.uint64))
              for _ in range(4000)]
    w = [v for p in pairs for v in p]
    a = _math(user_lib, 11, w=w, n=len(pairs))
    b = _math(user_lib, 12, w=w, n=len(pairs))
    assert np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))
    assert a[0] == 0.0
    exact = [mp.log(mp.mpf(2**53 - (((hi << 32) | lo) >> 11)) / mp.mpf(2) ** 53)
             for lo, hi in pairs]
    err = _ulp_err(a, exact)
    assert max(err) <= 2.5, max(err)


def test_dm_rsqrt_sqrt_accuracy(user_lib):
    """rsqrt_pos within 1.5 ulp and sqrt_nonneg within 2.5 ulp of mpmath on
    the trial's arguments (9d in [6, 1800], -2 ln(1-u) in [0, 74]) and
    across exponents; sqrt_nonneg(0) = 0."""
    import mpmath as mp
    mp.mp.dps = 40
    rng = np.random.default_rng(5)
    x = [6.0, 1800.0, 2.0**-53 * 2, 73.7, 1.0, 4.0, float(np.nextafter(1.0, 2.0))]
    x += list(rng.uniform(6, 1800, 2000)) + list(np.exp(rng.uniform(-700, 700, 2000)))
    r = _math(user_lib, 4, x=x)
    err = _ulp_err(r, [1 / mp.sqrt(mp.mpf(v)) for v in x])
    assert max(err) <= 1.5, (max(err), x[int(np.argmax(err))])
    xs = [0.0] + list(-2 * np.log1p(-rng.uniform(0, 1, 3000))) + x
    s = _math(user_lib, 5, x=xs)
    assert s[0] == 0.0
    err = _ulp_err(s[1:], [mp.sqrt(mp.mpf(v)) for v in xs[1:]])
    assert max(err) <= 2.5, (max(err), xs[1 + int(np.argmax(err))])


def _screen(user_lib, words, alpha):
    n = len(alpha)
    wd = torch.tensor(words.astype(np.uint32).view(np.int32), device=dev())
    ad = torch.tensor(alpha, dtype=torch.float64, device=dev())
    sc = torch.empty(n, dtype=torch.int8, device=dev())
    ex = torch.empty(n, dtype=torch.int8, device=dev())
    user_lib.dev_screen.argtypes = [C.c_void_p] * 4 + [C.c_uint64, C.c_void_p]
    assert user_lib.dev_screen(wd.data_ptr(), ad.data_ptr(), sc.data_ptr(), ex.data_ptr(), n,
                               _s()) == 0
    return sc.cpu().numpy(), ex.cpu().numpy()


@pytest.mark.parametrize("alpha_lo,alpha_hi,undecided", [(1.0, 1.5, 0.002), (1.0, 200.0, 0.01),
                                                         (150.0, 1e4, 0.05)])
def test_mt_screen_sound_at_the_boundary(user_lib, alpha_lo, alpha_hi, undecided):
    """The binary32 screen of the M-T acceptance test never contradicts the
    exact binary64 test.  Adversarial inputs: U is placed within a few 2^-32
    steps of exp(rhs), i.e. on the acceptance boundary, so every screen
    error would show; random inputs: the screen leaves few trials undecided
    (the band grows with d: < 1% up to the configs' alpha = 200)."""
    rng = np.random.default_rng(6)
    n = 400_000
    words = rng.integers(0, 2**32, (n, 4), dtype=np.uint64)
    alpha = np.exp(rng.uniform(np.log(alpha_lo), np.log(alpha_hi), n))
    # random words: decided almost always, never wrong
    sc, ex = _screen(user_lib, words.ravel(), alpha)
    live = sc != 2
    assert np.all((sc[live] == 0) | ((sc[live] > 0) == (ex[live] == 1)))
    assert np.mean(sc[live] == 0) < undecided
    # boundary words: w3 such that U = 1 - w3 2^-32 ~ exp(rhs) (host fp64 estimate)
    k = ((words[:, 1] << np.uint64(32)) | words[:, 0]) >> np.uint64(11)
    L = np.log((2.0**53 - k.astype(np.float64)) / 2.0**53)
    z = np.sqrt(-2 * L) * np.cos(2 * np.pi * words[:, 2].astype(np.float64) / 2.0**32)
    d = alpha - 1.0 / 3.0
    t = 1 + z / np.sqrt(9 * d)
    ok = t > 1e-3
    v = t**3
    rhs = 0.5 * z * z + d - d * v + d * np.log(np.where(ok, v, 1.0))
    ok &= (rhs < -1e-6) & (rhs > -20)
    w3 = np.round((1 - np.exp(rhs)) * 2.0**32) + rng.integers(-3, 4, n)
    ok &= (w3 >= 0) & (w3 < 2**32)
    words[:, 3] = np.where(ok, w3, 0).astype(np.uint64)
    sel = np.nonzero(ok)[0]
    sc, ex = _screen(user_lib, words[sel].ravel(), alpha[sel])
    live = sc != 2
    assert live.sum() > 0.5 * len(sel)
    bad = (sc[live] != 0) & ((sc[live] > 0) != (ex[live] == 1))
    assert not bad.any(), int(bad.sum())
    assert np.mean(sc[live] == 0) > 0.5      # the boundary really was hit


def test_dm_sincos2pi_u24_accuracy(user_lib):
    """binary32 {sin, cos}(2 pi (w>>8) 2^-24) (the f32 Box-Muller angle):
    absolute error <= 1.2e-7, exact at the quarter turns, and relative error
    <= 4 ulp wherever |value| >= 2^-8 or the angle is next to a quarter turn."""
    import mpmath as mp
    mp.mp.dps = 30
    rng = np.random.default_rng(7)
    q = [0, 1 << 30, 1 << 31, 3 << 30]
    near = [v + (d << 8) for v in q for d in (1, 2, 3, -1, -2, 5000, -5000)]
    w = q + [v % 2**32 for v in near] + list(rng.integers(0, 2**32, 6000, dtype=np.uint64))
    w = [int(v) for v in w]
    sn, cs = _math(user_lib, 6, w=w), _math(user_lib, 7, w=w)
    ang = [2 * mp.pi * (v >> 8) / mp.mpf(2) ** 24 for v in w]
    es, ec = [float(mp.sin(a)) for a in ang], [float(mp.cos(a)) for a in ang]
    assert list(sn[:4]) == [0.0, 1.0, 0.0, -1.0] and list(cs[:4]) == [1.0, 0.0, -1.0, 0.0]
    for got, ex in ((sn, es), (cs, ec)):
        err = np.abs(got - np.array(ex))
        assert err.max() <= 1.2e-7, err.max()
        big = np.abs(ex) >= 2.0**-8
        big[4:4 + len(near)] = True
        rel = err[big] / np.abs(np.array(ex)[big])
        assert rel.max() <= 4 * 2.0**-24, rel.max()


def test_dm_sincos2pi_u53_accuracy(user_lib):
    """binary64 {sin, cos}(2 pi u53(lo, hi)) (the f64 Box-Muller angle):
    absolute error <= 2^-53, exact values at the quarter turns, relative
    accuracy next to the zeros."""
    import mpmath as mp
    mp.mp.dps = 40
    rng = np.random.default_rng(8)
    ks = [0, 1 << 51, 1 << 52, 3 << 51, (1 << 51) + 1, (1 << 52) - 1, 2**53 - 1, 5, 2**53 - 5,
          (1 << 44), (1 << 44) - 1, (1 << 45) + (1 << 44)]
    ks += [int(v) for v in rng.integers(0, 2**53, 4000, dtype=np.int64)]
    w = []
    for k in ks:
        v = k << 11                      # u53 = (hi:lo) >> 11
        w += [v & 0xFFFFFFFF, v >> 32]
    sn, cs = _math(user_lib, 8, w=w, n=len(ks)), _math(user_lib, 9, w=w, n=len(ks))
    ang = [2 * mp.pi * k / mp.mpf(2) ** 53 for k in ks]
    es, ec = [float(mp.sin(a)) for a in ang], [float(mp.cos(a)) for a in ang]
    assert list(sn[:4]) == [0.0, 1.0, 0.0, -1.0] and list(cs[:4]) == [1.0, 0.0, -1.0, 0.0]
    for got, ex in ((sn, es), (cs, ec)):
        err = np.abs(got - np.array(ex))
        assert err.max() <= 2.0**-53, err.max()
    for idx in (4, 5, 6, 7, 8):          # next to zeros of sin or cos
        for got, ex in ((sn, es), (cs, ec)):
            if abs(ex[idx]) < 1e-6:
                assert abs(got[idx] - ex[idx]) <= 2 * abs(ex[idx]) * 2.0**-52


def test_dm_exp_small_accuracy(user_lib):
    """e^y for |y| <= 700 within 2 ulp (both signs: the Weibull transform's
    ln(e)/alpha), libdevice beyond (overflow to inf, underflow to 0)."""
    import math
    import mpmath as mp
    mp.mp.dps = 40
    rng = np.random.default_rng(9)
    y = [0.0, 1.0, -1.0, 700.0, -700.0, 709.0, 710.0, -745.5, 1e-300, -1e-300]
    y += list(rng.uniform(-700, 700, 3000)) + list(rng.normal(0, 1, 1000))
    got = _math(user_lib, 10, x=y)
    for g, v in zip(got, y):
        e = float(mp.exp(mp.mpf(v))) if v < 709.8 else math.inf
        if math.isinf(e):
            assert math.isinf(g)
        elif e >= 2.0**-1022:
            assert abs(g - e) <= 2 * math.ulp(e), (v, g, e)
        else:
            assert abs(g - e) <= 2 * math.ulp(0.0), (v, g, e)
