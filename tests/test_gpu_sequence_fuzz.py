"""A seeded random SEQUENCE of C-ABI calls of every family on one handle --
fills (all distributions, f32/f64), Gamma, Dirichlet, Gibbs, batch fills --
with random sizes (ragged, tiny, multi-CTA), misaligned pointers and a cursor
that starts near a 2^32 block boundary.  Each call is checked against the
oracle at the cursor it consumed (include/brng.h: the cursor advances by the
call's span at enqueue), so the test covers the cursor bookkeeping across
interleaved families as well as each family's values (R-12)."""
import numpy as np
import pytest
import torch

import oracle
import workloads
from tests import parity
from tests.gpu_util import dev, empty, handle

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
import paper_1412_4825_b200 as B  # noqa: E402

SEED, STREAM = 0x5EED5EED, 12


def _span(kind, n, dtype=None, k=None):
    if kind in ("uniform", "gaussian", "exponential", "weibull", "log_uniform"):
        return (n + 3) // 4 if dtype == np.float32 else (n + 1) // 2
    if kind == "laplace":
        return (n + 1) // 2 if dtype == np.float32 else n
    if kind == "gamma":
        return 256 * n
    if kind == "dirichlet":
        return 256 * n * k
    raise ValueError(kind)


def _fill(h, kind, n, dtype, rng, cursor):
    td = torch.float32 if dtype == np.float32 else torch.float64
    sfx = "f32" if dtype == np.float32 else "f64"
    off = int(rng.integers(0, 2))
    if kind == "log_uniform":
        out = empty(n, td, off)
        getattr(B, f"brng_log_uniform_{sfx}")(h, out, n)
        ref, scale = parity.fill_reference("log_uniform", SEED, STREAM, cursor, [n], 0, dtype)
        return out, ref, scale
    lo = np.exp(rng.uniform(-3, 3, n))
    if kind == "uniform":
        a = rng.uniform(-5, 5, n)
        params = [a, a + lo]
    elif kind == "gaussian":
        params = [rng.uniform(-5, 5, n), lo]
    elif kind == "exponential":
        params = [lo]
    elif kind == "laplace":
        params = [rng.uniform(-5, 5, n), lo]
    else:                                                  # weibull (shape, scale)
        params = [np.exp(rng.uniform(-1, 1, n)), lo]
    params = [p.astype(dtype) for p in params]
    dp = []
    for p in params:
        t = empty(n, td, off)
        t.copy_(torch.from_numpy(p))
        dp.append(t)
    out = empty(n, td, off)
    getattr(B, f"brng_{kind}_{sfx}")(h, *dp, out, n)
    ref, scale = parity.fill_reference(kind, SEED, STREAM, cursor, params, 0, dtype)
    return out, ref, scale


def test_random_call_sequence_matches_oracle():
    rng = np.random.default_rng(2014_12_15)
    kinds = ["uniform", "gaussian", "exponential", "laplace", "weibull", "log_uniform", "gamma",
             "dirichlet", "gibbs", "batch"]
    cursor = (1 << 32) - 3000
    with handle(SEED, STREAM, cursor) as h:
        for step in range(40):
            kind = kinds[int(rng.integers(0, len(kinds)))]
            n = int(rng.choice([1, 2, 3, 5, 31, 257, 1000, 4099, 20011]))
            dtype = np.float32 if rng.integers(0, 2) else np.float64
            assert B.brng_get_offset(h) == cursor, step
            if kind == "gamma":
                p = workloads.cfg3_params(n, seed=int(rng.integers(1, 1 << 30)))
                a = p["alpha"].numpy().astype(dtype); b = p["beta"].numpy().astype(dtype)
                td = torch.float32 if dtype == np.float32 else torch.float64
                g = torch.empty(n, dtype=td, device=dev())
                tr = torch.empty(n, dtype=torch.uint8, device=dev())
                fn = B.brng_gamma_f32 if dtype == np.float32 else B.brng_gamma_f64
                fn(h, torch.from_numpy(a).to(dev()), torch.from_numpy(b).to(dev()), g, n, tr)
                r = parity.gamma_compare(g, tr, a, b, SEED, STREAM, cursor, dtype=dtype)
                assert r["n_fail"] == 0 and r["n_tie"] == 0, (step, r)
                cursor += _span("gamma", n)
            elif kind == "dirichlet":
                k = int(rng.choice([1, 3, 64, 256]))
                rows = max(1, n // k)
                al = workloads.cfg4_params(rows, k, seed=int(rng.integers(1, 1 << 30)))
                al = al.numpy().astype(dtype)
                td = torch.float32 if dtype == np.float32 else torch.float64
                x = torch.empty(rows, k, dtype=td, device=dev())
                tr = torch.empty(rows, k, dtype=torch.uint8, device=dev())
                fn = B.brng_dirichlet_f32 if dtype == np.float32 else B.brng_dirichlet_f64
                fn(h, torch.from_numpy(al).to(dev()), rows, k, x, tr)
                r = parity.dirichlet_compare(x, tr, al, SEED, STREAM, cursor, dtype=dtype)
                assert r["n_fail"] == 0 and r["n_tie"] == 0, (step, r)
                cursor += _span("dirichlet", rows, k=k)
            elif kind == "gibbs":
                nc, ns = int(rng.integers(1, 600)), int(rng.integers(2, 40))
                ox = torch.empty(ns, nc, dtype=torch.float64, device=dev())
                st = torch.empty(5, nc, dtype=torch.float64, device=dev())
                B.brng_gibbs_triangle(h, nc, ns, None, None, 0, ox, None, st, None, None)
                ref = oracle.gibbs_triangle(SEED, STREAM, cursor, nc, ns)
                assert np.array_equal(ox.cpu().numpy(), ref["out_x"]), step
                assert np.array_equal(st.cpu().numpy(), ref["chain_stats"]), step
                cursor += ns
            elif kind == "batch":
                td = torch.float32 if dtype == np.float32 else torch.float64
                code = 0 if dtype == np.float32 else 1
                out = torch.empty(n, dtype=td, device=dev())
                B.brng_batch_fill(h, B.DIST["gaussian"], code, 2.0, 0.5, out, n)
                ref, scale = parity.fill_reference("gaussian", SEED, STREAM, cursor,
                                                   [np.full(n, 2.0, dtype), np.full(n, 0.5, dtype)],
                                                   0, dtype)
                parity.check_close(out, ref, scale, dtype, f"step {step} batch")
                cursor += _span("gaussian", n, dtype)
            else:
                out, ref, scale = _fill(h, kind, n, dtype, rng, cursor)
                parity.check_close(out, ref, scale, dtype, f"step {step} {kind}")
                cursor += _span(kind, n, dtype)
        assert B.brng_get_offset(h) == cursor
        assert B.brng_device_errors(h) == 0
