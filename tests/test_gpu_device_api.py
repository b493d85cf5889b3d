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


def test_fig1_user_gibbs_loop_matches_oracle_and_bulk(user_lib):
    nc, ns = 1024, 200
    ox = torch.empty(ns, nc, dtype=torch.float64, device=dev())
    oy = torch.empty_like(ox)
    assert user_lib.dev_gibbs(42, 0, 0, nc, ns, ox.data_ptr(), oy.data_ptr(), _s()) == 0
    r = oracle.gibbs_triangle(42, 0, 0, nc, ns)
    assert np.array_equal(ox.cpu().numpy(), r["out_x"])
    assert np.array_equal(oy.cpu().numpy(), r["out_y"])
