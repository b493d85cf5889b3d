"""Small calls of every C-ABI entry point, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck, one tool per run):
    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
Covers the vector and scalar (misaligned) fill paths, Gamma with the boost
queue, both Dirichlet kernels, both Gibbs launch shapes, the host-staging
pipeline and the fixed-parameter batch fill."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1412_4825_b200 as B  # noqa: E402
import workloads  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    h = B.brng_create(5, 1)
    B.brng_set_cuda_stream(h, torch.cuda.current_stream().cuda_stream)
    n = 1029
    for td, sfx in ((torch.float32, "f32"), (torch.float64, "f64")):
        for off in (0, 1):
            mk = lambda: torch.rand(n + off, dtype=td, device=dev)[off:]  # noqa: E731
            a, b, o = mk(), mk() + 1.0, torch.empty(n + off, dtype=td, device=dev)[off:]
            getattr(B, f"brng_uniform_{sfx}")(h, a, b, o, n)
            getattr(B, f"brng_gaussian_{sfx}")(h, a, b, o, n)
            getattr(B, f"brng_exponential_{sfx}")(h, b, o, n)
            getattr(B, f"brng_laplace_{sfx}")(h, a, b, o, n)
            getattr(B, f"brng_weibull_{sfx}")(h, b, b, o, n)
            getattr(B, f"brng_log_uniform_{sfx}")(h, o, n)
            getattr(B, f"brng_std_uniform_{sfx}")(h, o, n)
            B.brng_batch_fill(h, 3, 0 if sfx == "f32" else 1, 1.0, 2.0, o, n)
        p = workloads.cfg3_params(n, seed=1, device=dev, dtype=td)
        g = torch.empty(n, dtype=td, device=dev)
        tr = torch.empty(n, dtype=torch.uint8, device=dev)
        getattr(B, f"brng_gamma_{sfx}")(h, p["alpha"], p["beta"], g, n, tr)
        for rows, k in ((37, 64), (3, 2100)):
            al = workloads.cfg4_params(rows, k, seed=2, device=dev, dtype=td)
            x = torch.empty(rows, k, dtype=td, device=dev)
            getattr(B, f"brng_dirichlet_{sfx}")(h, al, rows, k, x, None)
    raw = torch.empty(n, dtype=torch.int32, device=dev)
    B.brng_raw_u32(h, raw, n)
    f = lambda *s: torch.empty(*s, dtype=torch.float64, device=dev)  # noqa: E731
    B.brng_gibbs_triangle(h, 300, 20, None, None, 5, f(20, 300), f(20, 300), f(5, 300),
                          f(2, 300), f(272))
    B.brng_gibbs_triangle(h, 200_000, 8, None, None, 0, None, None, f(5, 200_000),
                          f(2, 200_000), f(272))
    hp = np.random.rand(n)
    ho = np.empty(n)
    B.brng_gaussian_f64(h, hp, hp + 1.0, ho, n)
    B.brng_gibbs_triangle(h, 500, 10, None, None, 0, None, None, np.empty((5, 500)),
                          np.empty((2, 500)), np.empty(272))
    torch.cuda.synchronize()
    errs = B.brng_device_errors(h)
    B.brng_destroy(h)
    print("sanitize smoke ok, device_errors", errs)


if __name__ == "__main__":
    main()
