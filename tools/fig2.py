"""NEXT row N1: the paper's Fig. 2 experiment
re-run on one B200, binary64 like the paper's vd* calls (P:L7).

Columns, per distribution (GPU analogues of P:L79-85):
  batch        one fixed-parameter call (VSL-Batch): brng_batch_fill
  oaat_naive   one n=1 call per sample (VSL-OAAT, "n=1 is an extremely
               suboptimal scenario"): the same kernel launched per sample
  brng         per-sample parameters read from memory (BatchRNG OAAT):
               the fused per-sample kernels of this library
  two_pass     BatchRNG with a materialised buffer: standard deviates written
               to HBM by brng, then a separate transform pass (torch elementwise)
  torch        the closest stock PyTorch call with per-sample parameters, if any
The speedup column is oaat_naive / brng, as in Fig. 2.  Parameters are read
from HBM arrays; outputs go to HBM.  Gamma "batch" passes constant
parameter arrays (the Gamma kernel has no scalar mode; it is ALU-bound).

usage: python tools/fig2.py [--n 2^27] > profiles/r01_fig2.json
"""
import argparse
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1412_4825_b200 as B  # noqa: E402


def timed(fn, reps=5):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        best = min(best, ev[0].elapsed_time(ev[1]))
    return best * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 27)
    ap.add_argument("--oaat", type=int, default=20000)
    args = ap.parse_args()
    n = args.n
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(1412)
    f64 = torch.float64

    def U(lo, hi):
        return lo + (hi - lo) * torch.rand(n, generator=g, dtype=f64, device=dev)

    def LU(lo, hi):
        return torch.exp(math.log(lo) + torch.rand(n, generator=g, dtype=f64, device=dev)
                         * (math.log(hi) - math.log(lo)))

    a = U(-1, 0)
    params = {
        "uniform": (a, a + LU(1e-3, 1e3)),
        "gaussian": (U(-10, 10), LU(1e-3, 1e3)),
        "exponential": (LU(1e-3, 1e3), None),
        "laplace": (U(-10, 10), LU(1e-3, 1e3)),
        "weibull": (LU(0.5, 5), LU(0.1, 10)),
        "gamma": (U(2, 3), LU(0.1, 10)),
    }
    fixed = {"uniform": (0.0, 2.0), "gaussian": (1.0, 3.0), "exponential": (2.0, 0.0),
             "laplace": (0.0, 2.0), "weibull": (2.0, 1.0), "gamma": (2.5, 2.0)}
    out = torch.empty(n, dtype=f64, device=dev)
    buf = torch.empty(n, dtype=f64, device=dev)
    h = B.brng_create(1412, 0)
    B.brng_set_cuda_stream(h, torch.cuda.current_stream().cuda_stream)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    rows = {}
    for dist, (p0, p1) in params.items():
        r = {}
        np_ = 1 if p1 is None else 2
        # batch (fixed parameters)
        if dist == "gamma":
            ca = torch.full((n,), fixed[dist][0], dtype=f64, device=dev)
            cb = torch.full((n,), fixed[dist][1], dtype=f64, device=dev)
            t = timed(lambda: B.brng_gamma_f64(h, ca, cb, out, n, None))
        else:
            t = timed(lambda: B.brng_batch_fill(h, B.DIST[dist], 1, fixed[dist][0],
                                                fixed[dist][1], out, n))
        r["batch"] = t
        # OAAT naive: one launch per sample
        k = args.oaat
        if dist == "gamma":
            def oaat():
                for i in range(k):
                    B.brng_gamma_f64(h, ca[i:i + 1], cb[i:i + 1], out[i:i + 1], 1, None)
        else:
            def oaat():
                for i in range(k):
                    B.brng_batch_fill(h, B.DIST[dist], 1, float(fixed[dist][0]),
                                      float(fixed[dist][1]), out[i:i + 1], 1)
        r["oaat_naive"] = timed(oaat, reps=2) * n / k
        # fused per-sample parameters
        fn = getattr(B, f"brng_{dist}_f64")
        if dist == "gamma":
            t = timed(lambda: fn(h, p0, p1, out, n, None))
        elif np_ == 1:
            t = timed(lambda: fn(h, p0, out, n))
        else:
            t = timed(lambda: fn(h, p0, p1, out, n))
        r["brng"] = t
        # two-pass: standard deviates to HBM, then a separate transform pass
        if dist in ("uniform", "gaussian", "exponential"):
            if dist == "uniform":
                def std():
                    B.brng_std_uniform_f64(h, buf, n)

                def xf():
                    torch.addcmul(p0, p1 - p0, buf, out=out)
            elif dist == "gaussian":
                zeros = torch.zeros(n, dtype=f64, device=dev)
                ones = torch.ones(n, dtype=f64, device=dev)

                def std():
                    B.brng_gaussian_f64(h, zeros, ones, buf, n)

                def xf():
                    torch.addcmul(p0, p1, buf, out=out)
            else:
                def std():
                    B.brng_log_uniform_f64(h, buf, n)

                def xf():
                    torch.div(buf, p0, out=out).neg_()
            r["two_pass"] = timed(lambda: (std(), xf()))
        # stock torch with per-sample parameters
        if dist == "gaussian":
            r["torch"] = timed(lambda: torch.normal(p0, p1, generator=g, out=out))
        elif dist == "gamma":
            r["torch"] = timed(lambda: torch.mul(torch._standard_gamma(p0), p1, out=out))
        elif dist == "uniform":
            r["torch"] = timed(lambda: torch.addcmul(p0, p1 - p0,
                                                     torch.rand(n, generator=g, dtype=f64,
                                                                device=dev), out=out))
        # rates
        res = {m: {"ns_per_sample": round(t / n * 1e9, 5), "Gsamples_per_s": round(n / t / 1e9, 3)}
               for m, t in r.items()}
        bytes_fused = (np_ + 1) * 8
        res["brng"]["GB_per_s"] = round(bytes_fused * n / r["brng"] / 1e9, 1)
        res["brng"]["hbm_frac"] = round(res["brng"]["GB_per_s"] / peaks["hbm_gbs"], 4)
        res["batch"]["GB_per_s"] = round(8 * n / r["batch"] / 1e9, 1)
        res["speedup_oaat_over_brng"] = round(r["oaat_naive"] / r["brng"], 1)
        res["brng_over_batch_time"] = round(r["brng"] / r["batch"], 3)
        rows[dist] = res
    B.brng_destroy(h)
    print(json.dumps({"n": n, "dtype": "f64", "device": torch.cuda.get_device_name(0),
                      "rows": rows}))


if __name__ == "__main__":
    main()
