"""Time build variants of libbrng (tools/variants/*.so) on one kernel.

usage: python tools/variant_time.py gibbs|gibbs1|gamma|gamma32|dirichlet|gaussian|uniform|exponential [lib ...]
Each variant runs in its own process (BRNG_LIB=...); prints ms and a hash of
the outputs so variants can be checked for identical results.
"""
import glob
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import hashlib, json, sys, torch
sys.path.insert(0, ROOT)
import paper_1412_4825_b200 as B, workloads as W
what = WHAT
dev = torch.device("cuda:0")
s = torch.cuda.current_stream().cuda_stream
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if what == "gibbs1":
    nc, ns = 1024, 1000
    ox = torch.empty(ns, nc, dtype=torch.float64, device=dev)
    oy = torch.empty_like(ox)
    tot = torch.empty(B.TOTALS_LEN, dtype=torch.float64, device=dev)
    h = B.brng_create(42, 0); B.brng_set_cuda_stream(h, s)
    def run():
        B.brng_set_offset(h, 0)
        B.brng_gibbs_triangle(h, nc, ns, None, None, 0, ox, oy, None, None, tot)
    outs = [ox, oy, tot[16:]]
elif what == "gibbs":
    import os
    nc, ns = int(os.environ.get("GIBBS_NC", 1 << 24)), 4096
    st = torch.empty(5, nc, dtype=torch.float64, device=dev)
    fx = torch.empty(2, nc, dtype=torch.float64, device=dev)
    tot = torch.empty(B.TOTALS_LEN, dtype=torch.float64, device=dev)
    h = B.brng_create(42, 0); B.brng_set_cuda_stream(h, s)
    def run():
        B.brng_set_offset(h, 0)
        B.brng_gibbs_triangle(h, nc, ns, None, None, 0, None, None, st, fx, tot)
    outs = [st, fx, tot[16:]]
elif what == "gamma32":
    n = 1 << 26
    p = W.cfg3_params(n, seed=11, device=dev)
    a32, b32 = p["alpha"].float(), p["beta"].float()
    o = torch.empty(n, dtype=torch.float32, device=dev)
    h = B.brng_create(11, 0); B.brng_set_cuda_stream(h, s)
    def run():
        B.brng_set_offset(h, 0)
        B.brng_gamma_f32(h, a32, b32, o, n, None)
    outs = [o]
elif what == "gamma":
    n = 1 << 26
    p = W.cfg3_params(n, seed=11, device=dev)
    o = torch.empty(n, dtype=torch.float64, device=dev)
    h = B.brng_create(11, 0); B.brng_set_cuda_stream(h, s)
    def run():
        B.brng_set_offset(h, 0)
        B.brng_gamma_f64(h, p["alpha"], p["beta"], o, n, None)
    outs = [o]
elif what == "exponential":
    n = 1 << 28
    lam = W.exp_params(n, seed=7, device=dev)
    o = torch.empty(n, device=dev)
    h = B.brng_create(7, 5); B.brng_set_cuda_stream(h, s)
    def run():
        B.brng_set_offset(h, 0)
        B.brng_exponential_f32(h, lam, o, n)
    outs = [o]
elif what in ("gaussian", "uniform"):
    n = 1 << 28
    p = W.cfg2_params(n, seed=7, device=dev)
    o = torch.empty(n, device=dev)
    h = B.brng_create(7, 0); B.brng_set_cuda_stream(h, s)
    k0, k1 = ("mu", "sigma") if what == "gaussian" else ("a", "b")
    fn = getattr(B, f"brng_{what}_f32")
    def run():
        B.brng_set_offset(h, 0)
        fn(h, p[k0], p[k1], o, n)
    outs = [o]
else:
    D, K = 1000000, 256
    a = W.cfg4_params(D, K, seed=3, device=dev)
    o = torch.empty(D, K, device=dev)
    h = B.brng_create(3, 0); B.brng_set_cuda_stream(h, s)
    def run():
        B.brng_set_offset(h, 0)
        B.brng_dirichlet_f32(h, a, D, K, o, None)
    outs = [o]
run(); torch.cuda.synchronize()
ts = []
for _ in range(3):
    ev0.record(); run(); ev1.record(); torch.cuda.synchronize(); ts.append(ev0.elapsed_time(ev1))
hh = hashlib.sha1()
for t in outs: hh.update(t.cpu().numpy().tobytes())
print(json.dumps({"ms": min(ts), "hash": hh.hexdigest()[:12]}))
'''


def main():
    what = sys.argv[1]
    libs = sys.argv[2:] or sorted(glob.glob(os.path.join(ROOT, "tools", "variants", "*.so")))
    for lib in libs:
        env = dict(os.environ, BRNG_LIB=lib)
        code = CHILD.replace("ROOT", repr(ROOT)).replace("WHAT", repr(what))
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
        print(f"{os.path.basename(lib):28s} {line}", flush=True)


if __name__ == "__main__":
    main()
