"""Time the Gibbs latency-mode launch (chain/helper warp pairs) at a few chain
counts and output options (1000 sweeps).  usage: python tools/lat_probe.py
[n_chains ...]; BRNG_LIB selects a build variant."""
import sys, torch
sys.path.insert(0, '.')
import paper_1412_4825_b200 as B
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
import os
ns = int(os.environ.get("NS", 1000))
for nc in [int(x) for x in (sys.argv[1:] or "148 592 1024".split())]:
    for store, totals in ((True, True), (False, True), (False, False)):
        ox = torch.empty(ns, nc, dtype=torch.float64, device=dev) if store else None
        oy = torch.empty_like(ox) if store else None
        tot = torch.empty(B.TOTALS_LEN, dtype=torch.float64, device=dev) if totals else None
        h = B.brng_create(42, 0); B.brng_set_cuda_stream(h, s)
        def run():
            B.brng_set_offset(h, 0)
            B.brng_gibbs_triangle(h, nc, ns, None, None, 0, ox, oy, None, None, tot)
        run(); torch.cuda.synchronize()
        if os.environ.get("WARM"):          # keep the SM clock up (idle GPUs clock down)
            m = torch.randn(8192, 8192, device=dev)
            for _ in range(30):
                m = m @ m
                m = m / m.abs().max()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(5):
            e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        print(f"chains {nc:5d} store {int(store)} totals {int(totals)}: {min(ts) * 1000:6.1f} us")
        B.brng_destroy(h)
