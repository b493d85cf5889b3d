"""Probe the host-buffer (e2e) path's timing variance: times each row group of
bench.py's e2e step alone, and individual host-staged calls, several times in
one process (wall clock between synchronisations).

usage: python tools/e2e_probe.py [reps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1412_4825_b200 as B  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    torch.cuda.set_device(0)
    wl = bench.Workload(0, 1, torch, B)
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    hp2 = {k: pin(v) for k, v in wl.p2.items()}
    hp3 = {k: pin(v) for k, v in wl.p3.items()}
    hp4 = pin(wl.p4)
    o2 = torch.empty_like(hp2["mu"]).pin_memory()
    o3 = torch.empty_like(hp3["alpha"]).pin_memory()
    o4 = torch.empty_like(hp4).pin_memory()
    c5 = wl.c5
    st5 = torch.empty(5, c5["n_chains"], dtype=torch.float64).pin_memory()
    fx5 = torch.empty(2, c5["n_chains"], dtype=torch.float64).pin_memory()
    tot5 = torch.empty(B.TOTALS_LEN, dtype=torch.float64).pin_memory()
    n2, n3 = hp2["mu"].numel(), hp3["alpha"].numel()
    D, K = hp4.shape
    calls = {
        "gaussian_host": lambda: B.brng_gaussian_f32(wl.h2, hp2["mu"], hp2["sigma"], o2, n2),
        "gamma_host": lambda: B.brng_gamma_f64(wl.h3, hp3["alpha"], hp3["beta"], o3, n3, None),
        "dirichlet_host": lambda: B.brng_dirichlet_f32(wl.h4, hp4, D, K, o4, None),
        "gibbs5_host": lambda: B.brng_gibbs_triangle(wl.h5, c5["n_chains"], c5["n_sweeps"], None,
                                                     None, 0, None, None, st5, fx5, tot5),
        "h2d_2GB": lambda: wl.p2["mu"].copy_(hp2["mu"], non_blocking=True),
        "d2h_1GB": lambda: o2.copy_(wl.o2g, non_blocking=True),
    }
    for name, fn in calls.items():
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t) * 1e3)
        print(f"{name:16s} " + " ".join(f"{x:8.2f}" for x in ts) + " ms", flush=True)




def repeat_e2e(n):
    """bench.e2e_run n times in one process with nvidia-smi clocks sampled."""
    import argparse
    torch.cuda.set_device(0)
    wl = bench.Workload(0, 1, torch, B)
    args = argparse.Namespace(steps=2, e2e_steps=2)
    for r in range(n):
        ck = bench.Clocks(0)
        ck.start()
        e = bench.e2e_run(wl, torch, B, args, None, 1, None)
        c = ck.stop()
        print(f"e2e {r}: {e['ms_per_step']:8.1f} ms/step  serial {e['serial_ms_per_step']:8.1f}"
              f"  gibbs {e['gibbs_rows_alone_ms']:7.1f}  io {e['io_rows_alone_ms']:7.1f}  clocks {c}",
              flush=True)


def repeat_gibbs(n):
    """cfg5 Gibbs n times, device buffers and host buffers alternately, with
    CUDA-event kernel time and wall time, to locate outliers."""
    torch.cuda.set_device(0)
    wl = bench.Workload(0, 1, torch, B)
    c5 = wl.c5
    st_h = torch.empty(5, c5["n_chains"], dtype=torch.float64).pin_memory()
    fx_h = torch.empty(2, c5["n_chains"], dtype=torch.float64).pin_memory()
    tot_h = torch.empty(B.TOTALS_LEN, dtype=torch.float64).pin_memory()
    st_d = torch.empty(5, c5["n_chains"], dtype=torch.float64, device="cuda")
    fx_d = torch.empty(2, c5["n_chains"], dtype=torch.float64, device="cuda")
    tot_d = torch.empty(B.TOTALS_LEN, dtype=torch.float64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(n):
        for kind, (st, fx, tot) in (("dev", (st_d, fx_d, tot_d)), ("host", (st_h, fx_h, tot_h))):
            B.brng_set_offset(wl.h5, 0)
            torch.cuda.synchronize()
            t = time.perf_counter()
            e0.record()
            B.brng_gibbs_triangle(wl.h5, c5["n_chains"], c5["n_sweeps"], None, None, 0, None,
                                  None, st, fx, tot)
            e1.record()
            torch.cuda.synchronize()
            w = (time.perf_counter() - t) * 1e3
            print(f"{r:3d} {kind:4s} wall {w:8.1f} ms  events {e0.elapsed_time(e1):8.1f} ms",
                  flush=True)


def repeat_copies(n):
    """D2H / H2D copy bandwidth to pinned memory, n repetitions (outlier hunt)."""
    torch.cuda.set_device(0)
    d = torch.empty(7 << 27, dtype=torch.float64, device="cuda")          # 7.5 GB... / 8
    d = d[: (940 << 20) // 8]
    h = torch.empty(d.numel(), dtype=torch.float64).pin_memory()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(n):
        for kind in ("d2h", "h2d"):
            torch.cuda.synchronize()
            e0.record()
            if kind == "d2h":
                h.copy_(d, non_blocking=True)
            else:
                d.copy_(h, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            print(f"{r:3d} {kind} {ms:8.2f} ms  {h.numel() * 8 / ms / 1e6:6.1f} GB/s", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "e2e":
        repeat_e2e(int(sys.argv[1]))
    elif len(sys.argv) > 2 and sys.argv[2] == "copies":
        repeat_copies(int(sys.argv[1]))
    elif len(sys.argv) > 2 and sys.argv[2] == "gibbs":
        repeat_gibbs(int(sys.argv[1]))
    else:
        main()


