"""Time Dirichlet rows at several K (f64 and f32 output), ~2^27 components
each.  usage: python tools/dirichlet_k.py K [K ...]; BRNG_LIB selects a build."""
import sys, torch
sys.path.insert(0, '.')
import paper_1412_4825_b200 as B, workloads as W
dev = torch.device("cuda:0"); s = torch.cuda.current_stream().cuda_stream
for K in [int(k) for k in sys.argv[1:]]:
    D = (1 << 27) // K
    a = W.cfg4_params(D, K, seed=3, device=dev, dtype=torch.float64)
    for dt in (torch.float64, torch.float32):
        al = a.to(dt); o = torch.empty(D, K, dtype=dt, device=dev)
        h = B.brng_create(3, 0); B.brng_set_cuda_stream(h, s)
        fn = B.brng_dirichlet_f64 if dt == torch.float64 else B.brng_dirichlet_f32
        fn(h, al, D, K, o, None); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(3):
            B.brng_set_offset(h, 0); e0.record(); fn(h, al, D, K, o, None); e1.record()
            torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        print(f"K={K:5d} {str(dt):14s} {min(ts):7.3f} ms")
        B.brng_destroy(h)
