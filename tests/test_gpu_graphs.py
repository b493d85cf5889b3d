"""The C-ABI calls are capturable into a CUDA graph (torch.cuda.graph): every
launch is stream-ordered, with no allocation or synchronisation on the
device-pointer path once the handle's scratch exists.  A replayed graph
reproduces the eager results bit for bit (the cursor a call consumed at
capture is baked into its kernel arguments)."""
import pytest
import torch

import workloads

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
import paper_1412_4825_b200 as B  # noqa: E402


def _step(h, bufs):
    p2, p3, p4 = bufs["p2"], bufs["p3"], bufs["p4"]
    B.brng_set_offset(h, 0)
    B.brng_gaussian_f32(h, p2["mu"], p2["sigma"], bufs["g"], bufs["g"].numel())
    B.brng_gamma_f64(h, p3["alpha"], p3["beta"], bufs["gam"], bufs["gam"].numel(), None)
    B.brng_dirichlet_f32(h, p4, p4.shape[0], p4.shape[1], bufs["dir"], None)
    B.brng_gibbs_triangle(h, 256, 100, None, None, 0, bufs["ox"], bufs["oy"], None, None,
                          bufs["tot1"])
    B.brng_gibbs_triangle(h, 200_000, 6, None, None, 0, None, None, bufs["st"], bufs["fx"],
                          bufs["tot5"])


def test_graph_replay_equals_eager():
    dev = torch.device("cuda:0")
    f64 = dict(dtype=torch.float64, device=dev)
    bufs = dict(p2=workloads.cfg2_params(10_007, seed=7, device=dev),
                p3=workloads.cfg3_params(30_011, seed=11, device=dev),
                p4=workloads.cfg4_params(33, 256, seed=3, device=dev),
                g=torch.empty(10_007, device=dev), gam=torch.empty(30_011, **f64),
                dir=torch.empty(33, 256, device=dev), ox=torch.empty(100, 256, **f64),
                oy=torch.empty(100, 256, **f64), tot1=torch.empty(B.TOTALS_LEN, **f64),
                st=torch.empty(5, 200_000, **f64), fx=torch.empty(2, 200_000, **f64),
                tot5=torch.empty(B.TOTALS_LEN, **f64))
    outs = ("g", "gam", "dir", "ox", "oy", "tot1", "st", "fx", "tot5")
    s = torch.cuda.Stream()
    h = B.brng_create(123, 4)
    try:
        with torch.cuda.stream(s):
            B.brng_set_cuda_stream(h, s.cuda_stream)
            _step(h, bufs)                         # eager (also allocates the scratch)
            s.synchronize()
            eager = {k: bufs[k].clone() for k in outs}
            for k in outs:
                bufs[k].fill_(-1.0)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                _step(h, bufs)
            for k in outs:
                bufs[k].fill_(-1.0)
            for _ in range(2):
                graph.replay()
            s.synchronize()
            for k in outs:
                assert torch.equal(bufs[k], eager[k]), k
            assert B.brng_device_errors(h) == 0
    finally:
        B.brng_destroy(h)


def test_graph_survives_scratch_growth():
    """A graph captured with a large-K binary32 Dirichlet (handle scratch rows)
    stays valid after a later eager call on the same handle grows that scratch
    (the old buffer is retired, not freed), and a capture never allocates."""
    dev = torch.device("cuda:0")
    a1 = workloads.cfg4_params(40, 2048, seed=3, device=dev)
    a2 = workloads.cfg4_params(20, 4096, seed=4, device=dev)
    o1 = torch.empty(40, 2048, device=dev)
    o2 = torch.empty(20, 4096, device=dev)
    s = torch.cuda.Stream()
    h = B.brng_create(5, 0)
    try:
        with torch.cuda.stream(s):
            B.brng_set_cuda_stream(h, s.cuda_stream)
            B.brng_set_offset(h, 0)
            B.brng_dirichlet_f32(h, a1, 40, 2048, o1, None)      # eager: scratch for K = 2048
            s.synchronize()
            eager = o1.clone()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                B.brng_set_offset(h, 0)
                B.brng_dirichlet_f32(h, a1, 40, 2048, o1, None)
            B.brng_dirichlet_f32(h, a2, 20, 4096, o2, None)      # eager: grows the scratch
            s.synchronize()
            o1.fill_(-1.0)
            graph.replay()
            s.synchronize()
            assert torch.equal(o1, eager)
            # a capture that would need more scratch recomputes the rows instead
            g2 = torch.cuda.CUDAGraph()
            a3 = workloads.cfg4_params(8, 8192, seed=5, device=dev)
            o3 = torch.empty(8, 8192, device=dev)
            with torch.cuda.graph(g2, stream=s):
                B.brng_set_offset(h, 0)
                B.brng_dirichlet_f32(h, a3, 8, 8192, o3, None)
            g2.replay()
            s.synchronize()
            B.brng_set_offset(h, 0)
            ref = torch.empty_like(o3)
            B.brng_dirichlet_f32(h, a3, 8, 8192, ref, None)      # eager, with scratch
            s.synchronize()
            torch.testing.assert_close(o3, ref, rtol=2e-6, atol=0)
            assert B.brng_device_errors(h) == 0
    finally:
        B.brng_destroy(h)
