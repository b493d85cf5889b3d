"""Two-process strong-scaling check on one GPU (VERDICT r01
"Next round" item 4): world size 2 over gloo, both ranks on cuda:0, each rank
running ITS shard of every config through libbrng (paper_1412_4825_b200/
shard.py counter ranges) and the Gibbs totals summed with the hot path's one
collective (shard.reduce_totals).  The gathered shards must equal a
one-process run: samples, Dirichlet rows, per-chain statistics, final states
and the histogram bit for bit; the moment totals within 1e-12 (their
summation order depends on the sharding).

The two processes are independent (no kernel waits on the other rank), so
running them on one GPU is a valid test of the N > 1 host path."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

NC5, NS5 = 300_007, 24           # > one bulk wave: full rounds + one-chain tail rounds
N2, N3 = 1_000_003, 200_003
D4, K4 = 3001, 256


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_shard(rank, world, out_dir):
    """Rank `rank` of `world` computes its shard of every config."""
    import paper_1412_4825_b200 as B
    import workloads as W
    from paper_1412_4825_b200 import shard as S
    dev = torch.device("cuda:0")
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream().cuda_stream
    res = {}
    # cfg5-shaped Gibbs: chain range, stream = first chain
    lo, hi = S.shard_range(NC5, rank, world)
    st = torch.empty(5, hi - lo, dtype=torch.float64, device=dev)
    fx = torch.empty(2, hi - lo, dtype=torch.float64, device=dev)
    tot = torch.empty(B.TOTALS_LEN, dtype=torch.float64, device=dev)
    h = B.brng_create(42, S.gibbs_stream(0, lo))
    B.brng_set_cuda_stream(h, s)
    B.brng_gibbs_triangle(h, hi - lo, NS5, None, None, 0, None, None, st, fx, tot)
    torch.cuda.synchronize()
    B.brng_destroy(h)
    tot_cpu = tot.cpu()
    S.reduce_totals(tot_cpu)                       # the one collective (gloo here)
    res["st"], res["fx"], res["tot"] = st.cpu().numpy(), fx.cpu().numpy(), tot_cpu.numpy()
    # cfg2-shaped Gaussian fill: sample range on Philox-block boundaries
    lo, hi = S.shard_range(N2, rank, world, align=4)
    p2 = W.cfg2_params(N2, seed=7, device=dev)
    g = torch.empty(hi - lo, device=dev)
    h = B.brng_create(7, 0)
    B.brng_set_cuda_stream(h, s)
    B.brng_set_offset(h, S.fill_cursor(0, lo, 4))
    B.brng_gaussian_f32(h, p2["mu"][lo:hi].contiguous(), p2["sigma"][lo:hi].contiguous(), g,
                        hi - lo)
    torch.cuda.synchronize()
    B.brng_destroy(h)
    res["g"] = g.cpu().numpy()
    # cfg3-shaped Gamma: sample range, cursor 256 lo
    lo, hi = S.shard_range(N3, rank, world)
    p3 = W.cfg3_params(N3, seed=11, device=dev)
    gm = torch.empty(hi - lo, dtype=torch.float64, device=dev)
    h = B.brng_create(11, 0)
    B.brng_set_cuda_stream(h, s)
    B.brng_set_offset(h, S.gamma_cursor(0, lo))
    B.brng_gamma_f64(h, p3["alpha"][lo:hi].contiguous(), p3["beta"][lo:hi].contiguous(), gm,
                     hi - lo, None)
    torch.cuda.synchronize()
    B.brng_destroy(h)
    res["gamma"] = gm.cpu().numpy()
    # cfg4-shaped Dirichlet: document range
    lo, hi = S.shard_range(D4, rank, world)
    a4 = W.cfg4_params(D4, K4, seed=3, device=dev)
    x = torch.empty(hi - lo, K4, device=dev)
    h = B.brng_create(3, 0)
    B.brng_set_cuda_stream(h, s)
    B.brng_set_offset(h, S.dirichlet_cursor(0, lo, K4))
    B.brng_dirichlet_f32(h, a4[lo:hi].contiguous(), hi - lo, K4, x, None)
    torch.cuda.synchronize()
    B.brng_destroy(h)
    res["dir"] = x.cpu().numpy()
    np.savez(os.path.join(out_dir, f"rank{rank}_of{world}.npz"), **res)


def _worker(rank, world, port, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _run_shard(rank, world, out_dir)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_ranks_equal_one_process(tmp_path):
    import torch.multiprocessing as mp
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    _run_shard(0, 1, str(tmp_path))                  # the one-process run (no collective)
    one = np.load(tmp_path / "rank0_of1.npz")
    parts = [np.load(tmp_path / f"rank{r}_of2.npz") for r in range(2)]
    assert np.array_equal(np.concatenate([p["st"] for p in parts], axis=1), one["st"])
    assert np.array_equal(np.concatenate([p["fx"] for p in parts], axis=1), one["fx"])
    for k in ("g", "gamma", "dir"):
        assert np.array_equal(np.concatenate([p[k] for p in parts]), one[k]), k
    hdr = 16
    for p in parts:                                   # both ranks hold the reduced totals
        assert np.array_equal(p["tot"][hdr:], one["tot"][hdr:])
        np.testing.assert_allclose(p["tot"][:hdr], one["tot"][:hdr], rtol=1e-12, atol=0)
    assert one["tot"][8] == NC5 and one["tot"][hdr:].sum() == NC5 * NS5
