"""Multi-process (gloo, world_size 2, CPU) tests of the sharding host logic
and the totals reduction (paper_1412_4825_b200/shard.py).  Each rank computes
its shard with the CPU ORACLE as the stand-in compute (no GPU here) using the
shard helpers' counters; the reduced / gathered result must equal an
unsharded run bit for bit (histogram) or within 1e-12 (moment sums)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads
from paper_1412_4825_b200 import shard

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # Gibbs: chains sharded by stream range, totals all-reduced
        n_chains, n_sweeps = 3001, 64
        lo, hi = shard.shard_range(n_chains, rank, world)
        r = oracle.gibbs_triangle(42, shard.gibbs_stream(0, lo), 0, hi - lo, n_sweeps,
                                  want_samples=False)
        tot = torch.from_numpy(r["totals"].copy())
        shard.reduce_totals(tot)
        # Gamma: samples sharded by cursor
        n = 1001
        p = workloads.cfg3_params(n, seed=11)
        glo, ghi = shard.shard_range(n, rank, world)
        g, tr, _ = oracle.gamma(11, 0, shard.gamma_cursor(0, glo), p["alpha"][glo:ghi].numpy(),
                                p["beta"][glo:ghi].numpy())
        # f32 fill: shards aligned to Philox blocks (4 samples)
        nf = 1003
        fp = workloads.cfg2_params(nf, seed=7)
        flo, fhi = shard.shard_range(nf, rank, world, align=4)
        f, _ = oracle.gaussian(7, 0, shard.fill_cursor(0, flo, 4), fp["mu"][flo:fhi].numpy(),
                               fp["sigma"][flo:fhi].numpy())
        # Dirichlet rows
        D, K = 37, 16
        al = workloads.cfg4_params(D, K, seed=3)
        dlo, dhi = shard.shard_range(D, rank, world)
        x, _, _ = oracle.dirichlet(3, 0, shard.dirichlet_cursor(0, dlo, K), al[dlo:dhi].numpy())
        parts = [None] * world
        dist.all_gather_object(parts, dict(stats=r["chain_stats"], g=g, f=f, x=x))
        q.put((rank, tot.numpy(), parts))
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def gloo_results():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda t: t[0])


def test_gibbs_totals_allreduce_equals_unsharded(gloo_results):
    whole = oracle.gibbs_triangle(42, 0, 0, 3001, 64, want_samples=False)
    for rank, tot, parts in gloo_results:
        assert np.array_equal(tot[16:], whole["totals"][16:])          # histogram exact
        np.testing.assert_allclose(tot[:16], whole["totals"][:16], rtol=1e-12)
        stats = np.concatenate([p["stats"] for p in parts], axis=1)
        assert np.array_equal(stats, whole["chain_stats"])
    st = shard.pooled_stats(gloo_results[0][1])
    assert st["n_chains"] == 3001 and st["n_samples"] == 3001 * 64
    assert abs(sum(st["hist_prob"]) - 1) < 1e-12


def test_sample_shards_equal_unsharded(gloo_results):
    parts = gloo_results[0][2]
    p = workloads.cfg3_params(1001, seed=11)
    g, _, _ = oracle.gamma(11, 0, 0, p["alpha"].numpy(), p["beta"].numpy())
    assert np.array_equal(np.concatenate([q["g"] for q in parts]), g)
    fp = workloads.cfg2_params(1003, seed=7)
    f, _ = oracle.gaussian(7, 0, 0, fp["mu"].numpy(), fp["sigma"].numpy())
    assert np.array_equal(np.concatenate([q["f"] for q in parts]), f)
    al = workloads.cfg4_params(37, 16, seed=3)
    x, _, _ = oracle.dirichlet(3, 0, 0, al.numpy())
    assert np.array_equal(np.concatenate([q["x"] for q in parts]), x)


def test_shard_range_properties():
    for n in (0, 1, 5, 1003, 1 << 20):
        for world in (1, 2, 3, 8):
            for align in (1, 2, 4):
                cov = []
                for r in range(world):
                    lo, hi = shard.shard_range(n, r, world, align)
                    assert lo <= hi and (lo % align == 0 or lo == n)
                    cov.extend(range(lo, hi)) if n < 5000 else None
                if n < 5000:
                    assert cov == list(range(n))
    with pytest.raises(ValueError):
        shard.fill_cursor(0, 3, 4)
    assert shard.gamma_cursor(10, 3) == 10 + 768
    assert shard.dirichlet_cursor(0, 2, 256) == 2 * 256 * 256
