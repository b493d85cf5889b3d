"""GPU parity of K5-K7 (Gibbs chains on the triangle, per-chain statistics,
256-bin histogram, fixed-order reduction) against the CPU oracle.

Samples, final states, per-chain statistics and histogram counts are
BIT-EXACT; moment totals agree within 1e-12 (summation order differs).
cfg1 is checked in full; cfg5 (2^24 x 4096) on sampled chains plus
invariants and closed-form statistics.
"""
import math

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

HDR = B.TOTALS_HDR


def _run(seed, stream_id, cursor, n_chains, n_sweeps, burn_in=0, samples=True, x0=None, y0=None):
    f = lambda *s: torch.empty(*s, dtype=torch.float64, device=dev())  # noqa: E731
    ox = f(n_sweeps, n_chains) if samples else None
    oy = f(n_sweeps, n_chains) if samples else None
    st, fx, tot = f(5, n_chains), f(2, n_chains), f(B.TOTALS_LEN)
    with handle(seed, stream_id, cursor) as h:
        B.brng_gibbs_triangle(h, n_chains, n_sweeps, x0, y0, burn_in, ox, oy, st, fx, tot)
        assert B.brng_get_offset(h) == cursor + n_sweeps
        errs = B.brng_device_errors(h)
    cpu = lambda t: None if t is None else t.cpu().numpy()  # noqa: E731
    return dict(out_x=cpu(ox), out_y=cpu(oy), chain_stats=cpu(st), final_xy=cpu(fx),
                totals=cpu(tot), n_invalid=errs)


def _assert_match(g, r, samples=True):
    if samples:
        assert np.array_equal(g["out_x"], r["out_x"])
        assert np.array_equal(g["out_y"], r["out_y"])
    assert np.array_equal(g["chain_stats"], r["chain_stats"], equal_nan=True)
    assert np.array_equal(g["final_xy"], r["final_xy"], equal_nan=True)
    assert np.array_equal(g["totals"][HDR:], r["totals"][HDR:])          # histogram, exact
    np.testing.assert_allclose(g["totals"][:HDR], r["totals"][:HDR], rtol=1e-12, atol=1e-300,
                               equal_nan=True)


def test_cfg1_bit_exact():
    c = workloads.CFG1
    g = _run(c["seed"], 0, 0, c["n_chains"], c["n_sweeps"])
    r = oracle.gibbs_triangle(c["seed"], 0, 0, c["n_chains"], c["n_sweeps"])
    _assert_match(g, r)
    assert g["out_x"].size + g["out_y"].size == 2_048_000
    assert np.all(g["out_x"] + g["out_y"] < 1)


@pytest.mark.parametrize("n_chains,n_sweeps,burn", [(1, 1, 0), (37, 5, 2), (1000, 129, 64),
                                                    (70_001, 16, 3)])
def test_ragged_shapes_bit_exact(n_chains, n_sweeps, burn):
    g = _run(5, 1000, 7, n_chains, n_sweeps, burn)
    r = oracle.gibbs_triangle(5, 1000, 7, n_chains, n_sweeps, burn_in=burn)
    _assert_match(g, r)


def test_counter_carry_and_streams():
    # sweeps crossing the 2^32 block boundary; stream ids crossing 2^32
    g = _run(9, (1 << 32) - 3, (1 << 32) - 10, 64, 40)
    r = oracle.gibbs_triangle(9, (1 << 32) - 3, (1 << 32) - 10, 64, 40)
    _assert_match(g, r)


def test_chunk_invariance_and_start_states():
    whole = _run(42, 0, 0, 500, 300)
    a = _run(42, 0, 0, 500, 120)
    fx = torch.tensor(a["final_xy"], device=dev())
    b = _run(42, 0, 120, 500, 180, x0=fx[0].contiguous(), y0=fx[1].contiguous())
    assert np.array_equal(np.concatenate([a["out_x"], b["out_x"]]), whole["out_x"])
    assert np.array_equal(b["final_xy"], whole["final_xy"])


def test_invalid_start_state():
    y0 = torch.tensor([0.5, 1.5, float("nan"), 0.0], dtype=torch.float64, device=dev())
    g = _run(1, 0, 0, 4, 10, y0=y0)
    assert g["n_invalid"] == 2
    r = oracle.gibbs_triangle(1, 0, 0, 4, 10, y0=y0.cpu().numpy())
    assert np.array_equal(g["final_xy"], r["final_xy"], equal_nan=True)
    assert np.array_equal(g["totals"][HDR:], r["totals"][HDR:])


def test_host_buffers():
    g = _run(42, 0, 0, 300, 50)
    st = np.empty((5, 300)); fx = np.empty((2, 300)); tot = np.empty(B.TOTALS_LEN)
    ox = np.empty((50, 300))
    with handle(42) as h:
        B.brng_gibbs_triangle(h, 300, 50, None, None, 0, ox, None, st, fx, tot)
    assert np.array_equal(ox, g["out_x"]) and np.array_equal(st, g["chain_stats"])
    assert np.array_equal(tot, g["totals"])


def test_shards_reproduce_whole():
    # chains sharded by stream range (rank r: stream_id = r * n/G): identical
    n, G = 4096, 4
    whole = _run(42, 0, 0, n, 64, samples=False)
    hist = np.zeros(256)
    for r in range(G):
        part = _run(42, r * n // G, 0, n // G, 64, samples=False)
        lo, hi = r * n // G, (r + 1) * n // G
        assert np.array_equal(part["chain_stats"], whole["chain_stats"][:, lo:hi])
        hist += part["totals"][HDR:]
    assert np.array_equal(hist, whole["totals"][HDR:])


@pytest.mark.slow
def test_cfg5_full_size():
    c = workloads.CFG5
    nc, ns = c["n_chains"], c["n_sweeps"]
    g = _run(c["seed"], 0, 0, nc, ns, samples=False)
    assert g["n_invalid"] == 0
    tot = g["totals"]
    assert tot[HDR:].sum() == nc * ns and tot[8] == nc and tot[9] == nc * ns
    # sampled chains, bit-exact against the oracle
    rng = np.random.default_rng(5)
    for cidx in np.concatenate([[0, 1, nc - 1], rng.integers(0, nc, 200)]):
        r = oracle.gibbs_triangle(c["seed"], int(cidx), 0, 1, ns, want_samples=False)
        assert np.array_equal(g["chain_stats"][:, cidx], r["chain_stats"][:, 0]), cidx
        assert np.array_equal(g["final_xy"][:, cidx], r["final_xy"][:, 0]), cidx
    # cfg1 is the first 1024 chains over the first 1000 sweeps (same streams)
    # -> chain 0's final state after 1000 sweeps matches cfg1 (checked in cfg1 test)
    # transient-exact pooled means: 1/3 - (1-4^-n)/(9n), 1/3 + (1-4^-n)/(18n)
    ex = 1 / 3 - (1 - 4.0**-ns) / (9 * ns)
    ey = 1 / 3 + (1 - 4.0**-ns) / (18 * ns)
    sd = math.sqrt((5 / 3) * (1 / 18) / ns / nc)
    assert abs(tot[0] / nc - ex) < 6 * sd, (tot[0] / nc, ex)
    assert abs(tot[3] / nc - ey) < 6 * sd, (tot[3] / nc, ey)
    assert abs(tot[1] / nc - 1 / 18) < 1e-3 and abs(tot[6] / nc + 1 / 36) < 1e-3
    # every moment total equals its per-chain definition (R-18) summed over the
    # GPU's own chain statistics (bit-exact vs the oracle above) to 1e-12, and
    # the between-chain ones (totals[2], [5], [7]) meet their exact expectations
    # (tests/test_oracle_gibbs_moments.py)
    st = g["chain_stats"]
    mx, vx, my, vy, cxy = st
    for idx, v in ((0, mx), (1, vx), (2, mx * mx), (3, my), (4, vy), (5, my * my),
                   (6, cxy), (7, mx * my)):
        assert abs(tot[idx] - math.fsum(v)) <= 1e-12 * abs(math.fsum(v)), idx
    from tests.test_oracle_gibbs_moments import pin_failures
    assert pin_failures(tot, st, ns, 0) == []
    # final x of 2^24 chains ~ marginal CDF 2x - x^2 (KS)
    from tests.stats_util import assert_ks_uniform
    fxv = g["final_xy"][0]
    assert_ks_uniform(2 * fxv - fxv * fxv, "cfg5 final-x marginal")


@pytest.mark.slow
def test_cfg5_strong_scaling_shard_full_size():
    """The bench's N = 8 launch configuration (bench.py --scaling strong): rank
    7's shard of cfg5, 2^21 chains from stream 7 * 2^21, 4096 sweeps -- 9.22
    resident waves, i.e. full rounds plus one-chain tail rounds.  Sampled
    chains (incl. both ends and the tail rounds) bit-exact against the oracle,
    histogram complete, transient-exact pooled means."""
    from paper_1412_4825_b200 import shard as S
    c = workloads.CFG5
    lo, hi = S.shard_range(c["n_chains"], 7, 8)
    nc, ns = hi - lo, c["n_sweeps"]
    g = _run(c["seed"], S.gibbs_stream(0, lo), 0, nc, ns, samples=False)
    tot = g["totals"]
    assert g["n_invalid"] == 0 and tot[8] == nc and tot[HDR:].sum() == nc * ns
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    wave = 2 * 256 * 3 * sms
    tail0 = (nc // wave) * wave                       # first chain of the tail rounds
    rng = np.random.default_rng(8)
    picks = np.concatenate([[0, 1, tail0 - 1, tail0, tail0 + 1, nc - 1],
                            rng.integers(0, nc, 60), rng.integers(tail0, nc, 30)])
    for cidx in picks:
        r = oracle.gibbs_triangle(c["seed"], lo + int(cidx), 0, 1, ns, want_samples=False)
        assert np.array_equal(g["chain_stats"][:, cidx], r["chain_stats"][:, 0]), cidx
        assert np.array_equal(g["final_xy"][:, cidx], r["final_xy"][:, 0]), cidx
    ex = 1 / 3 - (1 - 4.0**-ns) / (9 * ns)
    sd = math.sqrt((5 / 3) * (1 / 18) / ns / nc)
    assert abs(tot[0] / nc - ex) < 6 * sd


def test_host_pipeline_multi_chunk_gibbs():
    nc, ns = 3_000_017, 16                            # chain_stats 120 MB -> 2 chunks
    g = _run(42, 0, 0, nc, ns, samples=False)
    st = np.empty((5, nc)); fx = np.empty((2, nc)); tot = np.empty(B.TOTALS_LEN)
    with handle(42) as h:
        B.brng_gibbs_triangle(h, nc, ns, None, None, 0, None, None, st, fx, tot)
        assert B.brng_get_offset(h) == ns
    assert np.array_equal(st, g["chain_stats"]) and np.array_equal(fx, g["final_xy"])
    assert np.array_equal(tot[HDR:], g["totals"][HDR:])
    np.testing.assert_allclose(tot[:HDR], g["totals"][:HDR], rtol=1e-12)


def test_host_samples_more_chains_than_a_wave():
    """Host out_x/out_y with more chains than one resident wave: the staging
    chunk is capped by bytes (a wave of chains x 64 sweeps x 8 B would exceed
    the 64 MB target), and the samples equal a device-pointer call bit for bit."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    nc, ns = 2 * 256 * 3 * sms + 1017, 64                 # > one bulk wave
    g = _run(42, 0, 0, nc, ns, samples=True)
    ox = np.empty((ns, nc)); oy = np.empty((ns, nc)); st = np.empty((5, nc))
    with handle(42) as h:
        B.brng_gibbs_triangle(h, nc, ns, None, None, 0, ox, oy, st, None, None)
        assert B.brng_get_offset(h) == ns
    assert np.array_equal(ox, g["out_x"]) and np.array_equal(oy, g["out_y"])
    assert np.array_equal(st, g["chain_stats"])


@pytest.mark.parametrize("extra", [0.66, 1.2, 1.5])
def test_bulk_tail_rounds_match_oracle(extra):
    """Bulk launches whose chain count is not a multiple of a resident wave run
    full three-chain rounds plus one-chain tail rounds (gibbs.cu grid_shape;
    strong scaling 2^24 / 8 = 9.2 waves): every chain's statistics and final
    state equal the oracle's, the histogram equals the oracle's exactly."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    wave = 2 * 256 * 3 * sms
    nc, ns = int(extra * wave) + 7, 6
    g = _run(42, 3, 11, nc, ns, samples=False)
    r = oracle.gibbs_triangle(42, 3, 11, nc, ns, want_samples=False)
    _assert_match(g, r, samples=False)


def test_launch_shapes_agree_across_the_latency_threshold():
    """Three launch shapes serve different chain counts (chain/helper warp
    pairs up to 32 chains per SM, thread per chain below half a bulk wave,
    three chains per thread above).  A chain's samples, statistics and final
    state must not depend on which one ran it: chains 0..n-1 of a run just
    above the latency-mode threshold equal the same chains of a run just below it,
    and both equal the oracle on sampled chains; histograms are exact."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    thr = 32 * sms                          # BRNG_GIBBS_LAT_PER_SM (gibbs.cu)
    ns, burn = 40, 3
    lo = _run(42, 5, 1000, thr, ns, burn)            # chain/helper warp pairs
    hi = _run(42, 5, 1000, thr + 37, ns, burn)       # thread per chain
    for k in ("out_x", "out_y"):
        assert np.array_equal(lo[k], hi[k][:, :thr]), k
    assert np.array_equal(lo["chain_stats"], hi["chain_stats"][:, :thr])
    assert np.array_equal(lo["final_xy"], hi["final_xy"][:, :thr])
    for c in (0, 1, thr // 2, thr - 1):
        r = oracle.gibbs_triangle(42, 5 + c, 1000, 1, ns, burn_in=burn)
        assert np.array_equal(lo["out_x"][:, c], r["out_x"][:, 0])
        assert np.array_equal(lo["chain_stats"][:, c], r["chain_stats"][:, 0])
    # histogram of the first thr chains is the same whichever kernel counted it
    extra = _run(42, 5 + thr, 1000, 37, ns, burn)
    assert np.array_equal(lo["totals"][HDR:] + extra["totals"][HDR:], hi["totals"][HDR:])


@pytest.mark.parametrize("stream_id", [0, (1 << 32) - 40_000, (5 << 32) + 123])
def test_bulk_launch_high_stream_word(stream_id):
    """The bulk launch computes round 2's M1 product once per sweep when every
    chain's stream has the same high word, per chain otherwise (a launch whose
    streams cross a 2^32 boundary).  Both must give the oracle's chains:
    sampled chains on both sides of the boundary, bit-exact."""
    n_chains, ns = 80_000, 12                      # above half a bulk wave
    g = _run(77, stream_id, 5, n_chains, ns, samples=True)
    for c in (0, 1, 39_999, 40_000, 40_001, n_chains - 1):
        r = oracle.gibbs_triangle(77, stream_id + c, 5, 1, ns)
        assert np.array_equal(g["out_x"][:, c], r["out_x"][:, 0]), c
        assert np.array_equal(g["out_y"][:, c], r["out_y"][:, 0]), c
        assert np.array_equal(g["chain_stats"][:, c], r["chain_stats"][:, 0]), c


@pytest.mark.parametrize("n_chains", [5, 4_737 + 3, 160_001])   # latency / small / bulk shapes
@pytest.mark.parametrize("n_sweeps,burn", [(0, 0), (4, 4), (33, 33)])
def test_degenerate_sweep_counts(n_chains, n_sweeps, burn):
    """No sweeps, or every sweep burnt in: no statistics samples (NaN
    moments, empty histogram), final state = start state (or the chain after
    its sweeps), cursor advanced by n_sweeps - the oracle's results, in
    every launch shape."""
    g = _run(3, 11, 5, n_chains, n_sweeps, burn, samples=n_sweeps > 0)
    cols = np.unique(np.array([0, 1, n_chains // 2, n_chains - 1]))
    r = oracle.gibbs_triangle(3, 11, 5, 1, n_sweeps, burn_in=burn)      # chain 0 only
    assert np.array_equal(g["final_xy"][:, :1], r["final_xy"], equal_nan=True)
    assert np.isnan(g["chain_stats"]).all()
    assert g["totals"][HDR:].sum() == 0
    assert g["totals"][8] == n_chains and g["totals"][9] == 0
    for c in cols:
        rc = oracle.gibbs_triangle(3, 11 + int(c), 5, 1, n_sweeps, burn_in=burn)
        assert np.array_equal(g["final_xy"][:, c], rc["final_xy"][:, 0]), c
        if n_sweeps:
            assert np.array_equal(g["out_x"][:, c], rc["out_x"][:, 0]), c
