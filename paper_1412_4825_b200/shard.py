"""Multi-GPU host logic: disjoint Philox counter ranges per rank and the one
collective of the hot path.

Samples, documents and chains are independent (Fig. 1
is per chain), so the path shards by COUNTER RANGE with no data-path
exchange: rank r draws exactly the samples an unsharded run would draw at the
same indices, so every sample, Dirichlet row, per-chain statistic, final state
and histogram count is bit-identical for any GPU count.  The Gibbs moment
totals (sums over chains) are added in a rank-dependent order and agree to
rounding (~1e-15 relative), not bit for bit.  The only
collective is the sum of the Gibbs totals (moment sums + 256-bin histogram,
BASELINE.json configs[4]), done with torch.distributed (NCCL on B200, gloo
in the CPU tests).
"""
from __future__ import annotations

GAMMA_STRIDE = 256


def shard_range(n: int, rank: int, world: int, align: int = 1) -> tuple[int, int]:
    """Contiguous [lo, hi) of n units for `rank`; boundaries are multiples of
    `align` (samples per Philox block for fills) except the final hi = n."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    units = -(-n // align)
    lo = (units * rank // world) * align
    hi = min(n, (units * (rank + 1) // world) * align)
    return min(lo, n), hi


def fill_cursor(base: int, lo: int, samples_per_block: int) -> int:
    """Cursor of a fill shard starting at sample lo (lo % samples_per_block == 0):
    4 for f32 fills and raw words, 2 for f64 fills (include/brng.h)."""
    if lo % samples_per_block:
        raise ValueError("fill shards must start on a Philox block boundary")
    return base + lo // samples_per_block


def gamma_cursor(base: int, lo: int) -> int:
    """Cursor of a Gamma shard starting at sample lo (256 blocks per sample)."""
    return base + GAMMA_STRIDE * lo


def dirichlet_cursor(base: int, row_lo: int, k: int) -> int:
    """Cursor of a Dirichlet shard starting at row row_lo of K components."""
    return base + GAMMA_STRIDE * row_lo * k


def gibbs_stream(stream_id: int, chain_lo: int) -> int:
    """Stream id of a Gibbs shard starting at chain chain_lo (chain c uses
    stream stream_id + c; the cursor is shared by all chains)."""
    return stream_id + chain_lo


def reduce_totals(totals, group=None):
    """In-place SUM of a Gibbs totals vector (f64[272]) over the process group:
    the hot path's only collective.  Counts stay exact (integers < 2^53)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(totals, op=dist.ReduceOp.SUM, group=group)
    return totals


def pooled_stats(totals) -> dict:
    """Pooled Gibbs statistics from a (reduced) totals vector (include/brng.h
    layout): mean of chain means, mean within-chain variance, between-chain
    variance of the means, mean covariance, histogram density."""
    t = [float(v) for v in totals]
    nc = t[8]
    if nc <= 0:
        raise ValueError("no chains in totals")
    mx, my = t[0] / nc, t[3] / nc
    out = {
        "n_chains": nc, "n_samples": t[9],
        "mean_x": mx, "mean_y": my,
        "within_var_x": t[1] / nc, "within_var_y": t[4] / nc,
        "between_var_x": t[2] / nc - mx * mx, "between_var_y": t[5] / nc - my * my,
        "cov_xy": t[6] / nc,
    }
    hist = t[16:16 + 256]
    tot = sum(hist)
    out["hist_prob"] = [h / tot for h in hist] if tot else hist
    return out
