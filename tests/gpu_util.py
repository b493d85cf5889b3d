"""Helpers for the -m gpu tests: a handle bound to torch's current stream."""
from __future__ import annotations

import contextlib

import torch


@contextlib.contextmanager
def handle(seed, stream_id=0, cursor=0):
    import paper_1412_4825_b200 as B
    h = B.brng_create(seed, stream_id)
    try:
        B.brng_set_cuda_stream(h, torch.cuda.current_stream().cuda_stream)
        if cursor:
            B.brng_set_offset(h, cursor)
        yield h
    finally:
        B.brng_destroy(h)


def dev():
    return torch.device("cuda:0")


def empty(n, dtype, offset=0):
    """Device tensor of n elements starting `offset` elements into a fresh
    allocation (offset != 0 -> not 16-byte aligned)."""
    base = torch.empty(n + offset, dtype=dtype, device=dev())
    return base[offset:]


def to_dev(x, offset=0):
    t = empty(x.numel(), x.dtype, offset)
    t.copy_(x.reshape(-1))
    return t.view(x.shape) if offset == 0 else t
