"""Pins for the oracle's base generator and word->uniform conversions.

Philox4x32-10 (R-01/R-02): checked against an INDEPENDENT implementation,
ATen's header-only at::philox_engine compiled here for the CPU (no Random123
known-answer file is in the container and none is written from memory).
Conversions (R-04): exact-integer properties checked with Fractions.
"""
import os
import shutil
import subprocess
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def aten_philox(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    inc = os.path.join(os.path.dirname(torch.__file__), "include")
    exe = str(tmp_path_factory.mktemp("aten") / "aten_philox")
    subprocess.check_call(["g++", "-O1", "-std=c++17", "-I", inc,
                           os.path.join(HERE, "aten_philox.cpp"), "-o", exe])

    def run(triples):
        inp = "\n".join(f"{s} {st} {p}" for s, st, p in triples) + "\n"
        out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True)
        return np.array([[int(v) for v in ln.split()] for ln in out.stdout.strip().splitlines()],
                        dtype=np.uint64)
    return run


def _edge_triples():
    M32, M64 = (1 << 32) - 1, (1 << 64) - 1
    vals = [0, 1, M32 - 1, M32, M32 + 1, 1 << 32, (1 << 33) + 5, M64 - 1, M64,
            0x0123456789ABCDEF, 0xFEDCBA9876543210]
    trip = []
    for s in vals:
        for st in (0, 1, M32, 1 << 32, M64):
            for p in (0, 1, M32, 1 << 32, M64 - 1):
                trip.append((s, st, p))
    return trip


def test_philox_matches_aten_edges(aten_philox):
    trip = _edge_triples()
    ref = aten_philox(trip)
    got = np.array([oracle.block(*t) for t in trip], dtype=np.uint64)
    assert np.array_equal(got, ref)


def test_philox_matches_aten_random(aten_philox):
    rng = np.random.default_rng(20141215)
    trip = [tuple(int(x) for x in rng.integers(0, 2**63, size=3, dtype=np.int64) * 2
                  + rng.integers(0, 2, size=3)) for _ in range(3000)]
    trip = [(s % 2**64, st % 2**64, p % 2**64) for s, st, p in trip]
    ref = aten_philox(trip)
    got = np.array([oracle.block(*t) for t in trip], dtype=np.uint64)
    assert np.array_equal(got, ref)


def test_philox_key_counter_layout():
    # seed/stream/pos split into (lo, hi) 32-bit halves exactly as R-02 states.
    s, st, p = 0x1122334455667788, 0x99AABBCCDDEEFF00, 0x0F1E2D3C4B5A6978
    direct = oracle.philox4x32_10([p & 0xFFFFFFFF, p >> 32, st & 0xFFFFFFFF, st >> 32],
                                  [s & 0xFFFFFFFF, s >> 32])
    assert np.array_equal(direct, oracle.block(s, st, p))


def test_raw_words_order():
    # word i of the call comes from block base + i//4, position i%4 (R-12).
    w = oracle.raw_u32(5, 3, 100, 11)
    for i in range(11):
        assert w[i] == oracle.block(5, 3, 100 + i // 4)[i % 4]


def test_u24_exact_range_monotone():
    rng = np.random.default_rng(1)
    ws = [0, 1, 255, 256, 257, 2**31, 2**32 - 256, 2**32 - 1] + list(
        rng.integers(0, 2**32, 2000, dtype=np.uint64))
    prev = None
    for w in sorted(int(x) for x in ws):
        v = oracle.u24(w)
        f = Fraction(v)
        assert f * 2**24 == (w >> 8)            # exact, 24 significant bits
        assert np.float32(v) == v               # representable in binary32
        assert 0 <= f <= 1 - Fraction(1, 2**24)
        if prev is not None:
            assert v >= prev
        prev = v
    assert oracle.u24(2**32 - 1) == 1 - 2**-24


def test_u53_exact_range():
    rng = np.random.default_rng(2)
    pairs = [(0, 0), (2**32 - 1, 2**32 - 1), (2**11 - 1, 0), (2**11, 0), (0, 1)] + [
        (int(a), int(b)) for a, b in rng.integers(0, 2**32, (2000, 2), dtype=np.uint64)]
    for lo, hi in pairs:
        v = oracle.u53(lo, hi)
        m = (hi << 32) | lo
        assert Fraction(v) * 2**53 == (m >> 11)
        assert 0 <= v <= 1 - 2**-53
    assert oracle.u53(2**32 - 1, 2**32 - 1) == 1 - 2**-53
    assert oracle.u53(2**11 - 1, 0) == 0.0 and oracle.u53(2**11, 0) == 2**-53


def test_u32d_exact():
    for w in (0, 1, 2**31, 2**32 - 1, 123456789):
        assert Fraction(oracle.u32d(w)) == Fraction(w, 2**32)


def test_std_uniform_maps():
    f32 = oracle.std_uniform(9, 2, 7, 10, np.float32)
    f64 = oracle.std_uniform(9, 2, 7, 6, np.float64)
    for i in range(10):
        assert f32[i] == np.float32(oracle.u24(int(oracle.block(9, 2, 7 + i // 4)[i % 4])))
    for i in range(6):
        w = oracle.block(9, 2, 7 + i // 2)
        j = i % 2
        assert f64[i] == oracle.u53(int(w[2 * j]), int(w[2 * j + 1]))


def test_uniform_words_equidistributed():
    # chi^2 on the top byte of 2^18 raw words: a generator defect fails this.
    from scipy import stats
    w = oracle.raw_u32(123, 0, 0, 1 << 18)
    counts = np.bincount((w >> 24).astype(np.int64), minlength=256)
    p = stats.chisquare(counts).pvalue
    assert p > 1e-3
