"""The ingest front end's CPU restatement (oracle/srla_oracle.c: orient_record,
SlicePartitioner, the SRLT reader) against the reference's own functions
(oracle/_ref, trace.hpp) on random traces, edge cases included."""
from __future__ import annotations

import numpy as np
import pytest

from oracle.pyoracle import LIBS, Checker


@pytest.fixture(scope="module")
def pair():
    import os
    if not os.path.exists(LIBS["ref"]):
        pytest.skip("oracle/_ref not built")
    return Checker("orc"), Checker("ref")


def _trace(rng, n, t0=1_700_000_000, span=50):
    ts = np.sort(rng.integers(t0, t0 + span, n)).astype(np.uint32)
    hosts = np.concatenate([rng.integers(0x0A000000, 0x0A00FFFF, n // 2),
                            rng.integers(0xC0A80000, 0xC0A8FFFF, n - n // 2)]).astype(np.uint32)
    rng.shuffle(hosts)
    other = rng.choice(np.array([0x0A000001, 0x08080808, 0xC0A80101, 0x0A00FF00], np.uint32), n)
    return np.stack([ts, hosts, other], 1).astype(np.uint32)


@pytest.mark.parametrize("bits", [0, 8, 16, 24, 32])
def test_orient_matches_reference(pair, bits):
    orc, ref = pair
    rng = np.random.default_rng(bits)
    recs = _trace(rng, 5000)
    a, sa = orc.orient(recs, 0x0A000000 | 0x1234, bits)  # host bits below the mask are masked off
    b, sb = ref.orient(recs, 0x0A000000 | 0x1234, bits)
    assert np.array_equal(a, b) and np.array_equal(sa, sb)
    assert sa.sum() == len(recs)


@pytest.mark.parametrize("seconds", [1, 7, 60, 300])
def test_slice_bounds_match_reference(pair, seconds):
    orc, ref = pair
    rng = np.random.default_rng(seconds)
    recs = _trace(rng, 3000, span=2000)
    assert np.array_equal(orc.slice_bounds(recs, seconds), ref.slice_bounds(recs, seconds))
    # gaps make empty slices
    gap = recs.copy()
    gap[1500:, 0] += 10 * seconds
    assert np.array_equal(orc.slice_bounds(gap, seconds), ref.slice_bounds(gap, seconds))
    assert len(orc.slice_bounds(recs[:0], seconds)) == 1


def _srlt(recs):
    return b"SRLT" + bytes([1]) + np.ascontiguousarray(recs, np.uint32).astype("<u4").tobytes()


def test_parse_srlt_matches_reference(pair):
    orc, ref = pair
    rng = np.random.default_rng(3)
    recs = _trace(rng, 4000)
    for data in (_srlt(recs), _srlt(recs)[:-5], _srlt(recs[:0]), b"SRLT\x02" + b"\0" * 24, b"XX"):
        a = orc.parse_srlt(data)
        b = ref.parse_srlt(data)
        assert a[1:] == b[1:], (a[1:], b[1:])
        assert np.array_equal(a[0], b[0])
    bad = recs.copy()
    bad[1234, 0] = bad[1233, 0] - 1
    a, b = orc.parse_srlt(_srlt(bad)), ref.parse_srlt(_srlt(bad))
    assert a[1:] == b[1:] == (3, 1234)
    assert np.array_equal(a[0], b[0])
