"""Exact sliding-window cardinalities on the device (srla_exact_*,
csrc/exact.cu) against the reference's own exact stores
(oracle.hpp: SliceRingStore and PairRecorderStore, compiled unmodified in
oracle/_ref): every window's (host, distinct count) list, the live pair count,
the out-of-window error, on scenario traces and on the C2 trace shape."""
from __future__ import annotations

import numpy as np
import pytest

import golden_flow as GF
import scenarios as S

pytestmark = pytest.mark.gpu


def _compare(ref, slices, k, bits=8):
    from oracle.pyoracle import ExactRef
    from paper_1803_10369_b200.srla import ExactStore
    mine = ExactStore(k)
    ring, pairs = ExactRef(ref, "ring", k), ExactRef(ref, "pairs", k, bits)
    windows = 0
    for s, recs in enumerate(slices):
        mine.observe(recs)
        ring.observe(recs)
        pairs.observe(recs)
        for kk in {1, min(k, s + 1)}:
            t = s + 1 - kk
            h, c = mine.cardinalities(t, kk)
            for other in (ring, pairs):
                h2, c2 = other.cardinalities(t, kk)
                assert np.array_equal(h, h2) and np.array_equal(c, c2), f"slice {s} window ({t}, {kk})"
            windows += 1
        assert mine.pair_count() == pairs.pair_count(), f"slice {s}: live pairs"
        mine.end_slice()
        ring.end_slice()
        pairs.end_slice()
    return windows


@pytest.mark.parametrize("name", ["pipeline_small", "contended", "drift_evict", "crit1_3", "c1_shape"])
def test_exact_store_matches_reference_stores(gpu, ref, oracle, name):
    cfg, _ = S.SCENARIOS[name]
    assert _compare(ref, GF.scenario_slices(name, oracle), cfg.window) > 0


def test_exact_store_c2_shape(gpu, ref):
    """The C2 trace shape (Zipf destinations, 50 planted hosts) at 1e6 pairs per
    slice over 12 slices, window 10."""
    from oracle.pyoracle import PlantSpec
    from paper_1803_10369_b200 import workloads as WL
    spec = PlantSpec(**WL.trace_spec(1_000_000, slices=12))
    slices = [ref.generate_slice(spec, s) for s in range(12)]
    assert _compare(ref, slices, 10, bits=4) == 1 + 2 * 11  # k = 1 and the full window, every slice


def test_exact_store_window_errors(gpu):
    from paper_1803_10369_b200.srla import ExactStore
    x = ExactStore(4)
    x.observe(np.array([[0, 1, 100], [0, 1, 100], [0, 2, 5]], np.uint32))
    h, c = x.cardinalities(0, 1)
    assert h.tolist() == [1, 2] and c.tolist() == [1, 1]  # a pair seen twice counts once
    with pytest.raises(IndexError, match=r"window \[0, \+2\) is not observable at slice 0"):
        x.cardinalities(0, 2)
    for _ in range(5):
        x.end_slice()
    with pytest.raises(IndexError):
        x.cardinalities(0, 5)  # wider than the ring
    assert x.cardinalities(2, 4)[0].size == 0
