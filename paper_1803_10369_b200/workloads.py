"""The named workloads of BASELINE.json / SURVEY.md §8d (data only).

c2: configs[1] — 1 GPU, ~1e8 packets/slice, k=10, v=2^20 (the headline).
c3: configs[2] — 1 GPU, v=2^24, ~1e6 candidate super points, latency-bound end-of-slice.
c5: configs[4] — adversarial skew: one host meeting 1e7 distinct peers in every
    slice ahead of a uniform 1e8-pair scan storm (PlantSpec.window = 1, so the
    rotation does not split the peers, generator.hpp:135-137).
c4 (configs[3]) is c2's shape at 1e9 packets/slice over 8 GPUs: bench.py --gpus N.
c1: configs[0] — the SPEC default on the CPU reference (acceptance criterion 5,
    acceptance_main.cpp:263-278): seeds 11-15, 120 one-second slices, k = 30,
    z = 8, v = 65536; a parity case, not a bench line. Its discrete-window
    variants (criteria 4 and 6, acceptance_main.cpp:347-400): three 300-second
    slices, z = 1, k = 1, v = 65536 with 150,000 pairs (seeds 1-5) and
    v = 1024 with 600,000 pairs (seeds 21-25).
"""
from __future__ import annotations

import math

SKETCH_SEED = 0x5EA00001
PAIRS = 100_000_000


def plant_cards():
    """The criterion-5 plants (acceptance_main.cpp:263-278): 1152 .. 16384, log-spaced."""
    return [int(math.floor(1152.0 * math.pow(16384.0 / 1152.0, i / 49.0) + 0.5)) for i in range(50)]


def sketch_cfg(cols):
    return dict(rows=4, cols=cols, rough_slots=8, linear_slots=1024, recorder_bits=4, window=10, theta=1024,
                seed=SKETCH_SEED)


def cols_of(workload):
    return 1 << 24 if workload == "c3" else 1 << 20


def trace_spec(pairs=PAIRS, slices=12, workload="c2"):
    if workload == "c3":  # uniform: ~1e6 candidate super points
        return dict(seed=3, slices=slices, window=10, a_hosts=1 << 20, b_hosts=1 << 24, pairs_per_slice=pairs,
                    skew=0.0, plants=[])
    if workload == "c5":  # one host x 1e7 peers every slice + a uniform scan storm
        return dict(seed=5, slices=slices, window=1, a_hosts=12_000_000, b_hosts=1 << 24, pairs_per_slice=pairs,
                    skew=0.0, plants=[(0x0AC80001, 10_000_000, 0, 0xFFFFFFFF)])
    return dict(seed=1, slices=slices, window=10, a_hosts=4194304, b_hosts=1 << 22, pairs_per_slice=pairs,
                skew=1.0, plants=[(0x0AC80001 + i, c, 0, 0xFFFFFFFF) for i, c in enumerate(plant_cards())])


DESCRIPTIONS = {
    "c2": "C2: u=4 v=2^20 g=8 g'=1024 z=4 k=10 theta=1024 seed=0x5EA00001; trace seed 1, 4M uniform sources, "
          "Zipf(1.0) 4M destinations, 50 plants",
    "c3": "C3: u=4 v=2^24 g=8 g'=1024 z=4 k=10 theta=1024 seed=0x5EA00001 (64 GiB linear table, epoch stamps); "
          "trace seed 3, 1M uniform sources, 16M uniform destinations (~1e6 candidates)",
    "c5": "C5: u=4 v=2^20 g=8 g'=1024 z=4 k=10 theta=1024 seed=0x5EA00001; trace seed 5, host 10.200.0.1 x 1e7 "
          "peers every slice ahead of 1e8 uniform pairs (12M sources, 16M destinations)",
}


def c1_sketch():
    return dict(rows=4, cols=65536, rough_slots=8, linear_slots=1024, recorder_bits=8, window=30, theta=1024,
                seed=SKETCH_SEED)


def c1_spec(seed, slices=120):
    """100,000 uniform sources, 65,536 Zipf(1.0) destinations, 8,000 background
    pairs per slice and the 50 always-active plants."""
    return dict(seed=seed, slices=slices, window=30, a_hosts=100_000, b_hosts=65_536, pairs_per_slice=8000,
                skew=1.0, plants=[(0x0AC80001 + i, c, 0, 0xFFFFFFFF) for i, c in enumerate(plant_cards())])


def discrete_sketch(cols):
    return dict(rows=4, cols=cols, rough_slots=8, linear_slots=1024, recorder_bits=1, window=1, theta=1024,
                seed=SKETCH_SEED)


def discrete_spec(seed, pairs):
    return dict(seed=seed, slices=3, window=1, slice_seconds=300, a_hosts=100_000, b_hosts=65_536,
                pairs_per_slice=pairs, skew=1.0,
                plants=[(0x0AC80001 + i, c, 0, 0xFFFFFFFF) for i, c in enumerate(plant_cards())])
