"""Deterministic parity scenarios shared by the golden-fixture generator
(tests/golden/make_golden.py), the oracle tests and the GPU parity tests.

Each scenario is a sketch configuration plus a list of slices of records
(ts, src, dst). Shapes follow the reference's own fixtures:
  * small_config()       tests/test_sea.cpp:16-27
  * small_run/small_spec tests/test_pipeline.cpp:28-53
  * make_small_trace     tests/acceptance/acceptance_main.cpp:86-121 (criterion 1)
  * snap_config()        tests/test_snapshot.cpp:31-42
  * accuracy_spec        tests/acceptance/acceptance_main.cpp:255-278 (criterion 5 shape)
plus contended / wide-word / many-row / non-power-of-two variants that
exercise every kernel path. Random pairs use numpy's PCG64 (stable across
numpy versions) so the GPU box regenerates identical traces.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

RATIO = 0.99 * (1.0 - math.exp(-1.0 / 3.0))  # estimators.hpp:19


@dataclass
class Cfg:
    rows: int = 4
    cols: int = 65536
    rough_slots: int = 8
    linear_slots: int = 1024
    recorder_bits: int = 1
    window: int = 1
    theta: int = 1024
    seed: int = 0x00C0FFEE

    def as_dict(self):
        return dict(rows=self.rows, cols=self.cols, rough_slots=self.rough_slots,
                    linear_slots=self.linear_slots, recorder_bits=self.recorder_bits,
                    window=self.window, theta=self.theta, seed=self.seed)


@dataclass
class Spec:
    """PlantSpec fields (generator.hpp:36-43)."""
    seed: int = 1
    start_ts: int = 1700000000
    slice_seconds: int = 1
    slices: int = 60
    window: int = 1
    a_base: int = 0x0A100000
    b_base: int = 0x64400000
    a_hosts: int = 1000
    b_hosts: int = 4096
    pairs_per_slice: int = 500
    skew: float = 1.0
    plants: list = field(default_factory=list)


def plant_cards():
    # acceptance_main.cpp:255-261
    return [int(math.floor(1152.0 * math.pow(16384.0 / 1152.0, i / 49.0) + 0.5)) for i in range(50)]


def random_slices(seed, n_slices, pairs, a_pool, b_pool, a_base=0x0A000000, b_base=0xB0000000,
                  heavy=None, a_shift=0):
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for s in range(n_slices):
        a_base_s = a_base + s * a_shift
        n = int(rng.integers(pairs[0], pairs[1] + 1))
        recs = np.zeros((n, 3), np.uint32)
        recs[:, 0] = 1700000000
        recs[:, 1] = a_base_s + rng.integers(0, a_pool, n)
        recs[:, 2] = b_base + rng.integers(0, b_pool, n)
        if heavy and rng.integers(0, 4) == 0:  # acceptance_main.cpp:113-118
            a = a_base_s + int(rng.integers(0, a_pool))
            h = np.zeros((heavy, 3), np.uint32)
            h[:, 0] = 1700000000
            h[:, 1] = a
            h[:, 2] = b_base + 0x1000 + rng.integers(0, 64, heavy)
            recs = np.concatenate([recs, h])
        out.append(recs)
    return out


def split_by_ts(recs, spec: Spec):
    """SlicePartitioner with the generator's anchored origin (trace.hpp:243-281)."""
    ids = (recs[:, 0].astype(np.int64) - int(recs[0, 0])) // spec.slice_seconds
    return [recs[ids == s] for s in range(int(ids.max()) + 1)] if len(recs) else []


# name -> (cfg, source) ; source is ("random", kwargs) or ("spec", Spec)
SCENARIOS = {
    "sea_small": (Cfg(rows=2, cols=16, rough_slots=8, linear_slots=32, recorder_bits=8, window=4,
                      theta=8, seed=0xFACE),
                  ("random", dict(seed=1, n_slices=7, pairs=(300, 500), a_pool=24, b_pool=128))),
    "pipeline_small": (Cfg(rows=2, cols=256, rough_slots=8, linear_slots=64, recorder_bits=8, window=3,
                           theta=32, seed=0xBEEF),
                       ("spec", Spec(seed=2, slices=9, window=3, a_hosts=50, b_hosts=512,
                                     pairs_per_slice=250, skew=1.0,
                                     plants=[(0x0AC80001, 80, 0, 0xFFFFFFFF), (0x0AC80002, 100, 0, 0xFFFFFFFF)]))),
    "pipeline_small_3000": (Cfg(rows=2, cols=256, rough_slots=8, linear_slots=64, recorder_bits=8, window=3,
                                theta=32, seed=0xBEEF),
                            ("spec", Spec(seed=3, slices=9, window=3, a_hosts=50, b_hosts=512,
                                          pairs_per_slice=3000, skew=1.0,
                                          plants=[(0x0AC80001, 80, 0, 0xFFFFFFFF),
                                                  (0x0AC80002, 100, 0, 0xFFFFFFFF)]))),
    "snapshot": (Cfg(rows=3, cols=8, rough_slots=8, linear_slots=16, recorder_bits=8, window=5, theta=16,
                     seed=0x1DEA),
                 ("random", dict(seed=404, n_slices=8, pairs=(200, 500), a_pool=16, b_pool=64))),
    "contended": (Cfg(rows=4, cols=1024, rough_slots=8, linear_slots=1024, recorder_bits=4, window=10,
                      theta=1024, seed=0x5EA00001),
                  ("random", dict(seed=77, n_slices=14, pairs=(150000, 250000), a_pool=3000, b_pool=200000))),
    "tiny_flagged": (Cfg(rows=3, cols=4, rough_slots=8, linear_slots=16, recorder_bits=8, window=3, theta=8,
                         seed=0x77),
                     ("random", dict(seed=5, n_slices=8, pairs=(50, 400), a_pool=200, b_pool=64))),
    "wide_w2": (Cfg(rows=3, cols=512, rough_slots=8, linear_slots=100, recorder_bits=16, window=300, theta=64,
                    seed=0xABCDEF),
                ("random", dict(seed=9, n_slices=6, pairs=(2000, 6000), a_pool=400, b_pool=3000))),
    "w4_rows5_npow2": (Cfg(rows=5, cols=100, rough_slots=12, linear_slots=48, recorder_bits=20, window=7,
                           theta=48, seed=0x1234567890),
                       ("random", dict(seed=11, n_slices=10, pairs=(500, 3000), a_pool=150, b_pool=900))),
    "rough70_tau0": (Cfg(rows=2, cols=64, rough_slots=70, linear_slots=40, recorder_bits=6, window=5, theta=40,
                         seed=0x99),
                     ("random", dict(seed=12, n_slices=7, pairs=(200, 1500), a_pool=60, b_pool=400))),
    "c1_shape": (Cfg(rows=4, cols=65536, rough_slots=8, linear_slots=1024, recorder_bits=8, window=30,
                     theta=1024, seed=0x5EA00001),
                 ("spec", Spec(seed=11, slices=33, window=30, a_hosts=100000, b_hosts=65536,
                               pairs_per_slice=8000, skew=1.0,
                               plants=[(0x0AC80001 + i, c, 0, 0xFFFFFFFF) for i, c in enumerate(plant_cards())]))),
    "drift_evict": (Cfg(rows=3, cols=128, rough_slots=8, linear_slots=64, recorder_bits=4, window=3, theta=16,
                        seed=0xD1F7),
                    ("random", dict(seed=21, n_slices=14, pairs=(800, 1600), a_pool=40, b_pool=300, heavy=60,
                                    a_shift=12))),
}
# criterion-1 corpus shapes (acceptance_main.cpp:93-101): rows 1/2/4, cols 16/64, k 2/4/8
for idx in range(6):
    SCENARIOS[f"crit1_{idx}"] = (
        Cfg(rows=1 << ((idx // 3) % 3), cols=64 if idx % 2 else 16, rough_slots=8, linear_slots=32,
            recorder_bits=4, window=(2, 4, 8)[idx % 3], theta=16, seed=0xC0FFEE00 + idx * 7919),
        ("random", dict(seed=0xC0FFEE00 + idx, n_slices=(2, 4, 8)[idx % 3] + 8, pairs=(40, 240), a_pool=32,
                        b_pool=256, heavy=30)))

FAST = [n for n in SCENARIOS if n not in ("contended", "c1_shape")]


def slices_for(name, generate=None):
    """The scenario's slices. `generate(spec) -> (n,3) records` is required
    for spec-driven scenarios (the oracle's or the device's generator)."""
    cfg, (kind, src) = SCENARIOS[name]
    if kind == "random":
        return random_slices(**src)
    recs = generate(src)
    return split_by_ts(recs, src)


def state_digest(state: dict, rows: int) -> str:
    """sha256 over the SSEA row order: per row indicator, rough, linear
    (snapshot.hpp:128-132), little-endian words."""
    h = hashlib.sha256()
    for i in range(rows):
        for k in (0, 1, 2):
            h.update(np.ascontiguousarray(state[(k, i)]).tobytes())
    return h.hexdigest()


def records_digest(slices) -> str:
    h = hashlib.sha256()
    for s in slices:
        h.update(np.ascontiguousarray(s, dtype=np.uint32).tobytes())
    return h.hexdigest()


def f64_bits(x: float) -> str:
    return np.float64(x).view(np.uint64).item().to_bytes(8, "little").hex()
