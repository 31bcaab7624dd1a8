"""Pin the C restatement (oracle/srla_oracle.c) to the reference: golden
vectors produced by the unmodified reference headers (tests/golden/), the
reference's own known-answer tests, and — where oracle/_ref is built — a live
comparison. CPU only."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import golden_flow as GF
import scenarios as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _bits(x):
    return format(np.float64(x).view(np.uint64).item(), "016x")


def test_kats_match_reference(oracle):
    k = json.load(open(os.path.join(GOLD, "kats.json")))
    assert _bits(oracle.super_test_ratio) == k["ratio"]
    for sd, idx, key, v in k["hash_u32"]:
        assert oracle.hash_u32(sd, idx, key) == v
    for sd, idx, key, rng, v in k["reduce"]:
        assert oracle.hash_reduce(sd, idx, key, rng) == v
    for th, g, v in k["sampling_exponent"]:
        assert oracle.f("sampling_exponent")(th, g) == v
    for g, v in k["threshold"]:
        assert oracle.f("super_weight_threshold")(oracle.super_test_ratio, g) == v
    for w, slots, v in k["linear_estimate"]:
        e = oracle.linear_estimate(w, slots)
        assert (None if e is None else _bits(e)) == v


def test_reference_unit_kats(oracle):
    # tests/test_estimators.cpp:11-29 — tau / threshold
    assert oracle.f("sampling_exponent")(1024, 8) == 7
    assert oracle.f("sampling_exponent")(8, 8) == 0
    assert oracle.f("super_weight_threshold")(oracle.super_test_ratio, 8) == 3
    # tests/test_estimators.cpp:164-183
    assert oracle.linear_estimate(100, 1024) == pytest.approx(105.22596757275539, rel=1e-12)
    assert oracle.linear_estimate(1024, 1024) is None
    # tests/test_sea.cpp:139-172 — Eq. 9
    from oracle.pyoracle import SeaConfig
    sk = oracle.sketch(SeaConfig(rows=4, cols=16, linear_slots=1024, recorder_bits=16, window=300, theta=1024))
    for w in (0, 1, 100, 500, 1023):
        assert sk.corrected_estimate_from(w, 0.0) == oracle.linear_estimate(w, 1024)
    assert sk.corrected_estimate_from(1024, 0.0) is None
    assert sk.corrected_estimate_from(4, 0.00390625) == 0.0
    assert sk.corrected_estimate_from(3, 0.00390625) == 0.0
    assert sk.corrected_estimate_from(300, 0.25 ** 4) == pytest.approx(350.99291022602281, rel=1e-12)
    assert sk.corrected_estimate_from(1024, 0.00390625) is None
    assert sk.corrected_estimate_from(100, 1.0 - 1e-13) == oracle.linear_estimate(100, 1024)


def test_row_fill_fraction_kat(oracle):
    # tests/test_sea.cpp:117-137
    from oracle.pyoracle import LINEAR, SeaConfig
    sk = oracle.sketch(SeaConfig(rows=1, cols=4, linear_slots=1024, recorder_bits=8, window=4, theta=8, seed=0xFACE))
    assert sk.row_fill_fraction(0) == 0.0
    row = sk.export_row(0, LINEAR)
    row[np.arange(512) * 8] = 0
    sk.import_row(0, LINEAR, row)
    assert sk.row_fill_fraction(0) == 0.125


@pytest.mark.parametrize("name", sorted(S.SCENARIOS))
def test_oracle_matches_golden(oracle, name):
    g = json.load(open(os.path.join(GOLD, f"{name}.json")))
    got = GF.run_flow_checker(oracle, name)
    assert got["records_sha256"] == g["records_sha256"], "trace recipe drifted"
    assert got["cfg"] == g["cfg"]
    msg = GF.compare(g["slices"], got["slices"])
    assert msg is None, msg


def test_config_validation_mirrors_reference(oracle):
    from oracle.pyoracle import SeaConfig
    bad = [dict(rows=0), dict(cols=0), dict(rough_slots=0), dict(linear_slots=1), dict(theta=0),
           dict(recorder_bits=0), dict(recorder_bits=33), dict(recorder_bits=1, window=2), dict(window=0),
           dict(rows=65)]
    for kw in bad:
        with pytest.raises(ValueError):
            oracle.sketch(SeaConfig(**kw))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_matches_reference_live(oracle, ref, seed):
    """Random contended configs, compared slice by slice with the live reference."""
    from oracle.pyoracle import SeaConfig
    rng = np.random.default_rng(seed)
    rows = int(rng.integers(1, 7))
    bits = int(rng.choice([4, 8, 12, 20]))
    cfg = SeaConfig(rows=rows, cols=int(rng.choice([8, 64, 1000, 4096])), rough_slots=int(rng.integers(1, 20)),
                    linear_slots=int(rng.integers(2, 200)), recorder_bits=bits,
                    window=int(rng.integers(1, min(15, (1 << bits) - 1))), theta=int(rng.integers(1, 300)),
                    seed=int(rng.integers(0, 2**63)))
    po, pr = oracle.pipeline(cfg) if cfg.cols & (cfg.cols - 1) == 0 else None, None
    so, sr = oracle.sketch(cfg), ref.sketch(cfg)
    co, cr = GF.CheckerBackend.__new__(GF.CheckerBackend), GF.CheckerBackend.__new__(GF.CheckerBackend)
    co.sk, co.csip, co.seen = so, [], set()
    cr.sk, cr.csip, cr.seen = sr, [], set()
    c = S.Cfg(**{k: getattr(cfg, k) for k in S.Cfg().__dict__})
    slices = S.random_slices(seed, 8, (0, 3000), int(rng.integers(5, 400)), int(rng.integers(10, 3000)))
    a = GF.run_flow(co, c, slices)
    b = GF.run_flow(cr, c, slices)
    assert GF.compare(b, a) is None


def test_generator_matches_reference(oracle, ref):
    from oracle.pyoracle import PlantSpec
    for sec in (1, 7):
        spec = PlantSpec(seed=5, slices=5, window=3, slice_seconds=sec, a_hosts=300, b_hosts=1000,
                         pairs_per_slice=700, skew=0.8,
                         plants=[(0x0AC80001, 90, 0, 3), (0x0AC80002, 200, 2, 0xFFFFFFFF)])
        assert np.array_equal(oracle.generate(spec), ref.generate(spec))


def test_generate_slice_matches_generate_trace(ref):
    """ref_generate_slice (parallel, counter-based jump-ahead over the
    reference's own generator pieces) equals slice s of generate_trace."""
    from oracle.pyoracle import PlantSpec
    for skew, window, plants in ((1.0, 10, [(0x0AC80001, 900, 0, 0xFFFFFFFF), (0x0AC80002, 50, 2, 3)]),
                                 (0.0, 1, [(0x0AC80001, 5000, 1, 0xFFFFFFFF)]), (0.7, 3, [])):
        spec = PlantSpec(seed=9, slices=5, window=window, a_hosts=3000, b_hosts=8192, pairs_per_slice=4001,
                         skew=skew, plants=plants)
        whole = ref.generate(spec)
        parts = [ref.generate_slice(spec, s, threads=t) for s, t in zip(range(5), (1, 2, 3, 7, 16))]
        assert np.array_equal(whole, np.concatenate(parts))


def test_block_sums_restated(ref):
    rng = np.random.default_rng(3)
    for n in (0, 1, 7, 8, 9, 4096, (1 << 20) - 1, 1 << 20, (1 << 20) + 5, 3 * (1 << 20) + 13):
        b = rng.integers(0, 256, n, dtype=np.uint8)
        assert np.array_equal(ref.block_sums(b, threads=3), GF.block_sums_np(b)), n
