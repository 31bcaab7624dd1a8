"""Parity of the CUDA engine (through the C ABI) with the reference.

* every golden scenario (tests/golden/, produced by the unmodified reference):
  candidate pushes, candidate list order, report entries with the estimate's
  exact double bits, retained list and a digest of every DR / indicator word;
* live comparisons with the C restatement on random and contended configs,
  host vs device input, arbitrary batch splits;
* ports of the reference's hot-path unit tests (tests/test_sea.cpp);
* the device trace generator byte-identical to generate_trace.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

import golden_flow as GF
import scenarios as S

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def engine(cfg: S.Cfg):
    from paper_1803_10369_b200.srla import EstimatorArray, SeaConfig
    return EstimatorArray(SeaConfig(**cfg.as_dict()))


@pytest.mark.parametrize("order", ["fast", "legacy"])
@pytest.mark.parametrize("name", sorted(S.SCENARIOS))
def test_engine_matches_reference_golden(gpu, oracle, name, order, monkeypatch):
    """Every golden scenario, with the ordering phase on device counts
    (order.cuh, the default) and with the sorted host-synchronised path."""
    monkeypatch.setenv("SRLA_ORDER", order)
    g = json.load(open(os.path.join(GOLD, f"{name}.json")))
    cfg, _ = S.SCENARIOS[name]
    slices = GF.scenario_slices(name, oracle)
    assert S.records_digest(slices) == g["records_sha256"]
    got = GF.run_flow(GF.EngineBackend(engine(cfg)), cfg, slices)
    msg = GF.compare(g["slices"], got)
    assert msg is None, msg


@pytest.mark.parametrize("dedup", ["auto", "0", "1"])
@pytest.mark.parametrize("epoch", ["1", "0"])
@pytest.mark.parametrize("name", [n for n in sorted(S.SCENARIOS) if S.SCENARIOS[n][0].rows <= 4])
def test_binned_marks_match_reference_golden(gpu, oracle, name, epoch, dedup, monkeypatch):
    """Same goldens with the binned linear-mark path forced on (~8 regions,
    tiny bins so the overflow-to-direct-mark path runs too), with epoch-stamp
    recorders (z <= 7) and with literal ones; K1's duplicate-mark filter on
    from the first bin overflow (auto), never, or always."""
    monkeypatch.setenv("SRLA_FORCE_BINS", "1")
    monkeypatch.setenv("SRLA_EPOCH", epoch)
    if dedup != "auto":
        monkeypatch.setenv("SRLA_K1_DEDUP", dedup)
    g = json.load(open(os.path.join(GOLD, f"{name}.json")))
    cfg, _ = S.SCENARIOS[name]
    slices = GF.scenario_slices(name, oracle)
    got = GF.run_flow(GF.EngineBackend(engine(cfg)), cfg, slices)
    msg = GF.compare(g["slices"], got)
    assert msg is None, msg


@pytest.mark.parametrize("sparse", ["0", "1000000"])
@pytest.mark.parametrize("name", ["contended", "drift_evict", "c1_shape"])
def test_epoch_stamp_paths_match_reference_golden(gpu, oracle, name, sparse, monkeypatch):
    """Epoch-stamp recorders with every fine slice forced through one of the
    two stamp kernels: the block-per-slice shared-memory path
    (SRLA_STAMP_SPARSE=0) or the warp-per-slice in-place path with its claim
    bitmap (every slice counts as sparse)."""
    monkeypatch.setenv("SRLA_FORCE_BINS", "1")
    monkeypatch.setenv("SRLA_EPOCH", "1")
    monkeypatch.setenv("SRLA_STAMP_SPARSE", sparse)
    g = json.load(open(os.path.join(GOLD, f"{name}.json")))
    cfg, _ = S.SCENARIOS[name]
    slices = GF.scenario_slices(name, oracle)
    got = GF.run_flow(GF.EngineBackend(engine(cfg)), cfg, slices)
    msg = GF.compare(g["slices"], got)
    assert msg is None, msg


def _oracle_backend(oracle, cfg):
    b = GF.CheckerBackend.__new__(GF.CheckerBackend)
    from oracle.pyoracle import SeaConfig
    b.sk, b.csip, b.seen = oracle.sketch(SeaConfig(**cfg.as_dict())), [], set()
    return b


@pytest.mark.parametrize("seed", range(6))
def test_engine_matches_oracle_random_configs(gpu, oracle, seed):
    rng = np.random.default_rng(100 + seed)
    bits = int(rng.choice([3, 4, 8, 12, 16, 20, 32]))
    cfg = S.Cfg(rows=int(rng.choice([1, 2, 3, 4, 5, 9])), cols=int(rng.choice([4, 8, 64, 1000, 4096, 65536])),
                rough_slots=int(rng.integers(1, 40)), linear_slots=int(rng.choice([2, 7, 32, 100, 1024])),
                recorder_bits=bits, window=int(rng.integers(1, min(40, (1 << min(bits, 30)) - 1) + 1)),
                theta=int(rng.choice([1, 8, 64, 300, 1024])), seed=int(rng.integers(0, 2**63)))
    slices = S.random_slices(seed, 10, (0, 20000), int(rng.integers(5, 2000)), int(rng.integers(10, 50000)))
    a = GF.run_flow(_oracle_backend(oracle, cfg), cfg, slices)
    b = GF.run_flow(GF.EngineBackend(engine(cfg)), cfg, slices)
    msg = GF.compare(a, b)
    assert msg is None, f"{cfg}: {msg}"


def test_engine_matches_oracle_c2_shape_medium(gpu, oracle):
    """The C2 trace shape (uniform 4M sources, Zipf 4M destinations, 50 plants)
    at 2e6 packets per slice on a 2^16-column sketch: heavy column sharing,
    thousands of candidates per slice, full bit-exact comparison."""
    from oracle.pyoracle import PlantSpec
    spec = S.Spec(seed=1, slices=12, window=10, a_hosts=4194304, b_hosts=1 << 22, pairs_per_slice=2_000_000,
                  skew=1.0, plants=[(0x0AC80001 + i, c, 0, 0xFFFFFFFF) for i, c in enumerate(S.plant_cards())])
    recs = oracle.generate(PlantSpec(**spec.__dict__))
    slices = S.split_by_ts(recs, spec)
    cfg = S.Cfg(rows=4, cols=1 << 16, rough_slots=8, linear_slots=1024, recorder_bits=4, window=10, theta=1024,
                seed=0x5EA00001)
    a = GF.run_flow(_oracle_backend(oracle, cfg), cfg, slices)
    b = GF.run_flow(GF.EngineBackend(engine(cfg)), cfg, slices)
    msg = GF.compare(a, b)
    assert msg is None, msg
    assert sum(s["pushes"]["n"] for s in a) > 50


def test_batch_splits_and_device_input(gpu, oracle):
    import torch
    cfg, _ = S.SCENARIOS["drift_evict"]
    slices = GF.scenario_slices("drift_evict", oracle)
    ref = GF.run_flow(_oracle_backend(oracle, cfg), cfg, slices)

    class Split(GF.EngineBackend):
        def scan(self, recs):
            rng = np.random.default_rng(len(recs))
            cuts = np.sort(rng.integers(0, len(recs) + 1, 5))
            parts = np.split(recs, cuts)
            out = []
            for i, p in enumerate(parts):
                if i % 2:
                    t = torch.from_numpy(p.astype(np.int32)).cuda()
                    torch.cuda.synchronize()
                    out.append(self.e.scan_collect(t))
                else:
                    out.append(self.e.scan_collect(p))
            return np.concatenate(out) if out else np.empty(0, np.uint32)

    got = GF.run_flow(Split(engine(cfg)), cfg, slices)
    assert GF.compare(ref, got) is None


# ---------------------------------------------------------------- test_sea.cpp ports

def small_config(**kw):
    c = dict(rows=2, cols=16, rough_slots=8, linear_slots=32, recorder_bits=8, window=4, theta=8, seed=0xFACE)
    c.update(kw)
    return S.Cfg(**c)


def test_single_pair_updates_one_slot_per_row(gpu, oracle):
    # tests/test_sea.cpp:39-60
    from paper_1803_10369_b200.srla import LINEAR, ROUGH
    cfg = small_config(rows=1)
    e = engine(cfg)
    assert e.tau == 0
    aip, bip = 0x0A000001, 0x08080808
    assert len(e.scan_ip_pair(aip, bip)) == 0
    col = e.column_of(0, aip)
    rslot = oracle.hash_reduce(cfg.seed, 1, bip, cfg.rough_slots)
    lslot = oracle.hash_u32(cfg.seed, 0, bip) % cfg.linear_slots
    rough, lin = e.export_row(0, ROUGH), e.export_row(0, LINEAR)
    assert rough[col * cfg.rough_slots + rslot] == 0 and lin[col * cfg.linear_slots + lslot] == 0
    assert (rough < cfg.window).sum() == 1 and (lin < cfg.window).sum() == 1
    assert e.union_rough_weight(aip) == 1


def test_indicator_suppresses_duplicates(gpu, oracle):
    # tests/test_sea.cpp:62-77
    from paper_1803_10369_b200.srla import INDICATOR
    e = engine(small_config())
    aip = 0x0A000002
    pushes = e.scan_pairs([(aip, 0xC0000000 + i) for i in range(64)])
    assert list(pushes) == [aip] and list(e.candidates()) == [aip]
    bit = 1 << oracle.hash_reduce(0xFACE, 2, aip, 16)
    for i in range(2):
        assert e.export_row(i, INDICATOR)[e.column_of(i, aip)] & bit


def test_union_view_max_semantics(gpu):
    # tests/test_sea.cpp:79-115
    from paper_1803_10369_b200.srla import ROUGH
    cfg = small_config()
    e = engine(cfg)
    ind, rough, lin = e.union_view(0x0A000003, True)
    assert ind == 0 and (rough == 255).all() and (lin == 255).all()
    aip = 0x0A000005
    for row, val in ((0, 5), (1, 9)):
        r = e.export_row(row, ROUGH)
        r[e.column_of(row, aip) * cfg.rough_slots + 3] = val
        e.import_row(row, ROUGH, r)
    ind, rough, lin = e.union_view(aip, False)
    assert rough[3] == 9 and lin is None


def test_row_fill_fraction(gpu):
    # tests/test_sea.cpp:117-137
    from paper_1803_10369_b200.srla import LINEAR
    e = engine(small_config(rows=1, cols=4, linear_slots=1024))
    assert e.row_fill_fraction(0) == 0.0
    with pytest.raises(ValueError):
        e.row_fill_fraction(1)
    row = e.export_row(0, LINEAR)
    row[np.arange(512) * 8] = 0
    e.import_row(0, LINEAR, row)
    assert e.row_fill_fraction(0) == 0.125
    full = engine(small_config(rows=1, cols=4, linear_slots=1024, window=1))
    full.import_row(0, LINEAR, np.zeros(4 * 1024, np.uint8))
    assert full.row_fill_fraction(0) == 1.0


def test_corrected_estimate(gpu, oracle):
    # tests/test_sea.cpp:139-172
    e = engine(small_config(rows=4, linear_slots=1024, recorder_bits=16, window=300, theta=1024))
    for w in (0, 1, 100, 500, 1023):
        assert e.corrected_estimate_from(w, 0.0) == oracle.linear_estimate(w, 1024)
    assert e.corrected_estimate_from(1024, 0.0) is None
    assert e.corrected_estimate_from(4, 0.00390625) == 0.0
    assert e.corrected_estimate_from(3, 0.00390625) == 0.0
    assert e.corrected_estimate_from(300, 0.25 ** 4) == pytest.approx(350.99291022602281, rel=1e-12)
    assert e.corrected_estimate_from(1024, 0.00390625) is None
    assert e.corrected_estimate_from(100, 1.0 - 1e-13) == oracle.linear_estimate(100, 1024)


def test_slide_retains_and_evicts(gpu):
    # tests/test_sea.cpp:204-254
    from paper_1803_10369_b200.srla import INDICATOR, LINEAR, ROUGH
    cfg = small_config()
    e = engine(cfg)
    e.scan_ip_pair(0x0A000006, 0xB0000001)
    assert len(e.slide([])) == 0
    e2 = engine(cfg)
    aip = 0x0A000007
    for i in range(cfg.rows):
        r = e2.export_row(i, ROUGH)
        b = e2.column_of(i, aip) * cfg.rough_slots
        r[b:b + 3] = 0
        e2.import_row(i, ROUGH, r)
    out = e2.slide([aip])
    assert list(out) == [aip]
    e3 = engine(cfg)
    aip = 0x0A000008
    e3.set_candidates([aip])
    e3.scan_pairs([(aip, 0xD0000000 + i) for i in range(40)])
    assert e3.union_rough_weight(aip) >= e3.threshold
    for _ in range(3):
        assert e3.slide_engine() == 1
    assert e3.slide_engine() == 0
    assert e3.union_rough_weight(aip) == 0


def test_window_report_sorted_with_theta_cut(gpu):
    # tests/test_sea.cpp:256-290
    e = engine(small_config(theta=30, rough_slots=32, linear_slots=128))
    assert e.tau == 0
    assert len(e.report_window([])) == 0
    pairs = [(0x0A0000FF, 0xE0000000 + i) for i in range(60)] + [(0x0A000001, 0xE1000000 + i) for i in range(5)]
    e.scan_pairs(pairs)
    csip = list(e.candidates())
    assert 0x0A0000FF in csip
    rep = e.report_window(csip + [0x0A000001])
    assert list(rep["host"]) == [0x0A000001, 0x0A0000FF]
    assert not rep["is_super"][0] and rep["is_super"][1]
    assert rep["has_estimate"].all() and (rep["estimate"] >= 0).all()


def test_errors_follow_reference(gpu):
    from paper_1803_10369_b200.srla import INDICATOR, LINEAR
    e = engine(small_config())
    with pytest.raises(IndexError):
        e.export_row(2, LINEAR)  # std::out_of_range from .at() (sea.hpp:341-346)
    with pytest.raises(ValueError):
        e.import_row(0, INDICATOR, np.zeros(3, np.uint16))


def test_device_generator_byte_identical(gpu, oracle):
    import torch
    from oracle.pyoracle import PlantSpec as OSpec
    from paper_1803_10369_b200.srla import DeviceTraceGenerator, PlantSpec
    for name in ("pipeline_small", "c1_shape"):
        _, (_, spec) = S.SCENARIOS[name]
        want = S.split_by_ts(oracle.generate(OSpec(**spec.__dict__)), spec)
        gen = DeviceTraceGenerator(PlantSpec(**spec.__dict__))
        for s in range(spec.slices):
            got = gen.slice_tensor(s).cpu().numpy().view(np.uint32)
            assert np.array_equal(got, want[s]), (name, s)
    # C2 shape, uniform and Zipf destinations, a later slice (counter skip-ahead)
    for skew in (1.0, 0.0):
        spec = S.Spec(seed=1, slices=3, window=10, a_hosts=4194304, b_hosts=1 << 22, pairs_per_slice=1_000_000,
                      skew=skew, plants=[(0x0AC80001 + i, c, 0, 0xFFFFFFFF) for i, c in enumerate(S.plant_cards())])
        want = S.split_by_ts(oracle.generate(OSpec(**spec.__dict__)), spec)
        gen = DeviceTraceGenerator(PlantSpec(**spec.__dict__))
        got = gen.slice_tensor(2).cpu().numpy().view(np.uint32)
        torch.cuda.synchronize()
        assert np.array_equal(got, want[2])


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("name", ["pipeline_small_3000", "c1_shape", "drift_evict", "contended"])
def test_async_end_slice_matches_sync(gpu, oracle, name, pinned):
    """srla_end_slice_async + the next slice's host scan (copies overlapping the
    end-of-slice work) give the reference pipeline's reports and state."""
    from oracle.pyoracle import SeaConfig as OCfg
    from paper_1803_10369_b200.srla import ENTRY_DTYPE
    cfg, _ = S.SCENARIOS[name]
    slices = GF.scenario_slices(name, oracle)
    pipe = oracle.pipeline(OCfg(**cfg.as_dict()))
    want = [pipe.process_slice(s, r, True) for s, r in enumerate(slices)]
    e = engine(cfg)
    if pinned:  # report entries mapped on the device straight into pinned memory (>= 16k entries)
        import torch
        bufs = [torch.zeros(200000 * 24, dtype=torch.uint8, pin_memory=True).numpy().view(ENTRY_DTYPE)
                for _ in range(2)]
    else:
        bufs = [np.zeros(200000, ENTRY_DTYPE) for _ in range(2)]
    got = []
    for s, recs in enumerate(slices):
        e.scan(recs)
        if s:
            n, _ = e.end_slice_wait()
            got.append(bufs[(s - 1) % 2][:n].copy() if s - 1 + 1 >= cfg.window else None)
        e.end_slice_async(s, bufs[s % 2])
    n, _ = e.end_slice_wait()
    got.append(bufs[(len(slices) - 1) % 2][:n].copy() if len(slices) >= cfg.window else None)
    for s, (g, w) in enumerate(zip(got, want)):
        if w is None:
            assert g is None or len(g) == 0
            continue
        assert np.array_equal(g["host"], w["host"]), s
        assert np.array_equal(g["union_weight"], w["weight"]), s
        assert np.array_equal(g["estimate"].view(np.uint64)[w["has_estimate"] == 1],
                              w["estimate"].view(np.uint64)[w["has_estimate"] == 1]), s
        assert np.array_equal(g["is_super"], w["is_super"]), s
    assert np.array_equal(e.candidates(), pipe.candidates())


@pytest.mark.parametrize("epoch", ["0", "1"])
@pytest.mark.parametrize("name", ["contended", "drift_evict", "c1_shape"])
def test_async_end_slice_overlaps_next_device_scan(gpu, oracle, name, epoch, monkeypatch):
    """srla_end_slice_async + the next slice's DEVICE scan: K1 bins into the
    second bin set while the end-of-slice runs (binned marks forced on), and
    the reports, candidate list and recorders stay the reference's."""
    import torch
    from oracle.pyoracle import SeaConfig as OCfg
    from paper_1803_10369_b200.srla import ENTRY_DTYPE
    monkeypatch.setenv("SRLA_FORCE_BINS", "1")
    monkeypatch.setenv("SRLA_EPOCH", epoch)
    monkeypatch.setenv("SRLA_OVERLAP", "1")
    monkeypatch.setenv("SRLA_SMALL_BIN_ENTRIES", str(1 << 20))  # room for a whole slice per bin set
    cfg, _ = S.SCENARIOS[name]
    slices = GF.scenario_slices(name, oracle)
    pipe = oracle.pipeline(OCfg(**cfg.as_dict()))
    want = [pipe.process_slice(s, r, True) for s, r in enumerate(slices)]
    e = engine(cfg)
    bufs = [np.zeros(200000, ENTRY_DTYPE) for _ in range(2)]
    dev = [torch.from_numpy(r.astype(np.int32)).cuda() for r in slices]
    torch.cuda.synchronize()
    got = []
    for s in range(len(slices)):
        e.scan(dev[s])
        if s:
            n, _ = e.end_slice_wait()
            got.append(bufs[(s - 1) % 2][:n].copy() if s >= cfg.window else None)
        e.end_slice_async(s, bufs[s % 2])
    n, _ = e.end_slice_wait()
    got.append(bufs[(len(slices) - 1) % 2][:n].copy() if len(slices) >= cfg.window else None)
    assert e.stats()["overlapped_chunks"] > 0
    for s, (g, w) in enumerate(zip(got, want)):
        if w is None:
            assert g is None or len(g) == 0
            continue
        assert np.array_equal(g["host"], w["host"]), s
        assert np.array_equal(g["union_weight"], w["weight"]), s
        assert np.array_equal(g["estimate"].view(np.uint64)[w["has_estimate"] == 1],
                              w["estimate"].view(np.uint64)[w["has_estimate"] == 1]), s
    assert np.array_equal(e.candidates(), pipe.candidates())
    for i in range(cfg.rows):
        for kind in (1, 2):
            assert np.array_equal(e.export_row(i, kind), pipe.sketch.export_row(i, kind)), (i, kind)


@pytest.mark.parametrize("bits,window", [(4, 5), (7, 100), (3, 7)])
def test_epoch_stamps_survive_counter_wrap(gpu, oracle, bits, window, monkeypatch):
    """600 slides (the u8 epoch counter wraps twice): hosts fall silent for
    hundreds of slices, so only the sweep keeps old stamps from aliasing."""
    monkeypatch.setenv("SRLA_FORCE_BINS", "1")
    cfg = S.Cfg(rows=2, cols=64, rough_slots=8, linear_slots=32, recorder_bits=bits, window=window, theta=16,
                seed=0xE90C + bits)
    rng = np.random.default_rng(bits)
    slices = []
    for s in range(600):
        n = int(rng.integers(0, 60)) if (s // 97) % 2 == 0 else int(rng.integers(0, 4))
        r = np.zeros((n, 3), np.uint32)
        r[:, 1] = 0x0A000000 + rng.integers(0, 40, n)
        r[:, 2] = 0xB0000000 + rng.integers(0, 300, n)
        slices.append(r)
    a = GF.run_flow(_oracle_backend(oracle, cfg), cfg, slices)
    b = GF.run_flow(GF.EngineBackend(engine(cfg)), cfg, slices)
    msg = GF.compare(a, b)
    assert msg is None, msg


def test_epoch_import_out_of_model_values_falls_back_to_literal(gpu, oracle, monkeypatch):
    """Recorder values above `expired` (possible through the row spans) are
    outside the epoch model: the engine converts to literal recorders."""
    from paper_1803_10369_b200.srla import LINEAR
    monkeypatch.setenv("SRLA_FORCE_BINS", "1")
    cfg = S.Cfg(rows=2, cols=64, rough_slots=8, linear_slots=32, recorder_bits=4, window=5, theta=16, seed=77)
    e, o = engine(cfg), _oracle_backend(oracle, cfg)
    slices = S.random_slices(3, 6, (100, 400), 30, 200)
    for s in slices[:3]:
        e.scan_collect(s)
        o.scan(s)
    row = e.export_row(1, LINEAR)
    assert np.array_equal(row, o.sk.export_row(1, LINEAR))
    row[::7] = 200  # > expired = 15
    e.import_row(1, LINEAR, row)
    o.sk.import_row(1, LINEAR, row)
    rest = GF.run_flow(GF.EngineBackend(e), cfg, slices[3:])
    want = GF.run_flow(o, cfg, slices[3:])
    assert GF.compare(want, rest) is None


def test_large_report_mapped_on_device_into_pinned_buffer(gpu, oracle):
    """>16k report entries: estimates are mapped on the GPU from the host LUT and
    written straight into a pinned caller buffer (UVA); must equal the reference."""
    import torch
    from oracle.pyoracle import SeaConfig as OCfg
    from paper_1803_10369_b200.srla import ENTRY_DTYPE
    cfg = S.Cfg(rows=2, cols=65536, rough_slots=8, linear_slots=64, recorder_bits=4, window=3, theta=8, seed=0x51A)
    slices = S.random_slices(8, 5, (200000, 200000), 50000, 1000)
    pipe = oracle.pipeline(OCfg(**cfg.as_dict()))
    e = engine(cfg)
    buf = torch.zeros(100000 * 24, dtype=torch.uint8, pin_memory=True).numpy().view(ENTRY_DTYPE)
    seen_large = False
    for s, recs in enumerate(slices):
        w = pipe.process_slice(s, recs, True)
        e.scan(recs)
        e.end_slice_async(s, buf)
        n, _ = e.end_slice_wait()
        if w is None:
            continue
        seen_large |= n >= (1 << 14)
        g = buf[:n]
        assert np.array_equal(g["host"], w["host"]) and np.array_equal(g["union_weight"], w["weight"])
        m = w["has_estimate"] == 1
        assert np.array_equal(g["has_estimate"], w["has_estimate"]) and np.array_equal(g["is_super"], w["is_super"])
        assert np.array_equal(g["estimate"].view(np.uint64)[m], w["estimate"].view(np.uint64)[m])
    assert seen_large


@pytest.mark.parametrize("name", ["pipeline_small_3000", "contended", "drift_evict"])
def test_compact_report_handoff(gpu, oracle, name):
    """srla_end_slice_compact: hosts + weights + the window's Eq. 9 table give
    the reference's entries exactly."""
    from oracle.pyoracle import SeaConfig as OCfg
    cfg, _ = S.SCENARIOS[name]
    slices = GF.scenario_slices(name, oracle)
    pipe = oracle.pipeline(OCfg(**cfg.as_dict()))
    e = engine(cfg)
    hosts, w = np.zeros(100000, np.uint32), np.zeros(100000, np.uint32)
    est, flags = np.zeros(cfg.linear_slots + 1), np.zeros(cfg.linear_slots + 1, np.uint8)
    for s, recs in enumerate(slices):
        want = pipe.process_slice(s, recs, True)
        e.scan(recs)
        n, _ = e.end_slice_compact(s, hosts, w, est, flags)
        if want is None:
            assert n == 0
            continue
        assert np.array_equal(hosts[:n], want["host"]) and np.array_equal(w[:n], want["weight"])
        has = flags[w[:n]] & 1
        assert np.array_equal(has, want["has_estimate"])
        assert np.array_equal(flags[w[:n]] >> 1, want["is_super"])
        m = has == 1
        assert np.array_equal(est[w[:n]][m].view(np.uint64), want["estimate"][m].view(np.uint64))
    assert np.array_equal(e.candidates(), pipe.candidates())


@pytest.mark.parametrize("mode", ["literal", "nibble", "epoch", "w2"])
def test_state_blocks_match_exported_rows(gpu, oracle, mode, monkeypatch):
    """srla_state_blocks (device digests in the reference layout) equals the
    digest of the exported rows for every table representation, and
    srla_block_sums equals it on raw device bytes of ragged sizes."""
    import torch
    from paper_1803_10369_b200 import srla
    name = {"w2": "wide_w2"}.get(mode, "contended")
    monkeypatch.setenv("SRLA_FORCE_BINS", "1")
    monkeypatch.setenv("SRLA_EPOCH", "1" if mode == "epoch" else "0")
    monkeypatch.setenv("SRLA_NIBBLE", "1" if mode == "nibble" else "0")
    cfg, _ = S.SCENARIOS[name]
    e = engine(cfg)
    for sid, recs in enumerate(GF.scenario_slices(name, oracle)[:4]):
        e.scan(recs)
        e.end_slice(sid)
    for i in range(cfg.rows):
        for k in (0, 1, 2):
            assert np.array_equal(e.state_blocks(i, k), GF.block_sums_np(e.export_row(i, k))), (i, k)
    rng = np.random.default_rng(1)
    for n in (1, 13, (1 << 20) + 3, 5 << 20):
        b = rng.integers(0, 256, n, dtype=np.uint8)
        assert np.array_equal(srla.block_sums(torch.from_numpy(b).cuda()), GF.block_sums_np(b)), n


def test_device_records_contract(gpu, oracle):
    """Device batches: read after the producer stream's work (torch's current
    stream is passed as srla_scan_device's producer), and rejected unless
    (n, 3) int32/uint32, contiguous, on the engine's GPU."""
    import torch
    name = "contended"
    cfg, _ = S.SCENARIOS[name]
    slices = GF.scenario_slices(name, oracle)[:3]
    want = engine(cfg)
    got = engine(cfg)
    side = torch.cuda.Stream()
    for s, recs in enumerate(slices):
        host = torch.from_numpy(np.ascontiguousarray(recs, dtype=np.uint32).view(np.int32))
        with torch.cuda.stream(side):  # produced (and scanned) on a non-default stream
            torch.cuda._sleep(2_000_000)  # the copy lands well after the call is queued
            dev = host.to("cuda", non_blocking=False)
            got.scan(dev)
        want.scan(recs)
        a, _ = want.end_slice(s)
        b, _ = got.end_slice(s)
        assert (a is None and b is None) or a.tobytes() == b.tobytes()
    assert np.array_equal(want.candidates(), got.candidates())
    t = torch.zeros((10, 3), dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError, match="int32"):
        got.scan(t)
    with pytest.raises(ValueError, match="shape"):
        got.scan(torch.zeros((10, 2), dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError, match="contiguous"):
        got.scan(torch.zeros((3, 10), dtype=torch.int32, device="cuda").t())
