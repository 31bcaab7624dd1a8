"""Adversarial-skew parity and size-independent properties
at BASELINE.json's full sizes, where the single-threaded oracle would take
minutes:

* C5 shape at reduced scale (one host contacted by every destination of the
  slice plus a uniform scan storm over many sources): bit-exact against the C
  restatement, literal and epoch-stamp recorders;
* C2 at full size (1e8 packets per slice, v = 2^20): every rough and linear
  recorder equal to the reference's own DetectPipeline run with all host
  threads (recorder end state is order independent; the candidate list is
  not — the multi-worker reference reorders it — so it is not compared here);
* C2 at full size: the two mark paths of the engine (binned two-level apply and
  epoch stamps) agree on every report entry, candidate list and recorder.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import golden_flow as GF
import scenarios as S

pytestmark = pytest.mark.gpu


def _oracle_backend(oracle, cfg):
    b = GF.CheckerBackend.__new__(GF.CheckerBackend)
    from oracle.pyoracle import SeaConfig
    b.sk, b.csip, b.seen = oracle.sketch(SeaConfig(**cfg.as_dict())), [], set()
    return b


def _engine(cfg: S.Cfg):
    from paper_1803_10369_b200.srla import EstimatorArray, SeaConfig
    return EstimatorArray(SeaConfig(**cfg.as_dict()))


C2_SKETCH = dict(rows=4, rough_slots=8, linear_slots=1024, recorder_bits=4, window=10, theta=1024, seed=0x5EA00001)


@pytest.mark.parametrize("epoch", ["0", "1"])
def test_c5_adversarial_skew_medium(gpu, oracle, epoch, monkeypatch):
    """C5 at 1/50 scale: PlantSpec.window = 1 so the hot host meets all of its
    200k peers in every slice (first in the slice, generator.hpp:132-154), then
    a uniform storm of 2e6 pairs from 240k sources over 2^24 destinations."""
    from oracle.pyoracle import PlantSpec
    monkeypatch.setenv("SRLA_FORCE_BINS", "1")
    monkeypatch.setenv("SRLA_EPOCH", epoch)
    spec = S.Spec(seed=5, slices=11, window=1, a_hosts=240_000, b_hosts=1 << 24, pairs_per_slice=2_000_000,
                  skew=0.0, plants=[(0x0AC80001, 200_000, 0, 0xFFFFFFFF)])
    recs = oracle.generate(PlantSpec(**spec.__dict__))
    slices = S.split_by_ts(recs, spec)
    assert len(slices) == 11 and all(len(s) == 2_200_000 for s in slices)
    cfg = S.Cfg(cols=1 << 16, **C2_SKETCH)
    a = GF.run_flow(_oracle_backend(oracle, cfg), cfg, slices)
    b = GF.run_flow(GF.EngineBackend(_engine(cfg)), cfg, slices)
    msg = GF.compare(a, b)
    assert msg is None, msg
    assert a[-1]["report"] is not None and sum(s["pushes"]["n"] for s in a) > 100


def _c2_slices(n_slices, pairs=100_000_000):
    from paper_1803_10369_b200.srla import DeviceTraceGenerator, PlantSpec
    spec = dict(seed=1, slices=n_slices, window=10, a_hosts=4194304, b_hosts=1 << 22, pairs_per_slice=pairs,
                skew=1.0, plants=[(0x0AC80001 + i, c, 0, 0xFFFFFFFF) for i, c in enumerate(S.plant_cards())])
    gen = DeviceTraceGenerator(PlantSpec(**spec))
    return [gen.slice_tensor(s) for s in range(n_slices)]


@pytest.mark.slow
def test_c2_fullsize_recorders_match_reference_threads(gpu):
    """Two full C2 slices (1e8 packets each, 4 GiB linear table): every rough
    and linear recorder of the engine equals the reference DetectPipeline's
    (oracle/_ref, workers = all host threads) after each slice's slide."""
    from oracle.pyoracle import LIBS, LINEAR, ROUGH, Checker, SeaConfig
    if not os.path.exists(LIBS["ref"]):
        pytest.skip("oracle/_ref not built")
    ref = Checker("ref")
    cfg = dict(cols=1 << 20, **C2_SKETCH)
    pipe = ref.pipeline(SeaConfig(**cfg), workers=os.cpu_count() or 1)
    eng = _engine(S.Cfg(**cfg))
    for sid, t in enumerate(_c2_slices(2)):
        host = t.cpu().numpy().view(np.uint32).reshape(-1, 3)
        pipe.process_slice(sid, host, True)
        eng.scan(t)
        eng.end_slice(sid, want_report=True)
        for i in range(4):
            for kind in (ROUGH, LINEAR):
                want = pipe.sketch.export_row(i, kind)
                got = eng.export_row(i, kind)
                assert np.array_equal(want, got), f"slice {sid} row {i} kind {kind}: recorders differ"
        del host


@pytest.mark.slow
def test_c2_fullsize_epoch_and_literal_paths_agree(gpu, monkeypatch):
    """Full C2 slices through two engines whose linear tables take different
    code paths (literal recorders with the fused count+age apply, and epoch
    stamps with histogram counts): identical candidates, report entries
    (estimate bits included) and recorders after 11 slices."""
    slices = _c2_slices(11)
    cfg = S.Cfg(cols=1 << 20, **C2_SKETCH)
    runs = []
    for epoch in ("0", "1"):
        monkeypatch.setenv("SRLA_EPOCH", epoch)
        eng = _engine(cfg)
        reps, cands = [], []
        for sid, t in enumerate(slices):
            eng.scan(t)
            cands.append(eng.candidates())
            r, _ = eng.end_slice(sid, want_report=True)
            if r is not None:
                reps.append(r.copy())
        rows = [(eng.export_row(i, 1), eng.export_row(i, 2)) for i in range(cfg.rows)]
        runs.append((reps, cands, rows))
        del eng
    (ra, ca, sa), (rb, cb, sb) = runs
    assert len(ra) == len(rb) == 2
    for x, y in zip(ca, cb):
        assert np.array_equal(x, y)
    for x, y in zip(ra, rb):
        assert x.tobytes() == y.tobytes()
        assert len(x) > 1000
    for (r1, l1), (r2, l2) in zip(sa, sb):
        assert np.array_equal(r1, r2) and np.array_equal(l1, l2)


@pytest.mark.slow
def test_c2_fullsize_overlapped_pipeline_matches_sync(gpu, monkeypatch):
    """The bench's overlapped pipeline (srla_end_slice_async, next slice's K1
    binned under it) against synchronous end-of-slice on the same full C2
    slices: identical report entries and recorders."""
    import torch
    from paper_1803_10369_b200.srla import ENTRY_DTYPE
    slices = _c2_slices(11)
    cfg = S.Cfg(cols=1 << 20, **C2_SKETCH)
    sync = _engine(cfg)
    want = []
    for sid, t in enumerate(slices):
        sync.scan(t)
        r, _ = sync.end_slice(sid, want_report=True)
        want.append(None if r is None else r.copy())
    want_rows = [(sync.export_row(i, 1), sync.export_row(i, 2)) for i in range(cfg.rows)]
    del sync
    monkeypatch.setenv("SRLA_OVERLAP", "1")
    e = _engine(cfg)
    bufs = [torch.empty((2 << 20) * ENTRY_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True).numpy().view(ENTRY_DTYPE)
            for _ in range(2)]
    got = []
    for sid, t in enumerate(slices):
        e.scan(t)
        if sid:
            n, _ = e.end_slice_wait()
            got.append(bufs[(sid - 1) % 2][:n].copy() if sid >= cfg.window else None)
        e.end_slice_async(sid, bufs[sid % 2])
    n, _ = e.end_slice_wait()
    got.append(bufs[(len(slices) - 1) % 2][:n].copy())
    assert e.stats()["overlapped_chunks"] >= 9
    for g, w in zip(got, want):
        assert (g is None) == (w is None)
        if w is not None:
            assert g.tobytes() == w.tobytes()
    for (r1, l1), (r2, l2) in zip(want_rows, [(e.export_row(i, 1), e.export_row(i, 2)) for i in range(cfg.rows)]):
        assert np.array_equal(r1, r2) and np.array_equal(l1, l2)


@pytest.mark.slow
def test_c3_row_export_import_on_device(gpu):
    """Snapshot rows at the 2^24-column scale (§8f rank 3): a 16 GiB
    epoch-stamp linear row exports as the reference's literal values (converted
    on the device), its active count equals count_active, and an import of a
    modified row round-trips exactly."""
    import time
    from paper_1803_10369_b200.srla import DeviceTraceGenerator, EstimatorArray, PlantSpec, SeaConfig
    cfg = SeaConfig(rows=4, cols=1 << 24, **{k: v for k, v in C2_SKETCH.items() if k != "rows"})
    e = EstimatorArray(cfg)
    gen = DeviceTraceGenerator(PlantSpec(seed=3, slices=2, window=10, a_hosts=1 << 20, b_hosts=1 << 24,
                                         pairs_per_slice=10_000_000, skew=0.0, plants=[]))
    for sid in range(2):
        e.scan(gen.slice_tensor(sid))
        e.end_slice(sid, want_report=True)
    t0 = time.perf_counter()
    row = e.export_row(1, 2)
    t_export = time.perf_counter() - t0
    assert row.nbytes == (1 << 24) * 1024 and int(row.max()) <= 15
    assert int(np.count_nonzero(row < cfg.window)) == int(e.row_active()[1])
    row[::4096] = 3
    t0 = time.perf_counter()
    e.import_row(1, 2, row)
    t_import = time.perf_counter() - t0
    back = e.export_row(1, 2)
    assert np.array_equal(back, row)
    assert int(e.row_active()[1]) == int(np.count_nonzero(row < cfg.window))
    print(f"16 GiB row: export {t_export:.2f} s, import {t_import:.2f} s")
