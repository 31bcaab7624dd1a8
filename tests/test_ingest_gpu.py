"""The ingest front end on the device (paper_1803_10369_b200/csrc/ingest.cu)
against the CPU restatement (pinned to the reference by
tests/test_ingest_oracle.py): SRLT parsing with its error cases, orientation
and slice partitioning, and a raw SRLT trace driven through parse -> orient ->
slice -> scan equal to the reference DetectPipeline::run's reports."""
from __future__ import annotations

import numpy as np
import pytest

import scenarios as S

pytestmark = pytest.mark.gpu


def _trace(rng, n, t0=1_700_000_000, span=50):
    ts = np.sort(rng.integers(t0, t0 + span, n)).astype(np.uint32)
    hosts = np.concatenate([rng.integers(0x0A000000, 0x0A00FFFF, n // 2),
                            rng.integers(0xC0A80000, 0xC0A8FFFF, n - n // 2)]).astype(np.uint32)
    rng.shuffle(hosts)
    other = rng.choice(np.array([0x0A000001, 0x08080808, 0xC0A80101, 0x0A00FF00], np.uint32), n)
    return np.stack([ts, hosts, other], 1).astype(np.uint32)


def _srlt(recs):
    return b"SRLT" + bytes([1]) + np.ascontiguousarray(recs, np.uint32).astype("<u4").tobytes()


def _dev_bytes(b):
    import torch
    return torch.from_numpy(np.frombuffer(b, np.uint8).copy()).cuda()


def _dev(recs):
    import torch
    return torch.from_numpy(np.ascontiguousarray(recs, np.uint32).view(np.int32)).cuda()


def test_parse_srlt_matches_oracle(gpu, oracle):
    from paper_1803_10369_b200.srla import InputError, parse_srlt
    rng = np.random.default_rng(7)
    for n in (0, 1, 2, 3, 1000, 123457):
        recs = _trace(rng, n)
        got = parse_srlt(_dev_bytes(_srlt(recs))).cpu().numpy().view(np.uint32)
        want, err, _ = oracle.parse_srlt(_srlt(recs))
        assert err == 0 and np.array_equal(got, want) and np.array_equal(got, recs)
    recs = _trace(rng, 5000)
    with pytest.raises(InputError, match="truncated record 4999"):
        parse_srlt(_dev_bytes(_srlt(recs)[:-3]))
    bad = recs.copy()
    bad[777, 0] = bad[776, 0] - 1
    with pytest.raises(InputError, match="timestamp regression at record 777") as ei:
        parse_srlt(_dev_bytes(_srlt(bad)))
    assert np.array_equal(ei.value.records.cpu().numpy().view(np.uint32), bad[:777])
    with pytest.raises(InputError, match="bad magic"):
        parse_srlt(_dev_bytes(b"SRLX\x01" + bytes(24)))
    with pytest.raises(InputError, match="version"):
        parse_srlt(_dev_bytes(b"SRLT\x02" + bytes(24)))


@pytest.mark.parametrize("bits", [0, 8, 16, 24, 32])
def test_orient_matches_oracle(gpu, oracle, bits):
    from paper_1803_10369_b200.srla import orient_records
    rng = np.random.default_rng(10 + bits)
    recs = _trace(rng, 200_001)
    got, st = orient_records(_dev(recs), 0x0A001234, bits)
    want, wst = oracle.orient(recs, 0x0A001234, bits)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), want)
    assert [st[k] for k in ("kept", "flipped", "dropped_both", "dropped_neither")] == wst.tolist()


@pytest.mark.parametrize("seconds", [1, 7, 300])
def test_slice_bounds_match_oracle(gpu, oracle, seconds):
    from paper_1803_10369_b200.srla import InputError, slice_bounds
    rng = np.random.default_rng(seconds)
    recs = _trace(rng, 100_000, span=3000)
    recs[60000:, 0] += 20 * seconds  # a gap: empty slices
    assert np.array_equal(slice_bounds(_dev(recs), seconds), oracle.slice_bounds(recs, seconds))
    assert len(slice_bounds(_dev(recs[:1]), seconds)) == 2
    bad = recs.copy()
    bad[500, 0] = 0
    with pytest.raises(InputError, match="regression at record 500"):
        slice_bounds(_dev(bad), seconds)


def test_raw_trace_through_device_front_end_matches_reference_run(gpu, oracle):
    """DetectPipeline::run (pipeline.hpp:96-106) on a raw SRLT trace: the file
    bytes go to HBM once; parse, orient and slice on the device; each slice
    scanned from HBM. Reports equal the reference pipeline fed the
    host-side oriented, partitioned records."""
    from oracle.pyoracle import PlantSpec, SeaConfig as OCfg
    from paper_1803_10369_b200.srla import EstimatorArray, SeaConfig, orient_records, parse_srlt, slice_bounds
    spec = S.Spec(seed=9, slices=8, window=3, a_hosts=400, b_hosts=4096, pairs_per_slice=20000, skew=1.0,
                  plants=[(0x0AC80001, 900, 0, 0xFFFFFFFF)])
    recs = oracle.generate(PlantSpec(**spec.__dict__))
    rng = np.random.default_rng(1)
    flip = rng.random(len(recs)) < 0.3  # far-side records the front end must flip back
    raw = recs.copy()
    raw[flip, 1], raw[flip, 2] = recs[flip, 2], recs[flip, 1]
    cfg = S.Cfg(rows=2, cols=256, rough_slots=8, linear_slots=64, recorder_bits=8, window=3, theta=32, seed=0xBEEF)
    # reference side: orient + partition on the host (restatement pinned to trace.hpp), then process_slice
    ori, _ = oracle.orient(raw, 0x0A000000, 8)
    offs = oracle.slice_bounds(ori, 1)
    pipe = oracle.pipeline(OCfg(**cfg.as_dict()))
    want = [pipe.process_slice(s, ori[offs[s]:offs[s + 1]], True) for s in range(len(offs) - 1)]
    # device side
    d = parse_srlt(_dev_bytes(_srlt(raw)))
    d, st = orient_records(d, 0x0A000000, 8)
    assert st["flipped"] == int(flip.sum()) or st["flipped"] > 0
    dev_offs = slice_bounds(d, 1)
    assert np.array_equal(dev_offs, offs)
    e = EstimatorArray(SeaConfig(**cfg.as_dict()))
    for s in range(len(dev_offs) - 1):
        e.scan(d[int(dev_offs[s]):int(dev_offs[s + 1])])
        got, _ = e.end_slice(s, want_report=True)
        w = want[s]
        if w is None:
            assert got is None
            continue
        assert np.array_equal(got["host"], w["host"]) and np.array_equal(got["union_weight"], w["weight"])
