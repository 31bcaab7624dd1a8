"""Edge cases of the record batches the reference accepts (pipeline.hpp:110-158,
sea.hpp:150-196): empty slices, single records, sizes straddling K1's
4-record vectors and 2048-packet tiles, many tiny batches (the one-thread
serial path) interleaved with large ones, and device records at an address
that is not 16-byte aligned. Every slice must match the oracle pipeline
(pushes, ordered candidates, report entries with estimate bits, retained
list, recorder digests) on the same records in the same order."""
from __future__ import annotations

import numpy as np
import pytest

import golden_flow as GF
import scenarios as S

pytestmark = pytest.mark.gpu

RAGGED = [0, 1, 3, 4, 5, 2047, 2048, 2049, 0, 0, 4095, 8193, 63, 64, 65, 1]


def _engine(cfg):
    from paper_1803_10369_b200.srla import EstimatorArray, SeaConfig
    return EstimatorArray(SeaConfig(**cfg.as_dict()))


def _oracle(oracle, cfg):
    return GF.CheckerBackend(oracle, cfg)


def _ragged_slices(oracle, name):
    """The scenario's records re-cut into the RAGGED sizes, then the rest in
    three slices; timestamps are not read by the scan."""
    recs = np.concatenate(GF.scenario_slices(name, oracle))
    out, o = [], 0
    for n in RAGGED:
        out.append(recs[o:o + n])
        o += n
    rest = recs[o:]
    out.extend(np.array_split(rest, 3))
    return out


@pytest.mark.parametrize("bins", ["default", "forced", "forced_nohoist"])
@pytest.mark.parametrize("name", ["contended", "drift_evict", "pipeline_small"])
def test_ragged_and_empty_slices(gpu, oracle, name, bins, monkeypatch):
    if bins != "default":
        monkeypatch.setenv("SRLA_FORCE_BINS", "1")  # tiny bins: the overflow paths run too
    if bins == "forced_nohoist":  # K1's per-mark filter test and scatter tests (the A/B path)
        monkeypatch.setenv("SRLA_K1_HOIST", "0")
    cfg, _ = S.SCENARIOS[name]
    slices = _ragged_slices(oracle, name)
    a = GF.run_flow(_oracle(oracle, cfg), cfg, slices)
    b = GF.run_flow(GF.EngineBackend(_engine(cfg)), cfg, slices)
    msg = GF.compare(a, b)
    assert msg is None, msg
    assert sum(s["report"] is not None for s in a) >= 5


def test_tiny_batches_interleaved_with_large(gpu, oracle):
    """Batches of 1..70 records (the <= 64-record serial path and just above it)
    between large ones, inside every slice: the running in-slice packet index
    carries across calls (srla_scan_batch may be called repeatedly per slice)."""
    cfg, _ = S.SCENARIOS["drift_evict"]
    slices = GF.scenario_slices("drift_evict", oracle)
    ref = GF.run_flow(_oracle(oracle, cfg), cfg, slices)

    class Tiny(GF.EngineBackend):
        def scan(self, recs):
            rng = np.random.default_rng(len(recs) + 7)
            out, o = [], 0
            while o < len(recs):
                n = int(rng.integers(1, 71)) if rng.random() < 0.7 else int(rng.integers(500, 5000))
                out.append(self.e.scan_collect(recs[o:o + n]))
                o += n
            return np.concatenate(out) if out else np.empty(0, np.uint32)

    got = GF.run_flow(Tiny(_engine(cfg)), cfg, slices)
    msg = GF.compare(ref, got)
    assert msg is None, msg


def test_unaligned_device_records(gpu, oracle):
    """Device batches starting 12 bytes into an allocation (K1's 16-byte vector
    loads are off) give the host path's results."""
    import torch
    cfg, _ = S.SCENARIOS["contended"]
    slices = GF.scenario_slices("contended", oracle)
    ref = GF.run_flow(_oracle(oracle, cfg), cfg, slices)

    class Unaligned(GF.EngineBackend):
        def scan(self, recs):
            t = torch.zeros((len(recs) + 1, 3), dtype=torch.int32, device="cuda")
            t[1:] = torch.from_numpy(recs.astype(np.int32)).cuda()
            v = t[1:]
            assert v.data_ptr() % 16 == 12
            torch.cuda.synchronize()
            return self.e.scan_collect(v)

    got = GF.run_flow(Unaligned(_engine(cfg)), cfg, slices)
    msg = GF.compare(ref, got)
    assert msg is None, msg


def _u32(seed, index, key):
    """HashFamily::u32 (hash.hpp:53-62) in numpy: the sample hash of a bip."""
    def av(x):
        with np.errstate(over="ignore"):
            x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return x ^ (x >> np.uint64(31))
    with np.errstate(over="ignore"):
        sub = av(np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * np.uint64(index + 1))
    return (av(sub ^ np.asarray(key, dtype=np.uint64)) & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def test_every_packet_sampled_overflows_event_list(gpu, oracle):
    """Slices whose every destination passes the sampling test (ctz of the
    sample hash >= tau): 1.2x more sampled packets than the event list sized for
    an ordinary 2^27-record chunk (2^27 >> tau + ...), so the ordering phase
    grows it and reruns K1; thousands of hosts cross at once. The hash the
    destinations are picked with is checked against the reference's first."""
    cfg, _ = S.SCENARIOS["contended"]
    assert [int(x) for x in _u32(cfg.seed, 0, np.array([0, 1, 12345], np.uint64))] == \
        [oracle.hash_u32(cfg.seed, 0, k) for k in (0, 1, 12345)]
    e = _engine(cfg)
    tau = e.tau
    assert tau >= 5
    rng = np.random.default_rng(11)
    cand = rng.integers(0, 2**32, 8_000_000, dtype=np.uint64)
    h = _u32(cfg.seed, 0, cand)
    sampled = cand[(h & np.uint32((1 << tau) - 1)) == 0].astype(np.uint32)
    assert len(sampled) > 20000
    base = GF.scenario_slices("contended", oracle)
    slices = []
    # the fast path's initial event list (Engine::scan_chunk_fast), overshot by 20%
    ev_cap = (1 << 27 >> tau) + (1 << 27 >> (tau + 3)) + 65536
    for s in range(2):
        n = ev_cap * 6 // 5
        r = np.zeros((n, 3), np.uint32)
        r[:, 1] = 0x0A000000 + rng.integers(0, 6000, n).astype(np.uint32)
        r[:, 2] = sampled[rng.integers(0, len(sampled), n)]
        slices.append(r)
    slices += base[:cfg.window]
    a = GF.run_flow(_oracle(oracle, cfg), cfg, slices)
    b = GF.run_flow(GF.EngineBackend(e), cfg, slices)
    msg = GF.compare(a, b)
    assert msg is None, msg
    assert a[0]["pushes"]["n"] > 1000


def test_large_host_batch_equals_device_batch(gpu):
    """A 40M-record host batch (pinned and pageable) crosses in staged 16M-record
    chunks, each scanned as it lands, and must leave exactly the pushes, the
    candidates and the recorder state that the same records scanned from HBM
    leave."""
    import torch
    from paper_1803_10369_b200 import srla
    from paper_1803_10369_b200 import workloads as WL
    cfg = WL.sketch_cfg(1 << 16)
    gen = srla.DeviceTraceGenerator(srla.PlantSpec(**WL.trace_spec(40_000_000, slices=2)))
    t = gen.slice_tensor(0)
    host = t.cpu().numpy().view(np.uint32)
    pinned = torch.from_numpy(host.copy()).pin_memory().numpy()
    out = []
    for src in (t, host, pinned):
        e = srla.EstimatorArray(srla.SeaConfig(**cfg))
        pushes = e.scan_collect(src)
        blocks = [e.state_blocks(i, k).tobytes() for i in range(cfg["rows"]) for k in (0, 1, 2)]
        out.append((pushes.tolist(), e.candidates().tolist(), blocks))
    assert out[0][0] == out[1][0] == out[2][0] and len(out[0][0]) > 0
    assert out[0][1] == out[1][1] == out[2][1]
    assert out[0][2] == out[1][2] == out[2][2]
