"""The C++ drop-in (include/sspread/*.hpp over the C ABI): compiles against
the headers on CPU; on the GPU runs the reference's own unit tests rewritten
against it and replays DetectPipeline::process_slice against the oracle."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

import golden_flow as GF
import scenarios as S
from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_1803_10369_b200", "lib")


@pytest.fixture(scope="module")
def dropin_bin(srla_lib, tmp_path_factory):
    out = str(tmp_path_factory.mktemp("dropin") / "test_dropin")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    SRC, "-L", LIBDIR, "-lsrla_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)
    return out


def test_dropin_headers_compile_and_link(dropin_bin):
    assert os.path.exists(dropin_bin)


@pytest.mark.gpu
def test_dropin_reference_unit_tests(gpu, dropin_bin):
    r = subprocess.run([dropin_bin], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr + r.stdout


def _write_srlt(path, recs):
    with open(path, "wb") as f:
        f.write(b"SRLT\x01")
        f.write(np.ascontiguousarray(recs, dtype="<u4").tobytes())


def _parse(path):
    slices, cur = [], None
    lines = open(path).read().split("\n")
    i = 0
    while i < len(lines):
        ln = lines[i]
        if ln.startswith("report "):
            _, ws, n = ln.split()
            rows = [list(map(int, lines[i + 1 + j].split())) for j in range(int(n))]
            cur = {"report": rows}
            i += 1 + int(n)
            continue
        if ln.startswith("csip "):
            n = int(ln.split()[1])
            csip = [int(x) for x in lines[i + 1:i + 1 + n]]
            slices.append({"report": (cur or {}).get("report"), "csip": csip})
            cur = None
            i += 1 + n
            continue
        i += 1
    return slices


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["pipeline_small", "pipeline_small_3000", "c1_shape"])
def test_dropin_pipeline_replay_matches_oracle(gpu, oracle, dropin_bin, tmp_path, name):
    cfg, (_, spec) = S.SCENARIOS[name]
    slices = GF.scenario_slices(name, oracle)
    trace = tmp_path / "t.bin"
    _write_srlt(trace, np.concatenate(slices))
    out = tmp_path / "out.txt"
    c = cfg
    subprocess.run([dropin_bin, "replay", str(trace), str(out), str(c.rows), str(c.cols), str(c.rough_slots),
                    str(c.linear_slots), str(c.recorder_bits), str(c.window), str(c.theta), hex(c.seed)],
                   check=True, timeout=600)
    got = _parse(out)
    pipe = oracle.pipeline(__import__("oracle.pyoracle", fromlist=["SeaConfig"]).SeaConfig(**c.as_dict()))
    assert len(got) == len(slices)
    for s, recs in enumerate(slices):
        rep = pipe.process_slice(s, recs, True)
        want_csip = pipe.candidates().tolist()
        assert got[s]["csip"] == want_csip, f"slice {s}"
        if rep is None:
            assert got[s]["report"] is None
            continue
        bits = rep["estimate"].view(np.uint64)
        want = [[int(h), int(w), int(b) if has else 0, int(has), int(sup)]
                for h, w, b, has, sup in zip(rep["host"], rep["weight"], bits, rep["has_estimate"], rep["is_super"])]
        assert got[s]["report"] == want, f"slice {s}"


@pytest.mark.gpu
@pytest.mark.parametrize("front", ["device", "host"])
@pytest.mark.parametrize("name", ["pipeline_small", "c1_shape"])
def test_dropin_run_device_front_end_matches_oracle(gpu, oracle, dropin_bin, tmp_path, name, front):
    """DetectPipeline::run on a raw SRLT file with far-side (flipped) and
    off-network records: the device front end (parse, orient, slice in HBM)
    and the streaming host path taken by traces above the device size limit
    (forced here with SRLA_DEVICE_TRACE_MAX=0) give the reports and candidates
    of the reference pipeline fed the host-oriented, partitioned records."""
    from oracle.pyoracle import SeaConfig as OCfg
    cfg, _ = S.SCENARIOS[name]
    slices = GF.scenario_slices(name, oracle)
    recs = np.concatenate(slices)
    rng = np.random.default_rng(5)
    raw = recs.copy()
    flip = rng.random(len(raw)) < 0.25
    raw[flip, 1], raw[flip, 2] = recs[flip, 2], recs[flip, 1]
    off = rng.random(len(raw)) < 0.05  # neither side in 10/8: dropped
    raw[off, 1] = 0xC0A80001
    raw[off, 2] = 0xC0A80002
    trace = tmp_path / "raw.bin"
    _write_srlt(trace, raw)
    out = tmp_path / "run.txt"
    c = cfg
    env = dict(os.environ, SRLA_DEVICE_TRACE_MAX="0") if front == "host" else None
    subprocess.run([dropin_bin, "run", str(trace), str(out), str(c.rows), str(c.cols), str(c.rough_slots),
                    str(c.linear_slots), str(c.recorder_bits), str(c.window), str(c.theta), hex(c.seed)],
                   check=True, timeout=600, env=env)
    lines = open(out).read().split("\n")
    ori, st = oracle.orient(raw, 0x0A000000, 8)
    assert lines[-2] == "orient " + " ".join(str(int(x)) for x in st)
    bounds = oracle.slice_bounds(ori, 1)
    pipe = oracle.pipeline(OCfg(**c.as_dict()))
    want = []
    for s in range(len(bounds) - 1):
        rep = pipe.process_slice(s, ori[bounds[s]:bounds[s + 1]], True)
        if rep is None:
            continue
        bits = rep["estimate"].view(np.uint64)
        want.append([[int(h), int(w), int(b) if has else 0, int(has), int(sup)]
                     for h, w, b, has, sup in zip(rep["host"], rep["weight"], bits, rep["has_estimate"],
                                                  rep["is_super"])])
    got, i = [], 0
    while i < len(lines):
        if lines[i].startswith("report "):
            n = int(lines[i].split()[2])
            got.append([list(map(int, lines[i + 1 + j].split())) for j in range(n)])
            i += 1 + n
            continue
        i += 1
    assert got == want
    k = lines.index(next(l for l in lines if l.startswith("csip ")))
    n = int(lines[k].split()[1])
    assert [int(x) for x in lines[k + 1:k + 1 + n]] == pipe.candidates().tolist()


def _sha_file(p):
    import hashlib
    h = hashlib.sha256()
    with open(p, "rb") as f:
        while True:
            b = f.read(1 << 24)
            if not b:
                return h.hexdigest()
            h.update(b)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["pipeline_small", "wide_w2", "c1_shape", "contended", "c2_v20"])
def test_dropin_snapshot_bytes_equal_reference(gpu, ref, oracle, dropin_bin, tmp_path, name):
    """save_snapshot of the drop-in (rows streamed from HBM through pinned
    pieces) writes the same bytes as the reference's save_snapshot
    (snapshot.hpp:109-136) after the same slices through DetectPipeline."""
    from oracle.pyoracle import PlantSpec, SeaConfig
    if name == "c2_v20":  # C2's sketch (v = 2^20: 4 GiB of linear recorders) on a reduced C2-shape trace
        from paper_1803_10369_b200 import workloads as WL
        c = S.Cfg(**WL.sketch_cfg(1 << 20))
        spec = PlantSpec(**WL.trace_spec(300_000, slices=3))
        slices = [ref.generate_slice(spec, s) for s in range(3)]
    else:
        c, _ = S.SCENARIOS[name]
        slices = GF.scenario_slices(name, oracle)
    if c.cols & (c.cols - 1):
        pytest.skip("DetectPipeline needs a power-of-two column count")
    slices = [np.array(x, dtype=np.uint32).reshape(-1, 3).copy() for x in slices]
    for s, x in enumerate(slices):  # one second per slice: the replay's partitioner cuts the same slices
        x[:, 0] = 1700000000 + s
    trace = tmp_path / "t.bin"
    _write_srlt(trace, np.concatenate(slices))
    mine, theirs = tmp_path / "dropin.ssea", tmp_path / "ref.ssea"
    subprocess.run([dropin_bin, "replay", str(trace), str(tmp_path / "out.txt"), str(c.rows), str(c.cols),
                    str(c.rough_slots), str(c.linear_slots), str(c.recorder_bits), str(c.window), str(c.theta),
                    hex(c.seed)], check=True, timeout=900, env={**os.environ, "SRLA_TEST_SNAPSHOT": str(mine)})
    pipe = ref.pipeline(SeaConfig(**c.as_dict()), workers=1)
    for s, recs in enumerate(slices):
        pipe.process_slice(s, recs, True)
    pipe.save_snapshot(str(theirs))
    assert os.path.getsize(mine) == os.path.getsize(theirs)
    assert _sha_file(mine) == _sha_file(theirs)
    os.remove(mine)
    os.remove(theirs)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["pipeline_small", "c1_shape"])
def test_dropin_run_oracle_matches_reference_ring(gpu, ref, oracle, dropin_bin, tmp_path, name):
    """run_oracle (device exact store) over an SRLT trace: every complete
    window's (host, cardinality) list equals the reference SliceRingStore's."""
    from oracle.pyoracle import ExactRef
    c, _ = S.SCENARIOS[name]
    slices = [np.array(x, dtype=np.uint32).reshape(-1, 3).copy() for x in GF.scenario_slices(name, oracle)]
    for s, x in enumerate(slices):
        x[:, 0] = 1700000000 + s
    trace = tmp_path / "t.bin"
    _write_srlt(trace, np.concatenate(slices))
    out = tmp_path / "truth.txt"
    subprocess.run([dropin_bin, "oracle", str(trace), str(out), str(c.rows), str(c.cols), str(c.rough_slots),
                    str(c.linear_slots), str(c.recorder_bits), str(c.window), str(c.theta), hex(c.seed)],
                   check=True, timeout=600)
    got = [tuple(map(int, ln.split())) for ln in open(out) if ln.strip()]
    ring = ExactRef(ref, "ring", c.window)
    want = []
    for s, recs in enumerate(slices):
        ring.observe(recs)
        if s + 1 >= c.window:
            h, n = ring.cardinalities(s + 1 - c.window, c.window)
            want += [(s + 1 - c.window, int(a), int(b)) for a, b in zip(h, n)]
        ring.end_slice()
    assert got == want and len(want) > 0
