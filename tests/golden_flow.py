"""The scripted scan -> report -> slide flow (tests/test_pipeline.cpp:101-118)
run on any backend, summarised into a golden record. Shared by the fixture
generator, the CPU oracle tests and the GPU parity tests."""
from __future__ import annotations

import hashlib

import numpy as np

import scenarios as S

FULL_LIST_MAX = 256      # lists up to this length are stored verbatim
BIG_STATE = 1 << 24      # above this many linear words, digest state every 8th slice


def _lst(a):
    a = np.asarray(a, dtype=np.uint32)
    d = {"n": int(len(a)), "sha": hashlib.sha256(a.tobytes()).hexdigest()}
    if len(a) <= FULL_LIST_MAX:
        d["v"] = [int(x) for x in a]
    return d


def _report(hosts, weights, est, has, sup):
    rows = np.zeros((len(hosts), 4), np.uint64)
    rows[:, 0] = hosts
    rows[:, 1] = weights
    rows[:, 2] = np.asarray(est, np.float64).view(np.uint64)
    rows[:, 3] = np.asarray(has, np.uint64) | (np.asarray(sup, np.uint64) << 1)
    d = {"n": int(len(hosts)), "sha": hashlib.sha256(rows.tobytes()).hexdigest()}
    if len(hosts) <= FULL_LIST_MAX:
        d["v"] = [[int(r[0]), int(r[1]), format(int(r[2]), "016x"), int(r[3])] for r in rows]
    return d


def digest_slices(cfg: S.Cfg):
    words = cfg.cols * cfg.linear_slots * cfg.rows
    return (lambda s, last: True) if words <= BIG_STATE else (lambda s, last: s % 8 == 7 or last)


def kats(chk):
    """Known-answer values of the scalar helpers (hash.hpp, estimators.hpp, sea.hpp:270-279)."""
    out = {"hash_u32": [], "reduce": [], "sampling_exponent": [], "threshold": [], "linear_estimate": [],
           "ratio": format(np.float64(chk.super_test_ratio).view(np.uint64).item(), "016x")}
    seeds = [0, 1, 0xC0FFEE, 0x5EA00001, 0xFFFFFFFFFFFFFFFF, 0x1234567890ABCDEF]
    keys = [0, 1, 0x0A000001, 0xFFFFFFFF, 0x64400000, 0xB0000000, 2654435761]
    for sd in seeds:
        for idx in (0, 1, 2, 3, 8, 9, 71):
            for k in keys:
                out["hash_u32"].append([sd, idx, k, chk.hash_u32(sd, idx, k)])
                out["reduce"].append([sd, idx, k, 1000003, chk.hash_reduce(sd, idx, k, 1000003)])
    for th in (1, 7, 8, 9, 16, 1023, 1024, 1025, 65536, 0xFFFFFFFF):
        for g in (1, 3, 8, 32):
            out["sampling_exponent"].append([th, g, chk.f("sampling_exponent")(th, g)])
    for g in (1, 2, 3, 8, 11, 16, 64, 1000):
        out["threshold"].append([g, chk.f("super_weight_threshold")(chk.super_test_ratio, g)])
    for w, slots in ((0, 1024), (1, 1024), (100, 1024), (500, 1024), (1023, 1024), (1024, 1024), (5, 32)):
        e = chk.linear_estimate(w, slots)
        out["linear_estimate"].append([w, slots, None if e is None else format(np.float64(e).view(np.uint64).item(), "016x")])
    return out


def run_flow(backend, cfg: S.Cfg, slices):
    """backend: object with scan(recs)->pushes, candidates(), report()->(h,w,e,has,sup),
    end_of_slice(s) -> retained, state()."""
    want_state = digest_slices(cfg)
    out = []
    for s, recs in enumerate(slices):
        pushes = backend.scan(recs)
        csip = backend.candidates()
        rec = {"pushes": _lst(pushes), "csip": _lst(csip), "report": None}
        if s + 1 >= cfg.window:
            rec["report"] = _report(*backend.report())
        rec["retained"] = _lst(backend.slide())
        rec["state"] = S.state_digest(backend.state(), cfg.rows) if want_state(s, s == len(slices) - 1) else None
        out.append(rec)
    return out


class CheckerBackend:
    """A checker sketch (oracle or reference) plus a CandidateList in Python."""

    def __init__(self, chk, cfg: S.Cfg):
        from oracle.pyoracle import SeaConfig
        self.sk = chk.sketch(SeaConfig(**cfg.as_dict()))
        self.csip, self.seen = [], set()

    def scan(self, recs):
        pushes = self.sk.scan(recs)
        for h in pushes.tolist():
            if h not in self.seen:
                self.seen.add(h)
                self.csip.append(h)
        return pushes

    def candidates(self):
        return np.array(self.csip, np.uint32)

    def report(self):
        r = self.sk.report(self.candidates())
        return r["host"], r["weight"], r["estimate"], r["has_estimate"], r["is_super"]

    def slide(self):
        ret = self.sk.slide(self.candidates())
        self.csip, self.seen = ret.tolist(), set(ret.tolist())
        return ret

    def state(self):
        return self.sk.state()


def scenario_slices(name, chk=None, generate=None):
    cfg, (kind, src) = S.SCENARIOS[name]
    if kind == "spec":
        if generate is None:
            from oracle.pyoracle import PlantSpec
            generate = lambda sp: chk.generate(PlantSpec(**sp.__dict__))  # noqa: E731
    return S.slices_for(name, generate)


def run_flow_checker(chk, name):
    cfg, _ = S.SCENARIOS[name]
    slices = scenario_slices(name, chk)
    return {"name": name, "cfg": cfg.as_dict(), "records_sha256": S.records_digest(slices),
            "slices": run_flow(CheckerBackend(chk, cfg), cfg, slices)}


class EngineBackend:
    """The CUDA engine through the C ABI (engine-owned candidate list)."""

    def __init__(self, engine):
        self.e = engine

    def scan(self, recs):
        return self.e.scan_collect(recs)

    def candidates(self):
        return self.e.candidates()

    def report(self):
        r = self.e.report()
        return r["host"], r["union_weight"], r["estimate"], r["has_estimate"], r["is_super"]

    def slide(self):
        self.e.slide_engine()
        return self.e.candidates()

    def state(self):
        return self.e.state()


def compare(golden_slices, got_slices):
    """First mismatch as a readable string, or None."""
    for s, (g, o) in enumerate(zip(golden_slices, got_slices)):
        for key in ("pushes", "csip", "report", "retained", "state"):
            if g[key] != o[key] and not (key == "state" and (g[key] is None or o[key] is None)):
                gv, ov = g[key], o[key]
                if isinstance(gv, dict) and isinstance(ov, dict) and "v" in gv and "v" in ov:
                    gl, ol = gv["v"], ov["v"]
                    i = next((i for i, (a, b) in enumerate(zip(gl, ol)) if a != b), min(len(gl), len(ol)))
                    return f"slice {s} {key}: first difference at {i}: golden {gl[i:i+3]} got {ol[i:i+3]} (n {gv['n']} vs {ov['n']})"
                return f"slice {s} {key}: golden {str(gv)[:200]} got {str(ov)[:200]}"
    if len(golden_slices) != len(got_slices):
        return f"slice count {len(golden_slices)} vs {len(got_slices)}"
    return None


def block_sums_np(buf) -> np.ndarray:
    """numpy restatement of the state block digest (digest.cuh, ref_capi.cpp
    block_sums): per 1 MiB block the wrapping sum of avalanche64(w ^
    avalanche64(i + 1)) over the little-endian 8-byte words w_i of the row."""
    b = np.ascontiguousarray(buf).view(np.uint8).reshape(-1)
    nb = (len(b) + (1 << 20) - 1) >> 20
    pad = np.zeros(nb << 20, np.uint8)
    pad[: len(b)] = b
    w = pad.view("<u8")
    i = np.arange(1, len(w) + 1, dtype=np.uint64)

    def av(x):
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))

    with np.errstate(over="ignore"):
        h = av(w ^ av(i))
        # words past the row end contribute nothing (zero padding is only within the last word)
        h[(len(b) + 7) // 8:] = 0
        return h.reshape(nb, -1).sum(axis=1, dtype=np.uint64) if nb else np.zeros(0, np.uint64)
