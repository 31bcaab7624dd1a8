"""ctypes front end for the two CPU checkers. TEST INFRASTRUCTURE ONLY.

* ``Checker("orc")`` loads ``oracle/build/libsrla_oracle.so`` — the C restatement
  (``oracle/srla_oracle.c``).
* ``Checker("ref")`` loads ``oracle/_ref/libsspread_ref.so`` — the unmodified
  reference headers behind ``oracle/ref_capi.cpp``.

Both export the same ABI (``srla_oracle.h``). Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline / reference arm)
may import this module, as the checker; the engine never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "orc": os.path.join(HERE, "build", "libsrla_oracle.so"),
    "ref": os.path.join(HERE, "_ref", "libsspread_ref.so"),
}
INDICATOR, ROUGH, LINEAR = 0, 1, 2


class OrcConfig(C.Structure):
    _fields_ = [
        ("rows", C.c_uint32), ("cols", C.c_uint32), ("rough_slots", C.c_uint32),
        ("linear_slots", C.c_uint32), ("recorder_bits", C.c_uint32), ("window", C.c_uint32),
        ("theta", C.c_uint32), ("_pad", C.c_uint32), ("fill_ratio", C.c_double),
        ("seed", C.c_uint64),
    ]


class OrcPlant(C.Structure):
    _fields_ = [("host", C.c_uint32), ("cardinality", C.c_uint32),
                ("first_slice", C.c_uint32), ("last_slice", C.c_uint32)]


class OrcSpec(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64), ("start_ts", C.c_uint32), ("slice_seconds", C.c_uint32),
        ("slices", C.c_uint32), ("window", C.c_uint32), ("a_base", C.c_uint32),
        ("b_base", C.c_uint32), ("a_hosts", C.c_uint32), ("b_hosts", C.c_uint32),
        ("pairs_per_slice", C.c_uint32), ("n_plants", C.c_uint32), ("skew", C.c_double),
        ("plants", C.POINTER(OrcPlant)),
    ]


@dataclass
class SeaConfig:
    """sspread::SeaConfig (sea.hpp:33-52) defaults."""
    rows: int = 4
    cols: int = 65536
    rough_slots: int = 8
    linear_slots: int = 1024
    recorder_bits: int = 1
    window: int = 1
    theta: int = 1024
    fill_ratio: float | None = None  # None -> kSuperTestRatio
    seed: int = 0x00C0FFEE


@dataclass
class PlantSpec:
    """sspread::PlantSpec (generator.hpp:36-64) defaults."""
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
    plants: list = field(default_factory=list)  # (host, cardinality, first, last)


def build(quiet: bool = True) -> None:
    """Build both checkers (the reference one only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


_U32P = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class Checker:
    def __init__(self, prefix: str = "orc"):
        path = LIBS[prefix]
        if not os.path.exists(path):
            raise FileNotFoundError(f"checker library {path} not built (run `make -f oracle/Makefile`)")
        self.prefix = prefix
        self.lib = C.CDLL(path)
        self._sig()
        self.super_test_ratio = self.f("super_test_ratio")()

    def f(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    def _sig(self):
        vp, u32, u64, dbl, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_double, C.c_int
        sigs = {
            "avalanche64": (u64, [u64]),
            "hash_u32": (u32, [u64, u32, u32]),
            "hash_reduce": (u32, [u64, u32, u32, u32]),
            "sampling_exponent": (u32, [u64, u64]),
            "super_weight_threshold": (u32, [dbl, u32]),
            "super_test_ratio": (dbl, []),
            "linear_estimate": (i32, [u32, u32, C.POINTER(dbl)]),
            "create": (vp, [C.POINTER(OrcConfig), C.c_char_p, C.c_size_t]),
            "destroy": (None, [vp]),
            "tau": (u32, [vp]), "threshold": (u32, [vp]), "word_bytes": (u32, [vp]),
            "column_of": (u32, [vp, u32, u32]),
            "row_len": (u64, [vp, i32]),
            "scan": (None, [vp, vp, u64, vp, C.POINTER(u64)]),
            "union_rough_weight": (u32, [vp, u32]),
            "union_linear_weight": (u32, [vp, u32]),
            "union_view": (C.c_uint16, [vp, u32, vp, vp]),
            "row_active": (u64, [vp, u32]),
            "row_fill_fraction": (dbl, [vp, u32]),
            "union_fill_product": (dbl, [vp]),
            "corrected_estimate_from": (i32, [vp, u32, dbl, C.POINTER(dbl)]),
            "report": (None, [vp, vp, u64, vp, vp, vp, vp, vp]),
            "slide": (u64, [vp, vp, u64, vp]),
            "export_row": (None, [vp, u32, i32, vp]),
            "import_row": (None, [vp, u32, i32, vp]),
            "pipeline_create": (vp, [C.POINTER(OrcConfig), u32, C.c_char_p, C.c_size_t]),
            "pipeline_destroy": (None, [vp]),
            "pipeline_sketch": (vp, [vp]),
            "pipeline_process_slice": (None, [vp, u64, vp, u64, i32, C.POINTER(i32), C.POINTER(u64),
                                              vp, vp, vp, vp, vp]),
            "pipeline_ncand": (u64, [vp]),
            "pipeline_candidates": (None, [vp, vp]),
            "pipeline_scan_ms": (dbl, [vp]),
            "pipeline_estimate_ms": (dbl, [vp]),
            "generate": (u64, [C.POINTER(OrcSpec), vp, C.c_char_p, C.c_size_t]),
            "orient": (u64, [vp, u64, u32, u32, vp, vp]),
            "slice_bounds": (u64, [vp, u64, u32, vp]),
            "parse_srlt": (u64, [vp, u64, vp, C.POINTER(i32), C.POINTER(u64)]),
        }
        if self.prefix == "ref":  # reference-only: parallel slice generator, record-order flow
            sigs.update({
                "pipeline_save_snapshot": (i32, [vp, C.c_char_p, C.c_char_p, C.c_size_t]),
                "exact_create": (vp, [i32, u32, u32, C.c_char_p, C.c_size_t]),
                "exact_destroy": (None, [vp]),
                "exact_observe": (None, [vp, vp, u64]),
                "exact_end_slice": (None, [vp]),
                "exact_pair_count": (u64, [vp]),
                "exact_cardinalities": (u64, [vp, u64, u32, vp, vp, C.c_char_p, C.c_size_t]),
                "generate_slice": (u64, [C.POINTER(OrcSpec), u64, u32, vp, C.c_char_p, C.c_size_t]),
                "flow_create": (vp, [C.POINTER(OrcConfig), u32, C.c_char_p, C.c_size_t]),
                "flow_destroy": (None, [vp]),
                "flow_scan": (u64, [vp, vp, u64]),
                "flow_pushes": (None, [vp, vp]),
                "flow_ncand": (u64, [vp]),
                "flow_candidates": (None, [vp, vp]),
                "flow_report": (u64, [vp, u64, vp, vp, vp, vp, vp]),
                "flow_slide": (u64, [vp]),
                "flow_row_bytes": (u64, [vp, i32]),
                "flow_state_blocks": (None, [vp, u32, i32, vp]),
                "block_sums": (None, [vp, u64, u32, vp]),
            })
        for name, (res, args) in sigs.items():
            fn = self.f(name)
            fn.restype = res
            fn.argtypes = args

    # ---- library helpers
    def hash_u32(self, seed, index, key):
        return self.f("hash_u32")(seed, index, key)

    def hash_reduce(self, seed, index, key, rng):
        return self.f("hash_reduce")(seed, index, key, rng)

    def linear_estimate(self, w, slots):
        out = C.c_double()
        return out.value if self.f("linear_estimate")(w, slots, C.byref(out)) else None

    # ---- ingest front end (trace.hpp)
    def orient(self, recs, prefix_addr, prefix_bits):
        """orient_record over a batch -> (records kept/flipped in order, [kept, flipped, both, neither])."""
        recs = np.ascontiguousarray(recs, dtype=np.uint32).reshape(-1, 3)
        out = np.empty((max(1, len(recs)), 3), np.uint32)
        st = np.zeros(4, np.uint64)
        m = self.f("orient")(_ptr(recs), len(recs), prefix_addr, prefix_bits, _ptr(out), _ptr(st))
        return out[:m].copy(), st

    def slice_bounds(self, recs, slice_seconds):
        """SlicePartitioner -> offsets (nslices + 1) of an ordered batch."""
        recs = np.ascontiguousarray(recs, dtype=np.uint32).reshape(-1, 3)
        ns = self.f("slice_bounds")(_ptr(recs), len(recs), slice_seconds, None)
        off = np.zeros(ns + 1, np.uint64)
        if ns:
            self.f("slice_bounds")(_ptr(recs), len(recs), slice_seconds, _ptr(off))
        return off

    def parse_srlt(self, data: bytes):
        """SRLT v1 file bytes -> (records, err, err_index)."""
        buf = np.frombuffer(data, np.uint8)
        err, idx = C.c_int(), C.c_uint64()
        n = self.f("parse_srlt")(_ptr(buf), len(buf), None, C.byref(err), C.byref(idx))
        out = np.empty((max(1, n), 3), np.uint32)
        n = self.f("parse_srlt")(_ptr(buf), len(buf), _ptr(out), C.byref(err), C.byref(idx))
        return out[:n].copy(), err.value, idx.value

    def config(self, cfg: SeaConfig) -> OrcConfig:
        fr = self.super_test_ratio if cfg.fill_ratio is None else cfg.fill_ratio
        return OrcConfig(cfg.rows, cfg.cols, cfg.rough_slots, cfg.linear_slots, cfg.recorder_bits,
                         cfg.window, cfg.theta, 0, fr, cfg.seed & 0xFFFFFFFFFFFFFFFF)

    def sketch(self, cfg: SeaConfig) -> "Sketch":
        err = C.create_string_buffer(256)
        c = self.config(cfg)
        h = self.f("create")(C.byref(c), err, 256)
        if not h:
            raise ValueError(err.value.decode())
        return Sketch(self, h, cfg, owned=True)

    def pipeline(self, cfg: SeaConfig, workers: int = 1) -> "Pipeline":
        err = C.create_string_buffer(256)
        c = self.config(cfg)
        h = self.f("pipeline_create")(C.byref(c), workers, err, 256)
        if not h:
            raise ValueError(err.value.decode())
        return Pipeline(self, h, cfg)

    @staticmethod
    def _spec(spec: PlantSpec):
        plants = (OrcPlant * max(1, len(spec.plants)))()
        for i, p in enumerate(spec.plants):
            plants[i] = OrcPlant(*p)
        s = OrcSpec(spec.seed, spec.start_ts, spec.slice_seconds, spec.slices, spec.window,
                    spec.a_base, spec.b_base, spec.a_hosts, spec.b_hosts, spec.pairs_per_slice,
                    len(spec.plants), spec.skew, plants)
        s._keep = plants
        return s

    def generate_slice(self, spec: PlantSpec, slice_id: int, threads: int = 0, out=None) -> np.ndarray:
        """Slice `slice_id` of generate_trace built in parallel from the reference's
        own generator pieces (ref_generate_slice; slice_seconds == 1)."""
        s = self._spec(spec)
        err = C.create_string_buffer(256)
        n = self.f("generate_slice")(C.byref(s), slice_id, 0, None, err, 256)
        if n == 0xFFFFFFFFFFFFFFFF:
            raise ValueError(err.value.decode())
        if out is None or len(out) < n:
            out = np.empty((n, 3), np.uint32)
        self.f("generate_slice")(C.byref(s), slice_id, threads or (os.cpu_count() or 1), _ptr(out), err, 256)
        return out[:n]

    def block_sums(self, buf, threads: int = 0) -> np.ndarray:
        """Per-MiB block sums of a byte buffer (the state digest of srla_state_blocks)."""
        b = np.ascontiguousarray(buf).view(np.uint8).reshape(-1)
        out = np.empty(max(1, (len(b) + (1 << 20) - 1) >> 20), np.uint64)
        self.f("block_sums")(_ptr(b), len(b), threads or (os.cpu_count() or 1), _ptr(out))
        return out[: (len(b) + (1 << 20) - 1) >> 20]

    def flow(self, cfg: SeaConfig, threads: int = 0) -> "Flow":
        err = C.create_string_buffer(256)
        c = self.config(cfg)
        h = self.f("flow_create")(C.byref(c), threads or (os.cpu_count() or 1), err, 256)
        if not h:
            raise ValueError(err.value.decode())
        return Flow(self, h, cfg)

    def generate(self, spec: PlantSpec) -> np.ndarray:
        plants = (OrcPlant * max(1, len(spec.plants)))()
        for i, p in enumerate(spec.plants):
            plants[i] = OrcPlant(*p)
        s = OrcSpec(spec.seed, spec.start_ts, spec.slice_seconds, spec.slices, spec.window,
                    spec.a_base, spec.b_base, spec.a_hosts, spec.b_hosts, spec.pairs_per_slice,
                    len(spec.plants), spec.skew, plants)
        err = C.create_string_buffer(256)
        if self.prefix == "orc":
            n = self.f("generate")(C.byref(s), None, err, 256)
            if n == 0xFFFFFFFFFFFFFFFF:
                raise ValueError(err.value.decode())
            out = np.empty((n, 3), np.uint32)
            self.f("generate")(C.byref(s), _ptr(out), err, 256)
            return out
        # the reference generates once; size the buffer from the restatement's count
        n = Checker("orc").f("generate")(C.byref(s), None, err, 256)
        if n == 0xFFFFFFFFFFFFFFFF:
            raise ValueError(err.value.decode())
        out = np.empty((n, 3), np.uint32)
        m = self.f("generate")(C.byref(s), _ptr(out), err, 256)
        assert m == n, (m, n)
        return out


class Sketch:
    """EstimatorArray<W> (sea.hpp:113-359) through the checker ABI."""

    def __init__(self, chk: Checker, h, cfg: SeaConfig, owned: bool):
        self.chk, self.h, self.cfg, self.owned = chk, h, cfg, owned
        self.tau = chk.f("tau")(h)
        self.threshold = chk.f("threshold")(h)
        self.word_bytes = chk.f("word_bytes")(h)
        self.wdtype = {1: np.uint8, 2: np.uint16, 4: np.uint32}[self.word_bytes]

    def __del__(self):
        if getattr(self, "owned", False) and self.h:
            self.chk.f("destroy")(self.h)
            self.h = None

    def column_of(self, row, aip):
        return self.chk.f("column_of")(self.h, row, aip)

    def scan(self, recs) -> np.ndarray:
        recs = np.ascontiguousarray(recs, dtype=np.uint32).reshape(-1, 3)
        sink = np.empty(max(1, len(recs)), np.uint32)
        ns = C.c_uint64()
        self.chk.f("scan")(self.h, _ptr(recs), len(recs), _ptr(sink), C.byref(ns))
        return sink[: ns.value].copy()

    def scan_pairs(self, pairs) -> np.ndarray:
        pairs = np.asarray(pairs, dtype=np.uint32).reshape(-1, 2)
        recs = np.zeros((len(pairs), 3), np.uint32)
        recs[:, 1:] = pairs
        return self.scan(recs)

    def union_rough_weight(self, aip):
        return self.chk.f("union_rough_weight")(self.h, aip)

    def union_linear_weight(self, aip):
        return self.chk.f("union_linear_weight")(self.h, aip)

    def union_view(self, aip, include_linear=True):
        rough = np.empty(self.cfg.rough_slots, np.uint32)
        lin = np.empty(self.cfg.linear_slots, np.uint32) if include_linear else None
        ind = self.chk.f("union_view")(self.h, aip, _ptr(rough), _ptr(lin))
        return ind, rough, lin

    def row_active(self, row):
        return self.chk.f("row_active")(self.h, row)

    def row_fill_fraction(self, row):
        return self.chk.f("row_fill_fraction")(self.h, row)

    def union_fill_product(self):
        return self.chk.f("union_fill_product")(self.h)

    def corrected_estimate_from(self, w, fp):
        out = C.c_double()
        return out.value if self.chk.f("corrected_estimate_from")(self.h, w, fp, C.byref(out)) else None

    def report(self, csip) -> dict:
        csip = np.ascontiguousarray(csip, dtype=np.uint32)
        n = len(csip)
        out = _report_buffers(n)
        self.chk.f("report")(self.h, _ptr(csip), n, *(_ptr(out[k]) for k in _REPORT_KEYS))
        return {k: v[:n] for k, v in out.items()}

    def slide(self, csip) -> np.ndarray:
        csip = np.ascontiguousarray(csip, dtype=np.uint32)
        ret = np.empty(max(1, len(csip)), np.uint32)
        m = self.chk.f("slide")(self.h, _ptr(csip), len(csip), _ptr(ret))
        return ret[:m].copy()

    def row_len(self, kind):
        return self.chk.f("row_len")(self.h, kind)

    def export_row(self, row, kind) -> np.ndarray:
        dt = np.uint16 if kind == INDICATOR else self.wdtype
        out = np.empty(self.row_len(kind), dt)
        self.chk.f("export_row")(self.h, row, kind, _ptr(out))
        return out

    def import_row(self, row, kind, data):
        dt = np.uint16 if kind == INDICATOR else self.wdtype
        data = np.ascontiguousarray(data, dtype=dt)
        assert len(data) == self.row_len(kind)
        self.chk.f("import_row")(self.h, row, kind, _ptr(data))

    def state(self) -> dict:
        """All rows, for bit-exact comparison."""
        return {(k, i): self.export_row(i, k) for i in range(self.cfg.rows)
                for k in (INDICATOR, ROUGH, LINEAR)}


_REPORT_KEYS = ("host", "weight", "estimate", "has_estimate", "is_super")


def _report_buffers(n):
    n1 = max(1, n)
    return {"host": np.empty(n1, np.uint32), "weight": np.empty(n1, np.uint32),
            "estimate": np.empty(n1, np.float64), "has_estimate": np.empty(n1, np.uint8),
            "is_super": np.empty(n1, np.uint8)}


class Pipeline:
    """DetectPipeline<W> (pipeline.hpp:80-168) fed slice by slice."""

    def __init__(self, chk: Checker, h, cfg: SeaConfig):
        self.chk, self.h, self.cfg = chk, h, cfg
        self.sketch = Sketch(chk, chk.f("pipeline_sketch")(h), cfg, owned=False)

    def __del__(self):
        if getattr(self, "h", None):
            self.chk.f("pipeline_destroy")(self.h)
            self.h = None

    def candidates(self) -> np.ndarray:
        n = self.chk.f("pipeline_ncand")(self.h)
        out = np.empty(max(1, n), np.uint32)
        self.chk.f("pipeline_candidates")(self.h, _ptr(out))
        return out[:n].copy()

    def process_slice(self, slice_id, recs, want_report=True):
        recs = np.ascontiguousarray(recs, dtype=np.uint32).reshape(-1, 3)
        cap = self.chk.f("pipeline_ncand")(self.h) + len(recs)
        out = _report_buffers(cap)
        rep, ne = C.c_int(), C.c_uint64()
        self.chk.f("pipeline_process_slice")(self.h, slice_id, _ptr(recs), len(recs), int(want_report),
                                             C.byref(rep), C.byref(ne),
                                             *(_ptr(out[k]) for k in _REPORT_KEYS))
        if not rep.value:
            return None
        return {k: v[: ne.value].copy() for k, v in out.items()}

    def save_snapshot(self, path: str):
        """The reference's save_snapshot(sketch, candidates, path) (reference checker only)."""
        err = C.create_string_buffer(256)
        if self.chk.f("pipeline_save_snapshot")(self.h, path.encode(), err, 256):
            raise OSError(err.value.decode())

    @property
    def scan_ms(self):
        return self.chk.f("pipeline_scan_ms")(self.h)

    @property
    def estimate_ms(self):
        return self.chk.f("pipeline_estimate_ms")(self.h)


class Flow:
    """The reference sketch + CandidateList driven like DetectPipeline::process_slice
    with ONE scan worker (record order, pipeline.hpp:110-139), bulk passes chunked
    over threads (sea.hpp:23-26). Full-size parity source (ref_flow_*)."""

    def __init__(self, chk: Checker, h, cfg: SeaConfig):
        self.chk, self.h, self.cfg = chk, h, cfg

    def __del__(self):
        if getattr(self, "h", None):
            self.chk.f("flow_destroy")(self.h)
            self.h = None

    def scan(self, recs) -> np.ndarray:
        recs = np.ascontiguousarray(recs, dtype=np.uint32).reshape(-1, 3)
        n = self.chk.f("flow_scan")(self.h, _ptr(recs), len(recs))
        out = np.empty(max(1, n), np.uint32)
        self.chk.f("flow_pushes")(self.h, _ptr(out))
        return out[:n]

    def candidates(self) -> np.ndarray:
        n = self.chk.f("flow_ncand")(self.h)
        out = np.empty(max(1, n), np.uint32)
        self.chk.f("flow_candidates")(self.h, _ptr(out))
        return out[:n]

    def report(self, window_start=0) -> dict:
        out = _report_buffers(self.chk.f("flow_ncand")(self.h))
        n = self.chk.f("flow_report")(self.h, window_start, *(_ptr(out[k]) for k in _REPORT_KEYS))
        return {k: v[:n] for k, v in out.items()}

    def slide(self) -> int:
        return self.chk.f("flow_slide")(self.h)

    def state_blocks(self, row, kind) -> np.ndarray:
        nb = (self.chk.f("flow_row_bytes")(self.h, kind) + (1 << 20) - 1) >> 20
        out = np.empty(max(1, nb), np.uint64)
        self.chk.f("flow_state_blocks")(self.h, row, kind, _ptr(out))
        return out[:nb]


class ExactRef:
    """The reference's exact stores (oracle.hpp): SliceRingStore (engine "ring")
    or PairRecorderStore (engine "pairs"). Reference checker only."""

    def __init__(self, chk: Checker, engine: str, max_window: int, recorder_bits: int = 8):
        err = C.create_string_buffer(256)
        self.chk = chk
        self.h = chk.f("exact_create")(0 if engine == "ring" else 1, recorder_bits, max_window, err, 256)
        if not self.h:
            raise ValueError(err.value.decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.chk.f("exact_destroy")(self.h)
            self.h = None

    def observe(self, recs):
        recs = np.ascontiguousarray(recs, dtype=np.uint32).reshape(-1, 3)
        self.chk.f("exact_observe")(self.h, _ptr(recs), len(recs))

    def end_slice(self):
        self.chk.f("exact_end_slice")(self.h)

    def pair_count(self):
        return self.chk.f("exact_pair_count")(self.h)

    def cardinalities(self, t, k):
        err = C.create_string_buffer(256)
        n = self.chk.f("exact_cardinalities")(self.h, t, k, None, None, err, 256)
        if n == 0xFFFFFFFFFFFFFFFF:
            raise IndexError(err.value.decode())
        hosts, counts = np.empty(max(1, n), np.uint32), np.empty(max(1, n), np.uint64)
        self.chk.f("exact_cardinalities")(self.h, t, k, _ptr(hosts), _ptr(counts), err, 256)
        return hosts[:n], counts[:n]
