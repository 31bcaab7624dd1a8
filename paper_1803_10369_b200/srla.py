"""Python host binding of the B200 SRLA engine (ctypes over include/srla.h).

Mirrors the reference's hot-path API (``sspread::EstimatorArray`` /
``DetectPipeline``, /root/reference/proj/include/sspread/{sea,pipeline}.hpp)
with the same names, argument meaning and error behaviour, so parity tests read
like the reference's own tests. The C++ drop-in (include/sspread/*.hpp) binds
the same C ABI.

There is no CPU fallback: constructing an engine without the built
``lib/libsrla_b200.so`` or without a CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libsrla_b200.so")

INDICATOR, ROUGH, LINEAR = 0, 1, 2
OK, E_INVALID, E_RANGE, E_CAPACITY, E_CUDA, E_INTERNAL, E_INPUT = range(7)

# estimators.hpp:19 — evaluated by the library on first load (host glibc)
KSUPER_TEST_RATIO = 0.99 * (1.0 - math.exp(-1.0 / 3.0))


class SrlaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class InputError(SrlaError):
    """sspread::InputError (trace.hpp / snapshot.hpp): malformed trace input."""


class CConfig(C.Structure):
    _fields_ = [
        ("rows", C.c_uint32), ("cols", C.c_uint32), ("rough_slots", C.c_uint32),
        ("linear_slots", C.c_uint32), ("recorder_bits", C.c_uint32), ("window", C.c_uint32),
        ("theta", C.c_uint32), ("flags", C.c_uint32), ("fill_ratio", C.c_double),
        ("seed", C.c_uint64),
    ]


ENTRY_DTYPE = np.dtype([("host", "<u4"), ("union_weight", "<u4"), ("estimate", "<f8"),
                        ("has_estimate", "u1"), ("is_super", "u1"), ("reserved", "u1", (6,))])
assert ENTRY_DTYPE.itemsize == 24


class CStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "packets", "sampled_events", "crossings", "first_crossings", "flagged", "pushed",
        "kernel_launches", "library_launches", "chunks", "slides", "overlapped_chunks")]


class CTiming(C.Structure):
    _fields_ = [("scan_kernel_ms", C.c_double), ("scan_kernel_launches", C.c_uint64),
                ("scan_kernel_records", C.c_uint64), ("end_slice_device_ms", C.c_double),
                ("end_slice_wall_ms", C.c_double), ("last_end_slice_device_ms", C.c_double),
                ("last_end_slice_wall_ms", C.c_double), ("end_slices", C.c_uint64),
                ("order_wall_ms", C.c_double), ("report_wall_ms", C.c_double), ("slide_wall_ms", C.c_double),
                ("split_kernel_ms", C.c_double), ("split_kernel_launches", C.c_uint64),
                ("split_entries", C.c_uint64), ("apply_kernel_ms", C.c_double),
                ("apply_kernel_launches", C.c_uint64), ("apply_entries", C.c_uint64),
                ("apply_stream_bytes", C.c_uint64), ("gather_kernel_ms", C.c_double),
                ("gather_kernel_launches", C.c_uint64), ("gather_bytes", C.c_uint64),
                ("sync_wait_ms", C.c_double), ("syncs", C.c_uint64), ("alloc_ms", C.c_double),
                ("allocs", C.c_uint64), ("serial_kernel_ms", C.c_double),
                ("serial_kernel_launches", C.c_uint64), ("flagged_hosts", C.c_uint64)]


class CPlant(C.Structure):
    _fields_ = [("host", C.c_uint32), ("cardinality", C.c_uint32),
                ("first_slice", C.c_uint32), ("last_slice", C.c_uint32)]


class CSpec(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64), ("start_ts", C.c_uint32), ("slice_seconds", C.c_uint32),
        ("slices", C.c_uint32), ("window", C.c_uint32), ("a_base", C.c_uint32),
        ("b_base", C.c_uint32), ("a_hosts", C.c_uint32), ("b_hosts", C.c_uint32),
        ("pairs_per_slice", C.c_uint32), ("n_plants", C.c_uint32), ("skew", C.c_double),
        ("plants", C.POINTER(CPlant)),
    ]


class COrientStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("kept", "flipped", "dropped_both", "dropped_neither")]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libsrla_b200.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"SRLA CUDA library not built: {path} (run python -m paper_1803_10369_b200.build)")
    lib = C.CDLL(path)
    vp, u32, u64, i32, dbl = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
    sigs = {
        "srla_last_error": (C.c_char_p, []),
        "srla_version": (C.c_char_p, []),
        "srla_create": (i32, [C.POINTER(CConfig), i32, C.POINTER(vp)]),
        "srla_destroy": (i32, [vp]),
        "srla_params": (i32, [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32)]),
        "srla_column_of": (i32, [vp, u32, u32, C.POINTER(u32)]),
        "srla_scan_batch": (i32, [vp, vp, u64, i32, vp, u64, C.POINTER(u64)]),
        "srla_candidates": (i32, [vp, vp, u64, C.POINTER(u64)]),
        "srla_set_candidates": (i32, [vp, vp, u64]),
        "srla_report": (i32, [vp, vp, u64, C.POINTER(u64), C.POINTER(dbl)]),
        "srla_slide": (i32, [vp, C.POINTER(u64)]),
        "srla_end_slice": (i32, [vp, u64, i32, vp, u64, C.POINTER(u64), C.POINTER(u64)]),
        "srla_end_slice_async": (i32, [vp, u64, i32, vp, u64]),
        "srla_end_slice_compact": (i32, [vp, u64, i32, vp, vp, u64, C.POINTER(u64), vp, vp, C.POINTER(u64)]),
        "srla_end_slice_wait": (i32, [vp, C.POINTER(u64), C.POINTER(u64)]),
        "srla_union_weights": (i32, [vp, vp, u64, vp, vp]),
        "srla_union_view": (i32, [vp, u32, vp, vp, vp]),
        "srla_row_active": (i32, [vp, vp]),
        "srla_estimate_from": (i32, [vp, u32, dbl, C.POINTER(dbl), C.POINTER(i32)]),
        "srla_row_bytes": (i32, [vp, i32, C.POINTER(u64)]),
        "srla_export_row": (i32, [vp, u32, i32, vp, u64]),
        "srla_import_row": (i32, [vp, u32, i32, vp, u64]),
        "srla_stats_get": (i32, [vp, C.POINTER(CStats)]),
        "srla_synchronize": (i32, [vp]),
        "srla_timing_get": (i32, [vp, C.POINTER(CTiming)]),
        "srla_timing_reset": (i32, [vp]),
        "srla_partition_records": (i32, [vp, u64, u64, u32, u32, vp, C.POINTER(u64), vp]),
        "srla_owner_of": (u32, [u64, u32, u32]),
        "srla_stream": (i32, [vp, C.POINTER(vp)]),
        "srla_generator_create": (i32, [C.POINTER(CSpec), i32, C.POINTER(vp)]),
        "srla_generator_destroy": (i32, [vp]),
        "srla_generate_slice": (i32, [vp, u64, vp, u64, C.POINTER(u64), vp]),
        "srla_parse_srlt": (i32, [vp, u64, vp, C.POINTER(u64), vp]),
        "srla_orient_records": (i32, [vp, u64, u32, u32, vp, C.POINTER(u64), C.POINTER(COrientStats), vp]),
        "srla_slice_bounds": (i32, [vp, u64, u32, vp, u64, C.POINTER(u64), vp]),
        "srla_exact_create": (i32, [u32, i32, C.POINTER(vp)]),
        "srla_exact_destroy": (i32, [vp]),
        "srla_exact_observe": (i32, [vp, vp, u64, i32]),
        "srla_exact_end_slice": (i32, [vp]),
        "srla_exact_current_slice": (i32, [vp, C.POINTER(u64)]),
        "srla_exact_pair_count": (i32, [vp, C.POINTER(u64)]),
        "srla_exact_cardinalities": (i32, [vp, u64, u32, vp, vp, u64, C.POINTER(u64)]),
        "srla_export_range": (i32, [vp, u32, i32, u64, vp, u64]),
        "srla_import_range": (i32, [vp, u32, i32, u64, vp, u64]),
        "srla_scan_device": (i32, [vp, vp, u64, vp, vp, u64, C.POINTER(u64)]),
        "srla_state_blocks": (i32, [vp, u32, i32, vp, u64, C.POINTER(u64)]),
        "srla_block_sums": (i32, [vp, u64, vp, u64, vp]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    _lib = lib
    return lib


EXPORTED_SYMBOLS = (
    "srla_last_error", "srla_version", "srla_create", "srla_destroy", "srla_params", "srla_column_of",
    "srla_scan_batch", "srla_candidates", "srla_set_candidates", "srla_report", "srla_slide",
    "srla_end_slice", "srla_union_weights", "srla_union_view", "srla_row_active", "srla_estimate_from",
    "srla_row_bytes", "srla_export_row", "srla_import_row", "srla_stats_get", "srla_synchronize",
    "srla_stream", "srla_generator_create", "srla_generator_destroy", "srla_generate_slice",
    "srla_timing_get", "srla_timing_reset", "srla_partition_records", "srla_owner_of",
    "srla_end_slice_async", "srla_end_slice_wait", "srla_end_slice_compact",
    "srla_parse_srlt", "srla_orient_records", "srla_slice_bounds", "srla_device_alloc", "srla_device_free",
    "srla_copy_to_device", "srla_state_blocks", "srla_block_sums", "srla_scan_device",
    "srla_nccl_unique_id", "srla_transport_nccl", "srla_transport_nccl_destroy", "srla_shard_create",
    "srla_shard_destroy", "srla_shard_engine", "srla_shard_last_report", "srla_shard_process_slice",
    "srla_export_range", "srla_import_range", "srla_host_alloc", "srla_host_free", "srla_copy_to_host",
    "srla_exact_create", "srla_exact_destroy", "srla_exact_observe", "srla_exact_end_slice",
    "srla_exact_current_slice", "srla_exact_pair_count", "srla_exact_cardinalities",
)


def _check(rc):
    if rc != OK:
        msg = _lib.srla_last_error().decode()
        if rc == E_INVALID:
            raise ValueError(msg)  # std::invalid_argument
        if rc == E_RANGE:
            raise IndexError(msg)  # std::out_of_range
        if rc == E_INPUT:
            raise InputError(rc, msg)
        raise SrlaError(rc, msg)


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


@dataclass
class SeaConfig:
    """sspread::SeaConfig (sea.hpp:33-52) with the reference defaults."""
    rows: int = 4
    cols: int = 65536
    rough_slots: int = 8
    linear_slots: int = 1024
    recorder_bits: int = 1
    window: int = 1
    theta: int = 1024
    fill_ratio: float = KSUPER_TEST_RATIO
    seed: int = 0x00C0FFEE

    def to_c(self) -> CConfig:
        return CConfig(self.rows, self.cols, self.rough_slots, self.linear_slots, self.recorder_bits,
                       self.window, self.theta, 0, self.fill_ratio, self.seed & 0xFFFFFFFFFFFFFFFF)


def _as_records(recs) -> np.ndarray:
    a = np.ascontiguousarray(recs, dtype=np.uint32)
    if a.ndim == 1:
        a = a.reshape(-1, 3)
    if a.ndim != 2 or a.shape[1] != 3:
        raise ValueError("records must be (n, 3) uint32 triples (ts, src, dst)")
    return a


class EstimatorArray:
    """sspread::EstimatorArray<W> on one B200 (state resident in HBM).

    Record batches may be numpy (host) arrays or CUDA torch tensors (device,
    shape (n, 3), dtype int32/uint32) on the engine's device.
    """

    def __init__(self, cfg: SeaConfig, device: int = 0):
        lib = load_library()
        self.cfg = cfg
        self.device = device
        h = C.c_void_p()
        c = cfg.to_c()
        _check(lib.srla_create(C.byref(c), device, C.byref(h)))
        self._h = h
        tau, thr, wb = C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(lib.srla_params(h, C.byref(tau), C.byref(thr), C.byref(wb)))
        self.tau, self.threshold, self.word_bytes = tau.value, thr.value, wb.value
        self.wdtype = {1: np.uint8, 2: np.uint16, 4: np.uint32}[self.word_bytes]

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.srla_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    # -- params
    def weight_threshold(self) -> int:
        return self.threshold

    def column_of(self, row: int, aip: int) -> int:
        out = C.c_uint32()
        _check(_lib.srla_column_of(self._h, row, aip, C.byref(out)))
        return out.value

    # -- scan
    def _device_records(self, t):
        """Validate a CUDA record tensor: (n, 3) int32/uint32, contiguous, on the engine's GPU."""
        import torch
        if t.dtype not in (torch.int32, getattr(torch, "uint32", torch.int32)):
            raise ValueError(f"device records must be int32/uint32, got {t.dtype}")
        if t.dim() != 2 or t.shape[1] != 3:
            raise ValueError(f"device records must have shape (n, 3), got {tuple(t.shape)}")
        if not t.is_contiguous():
            raise ValueError("device records must be contiguous")
        if t.device.index != self.device:
            raise ValueError(f"records on cuda:{t.device.index}, engine on cuda:{self.device}")
        return t.data_ptr(), t.shape[0], torch.cuda.current_stream(t.device).cuda_stream

    def _scan(self, recs, out):
        npushed = C.c_uint64()
        cap = len(out) if out is not None else 0
        if _is_torch_cuda(recs):
            ptr, n, stream = self._device_records(recs)
            _check(_lib.srla_scan_device(self._h, C.c_void_p(ptr), n, C.c_void_p(stream), _ptr(out), cap,
                                         C.byref(npushed) if out is not None else None))
        else:
            recs = _as_records(recs)
            _check(_lib.srla_scan_batch(self._h, C.c_void_p(recs.ctypes.data), recs.shape[0], 0, _ptr(out), cap,
                                        C.byref(npushed) if out is not None else None))
        return npushed.value

    def scan(self, recs) -> None:
        """scan_ip_pair over every record in order (pushes go to the engine's candidate list).
        CUDA tensors are read after the work queued on torch's current stream."""
        self._scan(recs, None)

    def scan_collect(self, recs) -> np.ndarray:
        """Scan and return pushes (bounded by the number of records)."""
        out = np.empty(max(1, recs.shape[0] if _is_torch_cuda(recs) else len(_as_records(recs))), np.uint32)
        n = self._scan(recs, out)
        return out[:n].copy()

    def scan_ip_pair(self, aip: int, bip: int) -> np.ndarray:
        return self.scan_collect(np.array([[0, aip, bip]], np.uint32))

    def scan_pairs(self, pairs) -> np.ndarray:
        p = np.asarray(pairs, dtype=np.uint32).reshape(-1, 2)
        recs = np.zeros((len(p), 3), np.uint32)
        recs[:, 1:] = p
        return self.scan_collect(recs)

    # -- candidate list owned by the engine
    def candidates(self) -> np.ndarray:
        n = C.c_uint64()
        rc = _lib.srla_candidates(self._h, None, 0, C.byref(n))
        if rc not in (OK, E_CAPACITY):
            _check(rc)
        out = np.empty(max(1, n.value), np.uint32)
        _check(_lib.srla_candidates(self._h, _ptr(out), len(out), C.byref(n)))
        return out[: n.value].copy()

    def set_candidates(self, hosts):
        h = np.ascontiguousarray(hosts, dtype=np.uint32)
        _check(_lib.srla_set_candidates(self._h, _ptr(h) if len(h) else None, len(h)))

    # -- queries
    def union_weights(self, hosts):
        h = np.ascontiguousarray(hosts, dtype=np.uint32)
        rw, lw = np.empty(max(1, len(h)), np.uint32), np.empty(max(1, len(h)), np.uint32)
        _check(_lib.srla_union_weights(self._h, _ptr(h), len(h), _ptr(rw), _ptr(lw)))
        return rw[: len(h)], lw[: len(h)]

    def union_rough_weight(self, aip: int) -> int:
        return int(self.union_weights([aip])[0][0])

    def union_linear_weight(self, aip: int) -> int:
        return int(self.union_weights([aip])[1][0])

    def union_view(self, aip: int, include_linear: bool = True):
        ind = C.c_uint16()
        rough = np.empty(self.cfg.rough_slots, np.uint32)
        lin = np.empty(self.cfg.linear_slots, np.uint32) if include_linear else None
        _check(_lib.srla_union_view(self._h, aip, C.byref(ind), _ptr(rough), _ptr(lin)))
        return ind.value, rough, lin

    def row_active(self) -> np.ndarray:
        out = np.empty(self.cfg.rows, np.uint64)
        _check(_lib.srla_row_active(self._h, _ptr(out)))
        return out

    def row_fill_fraction(self, row: int) -> float:
        if row >= self.cfg.rows:
            raise ValueError("row index out of range")  # sea.hpp:249
        return float(self.row_active()[row]) / float(self.cfg.cols * self.cfg.linear_slots)

    def union_fill_product(self) -> float:
        p = 1.0
        words = float(self.cfg.cols * self.cfg.linear_slots)
        for a in self.row_active():
            p *= float(a) / words
        return p

    def corrected_estimate_from(self, weight: int, fill_product: float):
        est, has = C.c_double(), C.c_int()
        _check(_lib.srla_estimate_from(self._h, weight, fill_product, C.byref(est), C.byref(has)))
        return est.value if has.value else None

    # -- end of slice
    def report(self) -> np.ndarray:
        """report_window over the engine's candidate list -> ENTRY_DTYPE array."""
        n, fp = C.c_uint64(), C.c_double()
        cap = len(self.candidates()) + 1
        out = np.empty(cap, ENTRY_DTYPE)
        _check(_lib.srla_report(self._h, _ptr(out), cap, C.byref(n), C.byref(fp)))
        self.last_fill_product = fp.value
        return out[: n.value].copy()

    def report_window(self, csip) -> np.ndarray:
        self.set_candidates(csip)
        return self.report()

    def slide_engine(self) -> int:
        n = C.c_uint64()
        _check(_lib.srla_slide(self._h, C.byref(n)))
        return n.value

    def slide(self, csip) -> np.ndarray:
        """EstimatorArray::slide(csip) -> retained list (insertion order)."""
        self.set_candidates(csip)
        self.slide_engine()
        return self.candidates()

    def end_slice(self, slice_id: int, want_report: bool = True, cap: int | None = None):
        if cap is None:
            cap = len(self.candidates()) + 1
        out = np.empty(max(1, cap), ENTRY_DTYPE)
        n, nr = C.c_uint64(), C.c_uint64()
        _check(_lib.srla_end_slice(self._h, slice_id, int(want_report), _ptr(out), len(out),
                                   C.byref(n), C.byref(nr)))
        due = want_report and slice_id + 1 >= self.cfg.window
        return (out[: n.value].copy() if due else None), nr.value

    def end_slice_async(self, slice_id: int, out: np.ndarray, want_report: bool = True):
        """Start end-of-slice into `out` (ENTRY_DTYPE, kept alive by the caller)."""
        _check(_lib.srla_end_slice_async(self._h, slice_id, int(want_report), _ptr(out), len(out)))

    def end_slice_compact(self, slice_id: int, hosts: np.ndarray, weights: np.ndarray, est: np.ndarray,
                          flags: np.ndarray, want_report: bool = True):
        """end_slice handing the report off as (hosts, weights) + Eq. 9 table.
        Returns (entries written, retained candidates)."""
        n, nr = C.c_uint64(), C.c_uint64()
        _check(_lib.srla_end_slice_compact(self._h, slice_id, int(want_report), _ptr(hosts), _ptr(weights),
                                           len(hosts), C.byref(n), _ptr(est), _ptr(flags), C.byref(nr)))
        return n.value, nr.value

    def end_slice_wait(self):
        """-> (report entries written to the async buffer, retained candidates)."""
        n, nr = C.c_uint64(), C.c_uint64()
        _check(_lib.srla_end_slice_wait(self._h, C.byref(n), C.byref(nr)))
        return n.value, nr.value

    # -- raw rows (sea.hpp:341-346)
    def row_bytes(self, kind: int) -> int:
        b = C.c_uint64()
        _check(_lib.srla_row_bytes(self._h, kind, C.byref(b)))
        return b.value

    def export_row(self, row: int, kind: int) -> np.ndarray:
        dt = np.uint16 if kind == INDICATOR else self.wdtype
        out = np.empty(self.row_bytes(kind) // np.dtype(dt).itemsize, dt)
        _check(_lib.srla_export_row(self._h, row, kind, _ptr(out), out.nbytes))
        return out

    def import_row(self, row: int, kind: int, data):
        dt = np.uint16 if kind == INDICATOR else self.wdtype
        d = np.ascontiguousarray(data, dtype=dt)
        _check(_lib.srla_import_row(self._h, row, kind, _ptr(d), d.nbytes))

    def export_range(self, row: int, kind: int, offset: int, nbytes: int) -> np.ndarray:
        """Reference-layout bytes [offset, offset + nbytes) of a raw row."""
        out = np.empty(nbytes, np.uint8)
        _check(_lib.srla_export_range(self._h, row, kind, offset, _ptr(out), nbytes))
        return out

    def import_range(self, row: int, kind: int, offset: int, data):
        d = np.ascontiguousarray(data).view(np.uint8).reshape(-1)
        _check(_lib.srla_import_range(self._h, row, kind, offset, _ptr(d), d.nbytes))

    def state(self) -> dict:
        return {(k, i): self.export_row(i, k) for i in range(self.cfg.rows)
                for k in (INDICATOR, ROUGH, LINEAR)}

    def state_blocks(self, row: int, kind: int) -> np.ndarray:
        """Device-side block digests of a raw row (srla_state_blocks)."""
        nb = C.c_uint64()
        _check(_lib.srla_state_blocks(self._h, row, kind, None, 0, C.byref(nb)))
        out = np.empty(max(1, nb.value), np.uint64)
        _check(_lib.srla_state_blocks(self._h, row, kind, _ptr(out), len(out), C.byref(nb)))
        return out[: nb.value]

    def stats(self) -> dict:
        s = CStats()
        _check(_lib.srla_stats_get(self._h, C.byref(s)))
        return {n: getattr(s, n) for n, _ in CStats._fields_}

    def timing(self) -> dict:
        t = CTiming()
        _check(_lib.srla_timing_get(self._h, C.byref(t)))
        return {n: getattr(t, n) for n, _ in CTiming._fields_}

    def timing_reset(self):
        _check(_lib.srla_timing_reset(self._h))

    def synchronize(self):
        _check(_lib.srla_synchronize(self._h))

    def stream_handle(self) -> int:
        p = C.c_void_p()
        _check(_lib.srla_stream(self._h, C.byref(p)))
        return p.value or 0


class DetectPipeline:
    """sspread::DetectPipeline<W>::process_slice (pipeline.hpp:110-129) on the engine."""

    def __init__(self, cfg: SeaConfig, device: int = 0):
        if cfg.cols & (cfg.cols - 1):  # RunConfig::validate, pipeline.hpp:43-44
            raise ValueError("cols must be a power of two")
        self.sea = EstimatorArray(cfg, device)
        self.cfg = cfg
        self.pairs_scanned = 0
        self.slices_seen = 0

    def process_slice(self, slice_id: int, recs, want_report: bool = True):
        self.sea.scan(recs)
        self.pairs_scanned += int(recs.shape[0])
        self.slices_seen += 1
        report, _ = self.sea.end_slice(slice_id, want_report)
        return report

    def candidates(self) -> np.ndarray:
        return self.sea.candidates()


@dataclass
class PlantSpec:
    """sspread::PlantSpec (generator.hpp:36-64)."""
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


class DeviceTraceGenerator:
    """generate_trace (generator.hpp:117-161) on the device, slice by slice."""

    def __init__(self, spec: PlantSpec, device: int = 0):
        lib = load_library()
        plants = (CPlant * max(1, len(spec.plants)))()
        for i, p in enumerate(spec.plants):
            plants[i] = CPlant(*p)
        s = CSpec(spec.seed, spec.start_ts, spec.slice_seconds, spec.slices, spec.window, spec.a_base,
                  spec.b_base, spec.a_hosts, spec.b_hosts, spec.pairs_per_slice, len(spec.plants),
                  spec.skew, plants)
        h = C.c_void_p()
        _check(lib.srla_generator_create(C.byref(s), device, C.byref(h)))
        self._h, self.spec, self.device = h, spec, device

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.srla_generator_destroy(self._h)
            self._h = None

    def count(self, s: int) -> int:
        n = C.c_uint64()
        _check(_lib.srla_generate_slice(self._h, s, None, 0, C.byref(n), None))
        return n.value

    def generate_into(self, s: int, dev_ptr: int, cap: int, stream: int = 0) -> int:
        n = C.c_uint64()
        _check(_lib.srla_generate_slice(self._h, s, C.c_void_p(dev_ptr), cap, C.byref(n),
                                        C.c_void_p(stream) if stream else None))
        return n.value

    def slice_tensor(self, s: int):
        import torch
        n = self.count(s)
        t = torch.empty((max(1, n), 3), dtype=torch.int32, device=f"cuda:{self.device}")
        self.generate_into(s, t.data_ptr(), n, torch.cuda.current_stream(self.device).cuda_stream)
        return t[:n]


class ExactStore:
    """Exact sliding-window cardinalities on the device (srla_exact_*): the
    reference's SliceRingStore (oracle.hpp:136-203) over HBM-resident sorted
    pair sets."""

    def __init__(self, max_window: int, device: int = 0):
        lib = load_library()
        h = C.c_void_p()
        _check(lib.srla_exact_create(max_window, device, C.byref(h)))
        self._h, self.max_window, self.device = h, max_window, device

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.srla_exact_destroy(self._h)
            self._h = None

    def observe(self, recs):
        if _is_torch_cuda(recs):
            ptr, n, on_dev = recs.data_ptr(), recs.shape[0], 1
        else:
            recs = _as_records(recs)
            ptr, n, on_dev = recs.ctypes.data, recs.shape[0], 0
        _check(_lib.srla_exact_observe(self._h, C.c_void_p(ptr), n, on_dev))

    def end_slice(self):
        _check(_lib.srla_exact_end_slice(self._h))

    @property
    def current_slice(self) -> int:
        v = C.c_uint64()
        _check(_lib.srla_exact_current_slice(self._h, C.byref(v)))
        return v.value

    def pair_count(self) -> int:
        v = C.c_uint64()
        _check(_lib.srla_exact_pair_count(self._h, C.byref(v)))
        return v.value

    def cardinalities(self, t: int, k: int):
        """-> (hosts ascending, counts) of every host with a nonzero count in [t, t+k)."""
        n = C.c_uint64()
        rc = _lib.srla_exact_cardinalities(self._h, t, k, None, None, 0, C.byref(n))
        if rc not in (OK, E_CAPACITY):
            _check(rc)
        hosts, counts = np.empty(max(1, n.value), np.uint32), np.empty(max(1, n.value), np.uint64)
        _check(_lib.srla_exact_cardinalities(self._h, t, k, _ptr(hosts), _ptr(counts), len(hosts), C.byref(n)))
        return hosts[: n.value], counts[: n.value]


def block_sums(t) -> np.ndarray:
    """Block digests (srla_block_sums) of a contiguous CUDA tensor's bytes."""
    nbytes = t.numel() * t.element_size()
    nb = (nbytes + (1 << 20) - 1) >> 20
    out = np.empty(max(1, nb), np.uint64)
    _check(load_library().srla_block_sums(C.c_void_p(t.data_ptr()), nbytes, _ptr(out), len(out),
                                          C.c_void_p(_stream_of(t))))
    return out[:nb]


def owner_of(seed: int, aip: int, nparts: int) -> int:
    """Shard owning host `aip`: HashFamily(seed).reduce(3, aip, nparts)."""
    return load_library().srla_owner_of(seed & 0xFFFFFFFFFFFFFFFF, aip, nparts)


def partition_records(d_in_ptr: int, n: int, seed: int, nparts: int, part: int, d_out_ptr: int,
                      stream: int = 0) -> int:
    """Keep the device records owned by `part` (stable). Returns the kept count."""
    out = C.c_uint64()
    _check(load_library().srla_partition_records(C.c_void_p(d_in_ptr), n, seed & 0xFFFFFFFFFFFFFFFF, nparts,
                                                 part, C.c_void_p(d_out_ptr), C.byref(out),
                                                 C.c_void_p(stream) if stream else None))
    return out.value


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


# ---------------------------------------------------------------- ingest front end (trace.hpp)

def _stream_of(t):
    import torch
    return torch.cuda.current_stream(t.device).cuda_stream


def parse_srlt(data_dev):
    """SRLT v1 file bytes (uint8 CUDA tensor) -> (n, 3) int32 CUDA tensor of records.
    Raises InputError like for_each_record; the records before the failure are in
    the exception's `records` attribute."""
    import torch
    nbytes = data_dev.numel()
    cap = max(1, (nbytes - 5) // 12) if nbytes >= 5 else 1
    out = torch.empty((cap, 3), dtype=torch.int32, device=data_dev.device)
    n = C.c_uint64()
    rc = load_library().srla_parse_srlt(C.c_void_p(data_dev.data_ptr()), nbytes, C.c_void_p(out.data_ptr()),
                                        C.byref(n), C.c_void_p(_stream_of(data_dev)))
    if rc != OK:
        try:
            _check(rc)
        except InputError as e:
            e.records = out[: n.value]
            raise
    return out[: n.value]


def orient_records(recs_dev, prefix_addr: int, prefix_bits: int):
    """orient_record over a CUDA (n, 3) int32 batch -> (oriented records, stats dict)."""
    import torch
    n = recs_dev.shape[0]
    out = torch.empty((max(1, n), 3), dtype=torch.int32, device=recs_dev.device)
    m, st = C.c_uint64(), COrientStats()
    _check(load_library().srla_orient_records(C.c_void_p(recs_dev.data_ptr()), n, prefix_addr & 0xFFFFFFFF,
                                              prefix_bits, C.c_void_p(out.data_ptr()), C.byref(m), C.byref(st),
                                              C.c_void_p(_stream_of(recs_dev))))
    return out[: m.value], {k: getattr(st, k) for k, _ in COrientStats._fields_}


def slice_bounds(recs_dev, slice_seconds: int):
    """SlicePartitioner over an ordered CUDA batch -> numpy offsets (n_slices + 1)."""
    n = recs_dev.shape[0]
    lib = load_library()
    ns = C.c_uint64()
    st = C.c_void_p(_stream_of(recs_dev))
    _check(lib.srla_slice_bounds(C.c_void_p(recs_dev.data_ptr()), n, slice_seconds, None, 0, C.byref(ns), st))
    off = np.zeros(ns.value + 1, np.uint64)
    if ns.value:
        _check(lib.srla_slice_bounds(C.c_void_p(recs_dev.data_ptr()), n, slice_seconds,
                                     off.ctypes.data_as(C.c_void_p), len(off), C.byref(ns), st))
    return off
