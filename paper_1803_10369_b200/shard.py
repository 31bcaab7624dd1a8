"""Multi-GPU sharding of the SRLA hot path.

Hosts are owner-partitioned: owner(aip) = HashFamily(seed).reduce(3, aip, N)
(hash index 3 is unused by the reference, hash.hpp:70-73). Every rank keeps an
independent full sketch for the hosts it owns, so a host's result equals what a
CPU reference pipeline fed the owner-filtered sub-trace (in order) produces.
The only collective is the per-slice report all-gather; entries of different
ranks are disjoint by host and merged by address (report_window sorts by host,
sea.hpp:294-295).
"""
from __future__ import annotations

import numpy as np

from .srla import ENTRY_DTYPE

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _avalanche64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        x = (x ^ (x >> np.uint64(30))) * _M1
        x = (x ^ (x >> np.uint64(27))) * _M2
    return x ^ (x >> np.uint64(31))


def owner_of(seed: int, aip, nparts: int) -> np.ndarray:
    """reduce(3, aip, nparts) for an array of hosts (host-side, vectorised)."""
    with np.errstate(over="ignore"):
        sub = _avalanche64(np.array([np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + _GOLDEN * np.uint64(4)],
                                    dtype=np.uint64))[0]
    h = _avalanche64(np.asarray(aip, dtype=np.uint64) ^ sub) & np.uint64(0xFFFFFFFF)
    return ((h * np.uint64(nparts)) >> np.uint64(32)).astype(np.uint32)


def partition_host(recs: np.ndarray, seed: int, nparts: int, part: int) -> np.ndarray:
    """Records (n, 3) whose src is owned by `part`, original order kept."""
    recs = np.asarray(recs, dtype=np.uint32).reshape(-1, 3)
    return recs[owner_of(seed, recs[:, 1], nparts) == part]


def merge_reports(parts) -> np.ndarray:
    """Disjoint per-shard reports -> one report sorted by host."""
    parts = [np.asarray(p) for p in parts if p is not None and len(p)]
    if not parts:
        return np.empty(0, ENTRY_DTYPE)
    merged = np.concatenate(parts)
    return merged[np.argsort(merged["host"], kind="stable")]


def allgather_report(entries: np.ndarray, dist, device=None) -> np.ndarray:
    """All-gather variable-length report arrays (ENTRY_DTYPE) and merge.

    Works with any torch.distributed backend: NCCL (pass the CUDA device) or
    gloo (CPU tensors)."""
    import torch
    world = dist.get_world_size()
    entries = np.ascontiguousarray(entries, dtype=ENTRY_DTYPE)
    n = torch.tensor([len(entries)], dtype=torch.int64, device=device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    mx = max(counts + [1])
    pad = np.zeros(mx, ENTRY_DTYPE)
    pad[: len(entries)] = entries
    t = torch.from_numpy(pad.view(np.uint8).copy()).to(device if device is not None else "cpu")
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)
    return merge_reports([o.cpu().numpy().view(ENTRY_DTYPE)[:c] for o, c in zip(outs, counts)])


class ShardedPipeline:
    """One rank of an owner-partitioned DetectPipeline.

    `sketch` is this rank's shard engine (an EstimatorArray on the rank's GPU
    in production); `process_slice` takes the rank's owned records for the
    slice, or the global slice with `filter_owned=True`."""

    def __init__(self, sketch, seed: int, window: int, dist=None, device=None):
        self.sketch, self.seed, self.window = sketch, seed, window
        self.dist, self.device = dist, device
        self.world = dist.get_world_size() if dist else 1
        self.rank = dist.get_rank() if dist else 0

    def process_slice(self, slice_id: int, recs, filter_owned: bool = False):
        if filter_owned:
            recs = partition_host(recs, self.seed, self.world, self.rank)
        self.sketch.scan(recs)
        report, _ = self.sketch.end_slice(slice_id, True)
        if report is None:
            return None
        return allgather_report(report, self.dist, self.device) if self.dist else merge_reports([report])


def allgather_report_compact(hosts, weights, est_lut, flag_lut, dist):
    """Device-resident report all-gather for the bench's N-GPU path.

    hosts, weights: this rank's report (ascending hosts) as 1-D tensors on the
    collective's device; est_lut (float64) and flag_lut (uint8: bit 0
    has_estimate, bit 1 is_super) this shard's Eq. 9 table over the g'+1
    weights (each shard has its own fill product). Returns the merged report
    (hosts ascending) as device tensors (host, weight, estimate, flags) — one
    all-gather of 8-byte (host, weight) words plus the tables, a merge on the
    device, nothing back to the host."""
    import torch
    world = dist.get_world_size()
    dev = hosts.device
    n = torch.tensor([hosts.numel()], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    mx = max(counts + [1])
    word = torch.zeros(mx, dtype=torch.int64, device=dev)
    word[: hosts.numel()] = (hosts.to(torch.int64) << 32) | weights.to(torch.int64)
    words = [torch.empty_like(word) for _ in range(world)]
    dist.all_gather(words, word)
    luts = [torch.empty_like(est_lut) for _ in range(world)]
    dist.all_gather(luts, est_lut)
    flags = [torch.empty_like(flag_lut) for _ in range(world)]
    dist.all_gather(flags, flag_lut)
    # shards own disjoint hosts: the merged order is a sort by host
    allw = torch.cat([w[:c] for w, c in zip(words, counts)])
    shard = torch.cat([torch.full((c,), r, dtype=torch.int64, device=dev) for r, c in enumerate(counts)])
    host = (allw >> 32) & 0xFFFFFFFF  # int64 words: undo the sign of hosts >= 2^31
    order = torch.argsort(host)
    host, weight, shard = host[order], (allw & 0xFFFFFFFF)[order], shard[order]
    L = est_lut.numel()
    est = torch.stack(luts).reshape(-1)[shard * L + weight]
    flg = torch.stack(flags).reshape(-1)[shard * L + weight]
    return host, weight, est, flg


def allgather_report_entries(entries: np.ndarray, dist, device):
    """allgather_report with the merge on the device: this rank's srla_entry
    array (24 bytes each, hosts ascending) is gathered from every rank and
    merged by host on `device`; returns the merged entries as a (n, 24)
    uint8 tensor on `device` (nothing copied back to the host)."""
    import torch
    world = dist.get_world_size()
    entries = np.ascontiguousarray(entries, dtype=ENTRY_DTYPE)
    n = torch.tensor([len(entries)], dtype=torch.int64, device=device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    mx = max(counts + [1])
    rows = torch.zeros((mx, ENTRY_DTYPE.itemsize), dtype=torch.uint8, device=device)
    if len(entries):
        rows[: len(entries)] = torch.from_numpy(entries.view(np.uint8).reshape(-1, ENTRY_DTYPE.itemsize)).to(device)
    outs = [torch.empty_like(rows) for _ in range(world)]
    dist.all_gather(outs, rows)
    merged = torch.cat([o[:c] for o, c in zip(outs, counts)])
    host = merged[:, :4].contiguous().view(torch.int32).reshape(-1).to(torch.int64) & 0xFFFFFFFF
    return merged[torch.argsort(host)]


# ---------------------------------------------------------------- C-ABI sharded pipeline (srla_shard_*)

import ctypes as C  # noqa: E402

OWNED, RANGE = 0, 1  # SRLA_SHARD_OWNED / SRLA_SHARD_RANGE

_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)
_ALLTOALLV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_void_p,
                         C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_void_p)


class CTransport(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("rank", C.c_uint32), ("world", C.c_uint32), ("host_memory", C.c_int),
                ("allgather", _ALLGATHER), ("alltoallv", _ALLTOALLV)]


def _lib():
    from .srla import load_library
    lib = load_library()
    if not getattr(lib, "_shard_sigs", False):
        vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
        for name, res, args in (
                ("srla_nccl_unique_id", i32, [vp]),
                ("srla_transport_nccl", i32, [vp, u32, u32, i32, C.POINTER(CTransport)]),
                ("srla_transport_nccl_destroy", i32, [C.POINTER(CTransport)]),
                ("srla_shard_create", i32, [vp, i32, C.POINTER(CTransport), C.POINTER(vp)]),
                ("srla_shard_destroy", i32, [vp]),
                ("srla_shard_engine", i32, [vp, C.POINTER(vp)]),
                ("srla_shard_last_report", i32, [vp, vp, u64, C.POINTER(u64)]),
                ("srla_shard_process_slice", i32, [vp, u64, vp, u64, i32, i32, i32, vp, u64, C.POINTER(u64),
                                                   C.POINTER(u64)])):
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        lib._shard_sigs = True
    return lib


class GlooTransport:
    """srla_transport over a torch.distributed process group on host memory
    (gloo): the library stages device data through pinned buffers. For tests
    and for ranks that share a GPU (NCCL refuses two ranks on one device)."""

    def __init__(self, dist):
        import torch
        self.dist, self.torch = dist, torch
        self.rank, self.world = dist.get_rank(), dist.get_world_size()

        def allgather(ctx, send, recv, nbytes, stream):
            try:
                src = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), (max(1, nbytes),))[:nbytes]
                t = torch.from_numpy(src.copy())
                outs = [torch.empty_like(t) for _ in range(self.world)]
                dist.all_gather(outs, t)
                if nbytes:
                    dst = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)), (nbytes * self.world,))
                    dst[:] = torch.cat(outs).numpy()
                return 0
            except Exception as e:  # noqa: BLE001 (reported as a transport failure)
                print("gloo allgather:", e)
                return 1

        def alltoallv(ctx, send, sb, so, recv, rb, ro, stream):
            try:
                W = self.world
                sbytes = [sb[j] for j in range(W)]
                soff = [so[j] for j in range(W)]
                total = soff[-1] + sbytes[-1] if W else 0
                src = np.ctypeslib.as_array(C.cast(send, C.POINTER(C.c_uint8)), (max(1, total),))[:total].copy()
                # variable all-to-all as an all-gather of (sizes, payload)
                mx = torch.tensor([total], dtype=torch.int64)
                mxs = [torch.zeros_like(mx) for _ in range(W)]
                dist.all_gather(mxs, mx)
                cap = max(int(m.item()) for m in mxs + [torch.tensor([1])])
                pay = torch.zeros(cap, dtype=torch.uint8)
                pay[:total] = torch.from_numpy(src)
                meta = torch.tensor(sbytes + soff, dtype=torch.int64)
                pays = [torch.empty_like(pay) for _ in range(W)]
                metas = [torch.empty_like(meta) for _ in range(W)]
                dist.all_gather(pays, pay)
                dist.all_gather(metas, meta)
                rtotal = ro[W - 1] + rb[W - 1]
                dst = np.ctypeslib.as_array(C.cast(recv, C.POINTER(C.c_uint8)), (max(1, rtotal),))
                for i in range(W):
                    m = metas[i].numpy()
                    nb, off = int(m[self.rank]), int(m[W + self.rank])
                    assert nb == rb[i]
                    dst[ro[i]:ro[i] + nb] = pays[i].numpy()[off:off + nb]
                return 0
            except Exception as e:  # noqa: BLE001
                print("gloo alltoallv:", e)
                return 1

        self._cb = (_ALLGATHER(allgather), _ALLTOALLV(alltoallv))
        self.c = CTransport(None, self.rank, self.world, 1, self._cb[0], self._cb[1])


class NcclTransport:
    """srla_transport_nccl: the library's own NCCL communicator (one rank per
    GPU); the unique id travels over the caller's process group."""

    def __init__(self, dist, device):
        from .srla import _check
        lib = _lib()
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            _check(lib.srla_nccl_unique_id(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0)
        uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        self.c = CTransport()
        _check(lib.srla_transport_nccl(uid, self.rank, self.world, device, C.byref(self.c)))

    def close(self):
        if self.c.ctx:
            _lib().srla_transport_nccl_destroy(C.byref(self.c))

    def __del__(self):
        self.close()


class EngineShard:
    """One rank of the owner-partitioned pipeline through the C ABI
    (srla_shard_*): scan, report all-gather merged by host on the device, slide."""

    def __init__(self, cfg, transport, device: int = 0):
        from .srla import _check
        lib = _lib()
        self.cfg, self.transport, self.device = cfg, transport, device
        h = C.c_void_p()
        c = cfg.to_c()
        _check(lib.srla_shard_create(C.byref(c), device, C.byref(transport.c), C.byref(h)))
        self._h = h
        e = C.c_void_p()
        _check(lib.srla_shard_engine(h, C.byref(e)))
        from .srla import EstimatorArray
        self.engine = EstimatorArray.__new__(EstimatorArray)  # a view: the shard owns the engine
        self.engine.cfg, self.engine.device, self.engine._h = cfg, device, e
        self.engine.word_bytes = 1 if cfg.recorder_bits <= 8 else 2 if cfg.recorder_bits <= 16 else 4
        self.engine.wdtype = {1: np.uint8, 2: np.uint16, 4: np.uint32}[self.engine.word_bytes]
        self.engine.close = lambda: None
        self.cap = 1 << 12
        self.out = np.empty(self.cap, ENTRY_DTYPE)

    def process_slice(self, slice_id, recs, mode=OWNED, want_report=True):
        """-> (merged report or None, records this rank scanned)."""
        from .srla import E_CAPACITY, _as_records, _check, _is_torch_cuda
        if _is_torch_cuda(recs):
            import torch
            # srla_shard_process_slice orders after the legacy default stream;
            # records produced on another stream are waited for here
            torch.cuda.current_stream(recs.device).synchronize()
            ptr, n, on_dev = recs.data_ptr(), recs.shape[0], 1
        else:
            recs = _as_records(recs)
            ptr, n, on_dev = recs.ctypes.data, recs.shape[0], 0
        lib = _lib()
        n_out, n_scan = C.c_uint64(), C.c_uint64()
        rc = lib.srla_shard_process_slice(self._h, slice_id, C.c_void_p(ptr), n, on_dev, mode, int(want_report),
                                          C.c_void_p(self.out.ctypes.data), self.cap, C.byref(n_out), C.byref(n_scan))
        if rc == E_CAPACITY:  # the slice completed; fetch the merged report with room
            self.reserve(n_out.value)
            _check(lib.srla_shard_last_report(self._h, C.c_void_p(self.out.ctypes.data), self.cap, C.byref(n_out)))
        else:
            _check(rc)
        due = want_report and slice_id + 1 >= self.cfg.window
        return (self.out[: n_out.value].copy() if due else None), n_scan.value

    def reserve(self, entries):
        if entries > self.cap:
            self.cap = max(entries, 2 * self.cap)
            self.out = np.empty(self.cap, ENTRY_DTYPE)

    def close(self):
        if getattr(self, "_h", None):
            _lib().srla_shard_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()
