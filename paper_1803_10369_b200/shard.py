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
