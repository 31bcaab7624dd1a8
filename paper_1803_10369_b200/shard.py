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
