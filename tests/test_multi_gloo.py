"""Multi-GPU host logic on CPU: owner partition, report all-gather and merge
(paper_1803_10369_b200/shard.py) with world_size 2 over gloo. Each rank's
shard engine here is the CPU oracle pipeline (the checker); on GPUs it is the
engine, exercised by bench.py --gpus N."""
from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import golden_flow as GF
import scenarios as S

SCEN = "pipeline_small_3000"


def test_owner_matches_reference_hash_family(oracle, srla_lib):
    from paper_1803_10369_b200.shard import owner_of
    rng = np.random.default_rng(3)
    aips = rng.integers(0, 2**32, 5000, dtype=np.uint64).astype(np.uint32)
    for seed in (0, 0x5EA00001, 0xFFFFFFFFFFFFFFFF):
        for n in (1, 2, 3, 8):
            got = owner_of(seed, aips, n)
            want = [oracle.hash_reduce(seed, 3, int(a), n) for a in aips[:300]]
            assert got[:300].tolist() == want
            assert [srla_lib.srla_owner_of(seed, int(a), n) for a in aips[:50]] == got[:50].tolist()
            assert got.max() < n


class OracleShard:
    """Shard adapter: the oracle pipeline behind the engine's scan/end_slice calls."""

    def __init__(self, cfg):
        from oracle.pyoracle import Checker, SeaConfig
        self.p = Checker("orc").pipeline(SeaConfig(**cfg.as_dict()))
        self.recs = np.zeros((0, 3), np.uint32)

    def scan(self, recs):
        self.recs = np.asarray(recs, np.uint32).reshape(-1, 3)

    def end_slice(self, slice_id, want):
        from paper_1803_10369_b200.srla import ENTRY_DTYPE
        r = self.p.process_slice(slice_id, self.recs, want)
        if r is None:
            return None, 0
        out = np.zeros(len(r["host"]), ENTRY_DTYPE)
        out["host"], out["union_weight"], out["estimate"] = r["host"], r["weight"], r["estimate"]
        out["has_estimate"], out["is_super"] = r["has_estimate"], r["is_super"]
        return out, len(out)


def _worker(rank, world, port, outdir, slices, cfg):
    import torch.distributed as dist
    from paper_1803_10369_b200.shard import ShardedPipeline
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sp = ShardedPipeline(OracleShard(cfg), cfg.seed, cfg.window, dist=dist)
    reports = [sp.process_slice(s, recs, filter_owned=True) for s, recs in enumerate(slices)]
    np.save(os.path.join(outdir, f"r{rank}.npy"), np.array(reports, dtype=object), allow_pickle=True)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_gloo_sharded_reports(oracle):
    from paper_1803_10369_b200.shard import merge_reports, partition_host
    cfg, _ = S.SCENARIOS[SCEN]
    slices = GF.scenario_slices(SCEN, oracle)
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(2, _free_port(), d, slices, cfg), nprocs=2, join=True,
                           start_method="spawn")
        got = [np.load(os.path.join(d, f"r{r}.npy"), allow_pickle=True) for r in range(2)]
    # single-process emulation: two independent shard pipelines on owner-filtered sub-traces
    shards = [OracleShard(cfg) for _ in range(2)]
    for s, recs in enumerate(slices):
        parts = []
        for r in range(2):
            shards[r].scan(partition_host(recs, cfg.seed, 2, r))
            parts.append(shards[r].end_slice(s, True)[0])
        want = merge_reports(parts) if parts[0] is not None else None
        for r in range(2):
            g = got[r][s]
            if want is None:
                assert g is None
            else:
                assert np.array_equal(g, want), f"slice {s} rank {r}"
    assert any(x is not None and len(x) for x in got[0])


def _compact_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    from paper_1803_10369_b200.shard import allgather_report_compact, merge_reports
    from paper_1803_10369_b200.srla import ENTRY_DTYPE
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(10 + rank)
    L = 65
    est = rng.random(L) * 1000
    flg = rng.integers(0, 4, L).astype(np.uint8)
    hosts = np.sort(rng.choice(2**31, 500 + 100 * rank, replace=False).astype(np.uint32) * 2 + rank)  # disjoint
    w = rng.integers(0, L, len(hosts)).astype(np.uint32)
    ent = np.zeros(len(hosts), ENTRY_DTYPE)
    ent["host"], ent["union_weight"], ent["estimate"] = hosts, w, est[w]
    ent["has_estimate"], ent["is_super"] = flg[w] & 1, flg[w] >> 1
    h, wt, e, f = allgather_report_compact(torch.from_numpy(hosts.astype(np.int64)), torch.from_numpy(w.astype(np.int64)),
                                           torch.from_numpy(est), torch.from_numpy(flg), dist)
    parts = [None] * world
    dist.all_gather_object(parts, ent)
    want = merge_reports(parts)
    from paper_1803_10369_b200.shard import allgather_report_entries
    dev_rows = allgather_report_entries(ent, dist, torch.device("cpu"))
    ok_rows = dev_rows.numpy().tobytes() == want.tobytes()
    ok = (np.array_equal(h.numpy(), want["host"].astype(np.int64)) and np.array_equal(wt.numpy(), want["union_weight"])
          and np.array_equal(e.numpy(), want["estimate"]) and np.array_equal(f.numpy() & 1, want["has_estimate"])
          and np.array_equal(f.numpy() >> 1, want["is_super"]) and ok_rows)
    open(os.path.join(out_dir, f"ok{rank}"), "w").write("1" if ok else "0")
    dist.destroy_process_group()


def test_two_rank_gloo_compact_report_allgather():
    """The bench's device-resident report all-gather (hosts + weights + each
    shard's Eq. 9 table, merged by host) equals the entry-level merge."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_compact_worker, args=(2, port, d), nprocs=2, join=True)
        assert open(os.path.join(d, "ok0")).read() == "1" and open(os.path.join(d, "ok1")).read() == "1"
