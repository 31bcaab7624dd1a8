"""Two or three ranks, each running the CUDA engine through the C ABI's sharded
pipeline (srla_shard_*), on one GPU over gloo (NCCL refuses two ranks on one
device; the transport is the only difference from the NCCL path).

For each input mode — records already owner-partitioned (SRLA_SHARD_OWNED,
the north star's host-hash ingest) and contiguous slice ranges exchanged
all-to-all on the device (SRLA_SHARD_RANGE) — every merged report must equal
the host-sorted merge of two reference pipelines (the C restatement, pinned
to the reference) run on the owner-filtered sub-traces in order
(pipeline.hpp:110-129), and each rank's candidate list must equal its
reference shard's. A world-1 NCCL transport checks the library's NCCL path.
"""
from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

import golden_flow as GF
import scenarios as S

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir, name, mode, force_bins):
    import torch.distributed as dist

    if force_bins:
        os.environ["SRLA_FORCE_BINS"] = "1"
    from oracle.pyoracle import Checker
    from paper_1803_10369_b200.shard import OWNED, EngineShard, GlooTransport, partition_host
    from paper_1803_10369_b200.srla import SeaConfig
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, _ = S.SCENARIOS[name]
    slices = GF.scenario_slices(name, Checker("orc"))
    shard = EngineShard(SeaConfig(**cfg.as_dict()), GlooTransport(dist), device=0)
    reps, cands, scanned = [], [], []
    for s, recs in enumerate(slices):
        if mode == OWNED:
            mine = partition_host(recs, cfg.seed, world, rank)
        else:  # contiguous range of the slice, ranks in order
            lo, hi = len(recs) * rank // world, len(recs) * (rank + 1) // world
            mine = recs[lo:hi]
        rep, n = shard.process_slice(s, mine, mode=mode)
        reps.append(rep)
        scanned.append(n)
        cands.append(shard.engine.candidates())
    np.save(os.path.join(outdir, f"r{rank}.npy"), np.array([reps, cands, scanned], dtype=object), allow_pickle=True)
    shard.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("name,force_bins,world", [("contended", False, 2), ("c1_shape", False, 2),
                                                    ("drift_evict", True, 2), ("pipeline_small_3000", False, 3)])
def test_engine_shards_match_reference(gpu, oracle, name, force_bins, world, mode):
    from paper_1803_10369_b200.shard import merge_reports, partition_host
    cfg, _ = S.SCENARIOS[name]
    slices = GF.scenario_slices(name, oracle)
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _port(), d, name, mode, force_bins), nprocs=world, join=True,
                           start_method="spawn")
        got = [np.load(os.path.join(d, f"r{r}.npy"), allow_pickle=True) for r in range(world)]
    from oracle.pyoracle import SeaConfig as OC
    pipes = [oracle.pipeline(OC(**cfg.as_dict())) for _ in range(world)]
    nonempty = 0
    for s, recs in enumerate(slices):
        parts = []
        for r in range(world):
            sub = partition_host(recs, cfg.seed, world, r)
            rep = pipes[r].process_slice(s, sub, True)
            assert got[r][2][s] == len(sub), f"slice {s} rank {r}: scanned {got[r][2][s]} of {len(sub)} owned"
            assert np.array_equal(got[r][1][s], pipes[r].candidates()), f"slice {s} rank {r}: candidates differ"
            if rep is not None:
                from paper_1803_10369_b200.srla import ENTRY_DTYPE
                e = np.zeros(len(rep["host"]), ENTRY_DTYPE)
                e["host"], e["union_weight"], e["estimate"] = rep["host"], rep["weight"], rep["estimate"]
                e["has_estimate"], e["is_super"] = rep["has_estimate"], rep["is_super"]
                parts.append(e)
        want = merge_reports(parts) if parts else None
        for r in range(world):
            g = got[r][0][s]
            if want is None:
                assert g is None
            else:
                assert g.tobytes() == want.tobytes(), f"slice {s} rank {r}: merged report differs"
                nonempty += len(want) > 0
    assert nonempty > 0


def test_world1_nccl_transport_shard(gpu, oracle):
    """The library's NCCL transport (dlopen'd libnccl) at world size 1: the
    sharded pipeline equals the plain engine flow."""
    import torch.distributed as dist
    from paper_1803_10369_b200.shard import RANGE, EngineShard, NcclTransport
    from paper_1803_10369_b200.srla import SeaConfig
    name = "contended"
    cfg, _ = S.SCENARIOS[name]
    slices = GF.scenario_slices(name, oracle)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        t = NcclTransport(dist, device=0)
        shard = EngineShard(SeaConfig(**cfg.as_dict()), t, device=0)
        from oracle.pyoracle import SeaConfig as OC
        pipe = oracle.pipeline(OC(**cfg.as_dict()))
        for s, recs in enumerate(slices):
            got, _ = shard.process_slice(s, recs, mode=RANGE)
            want = pipe.process_slice(s, recs, True)
            if want is None:
                assert got is None
            else:
                assert np.array_equal(got["host"], want["host"]) and np.array_equal(got["union_weight"], want["weight"])
                assert got["estimate"].tobytes() == want["estimate"].tobytes()
        shard.close()
        t.close()
    finally:
        dist.destroy_process_group()
