"""Full-size parity digests from the REFERENCE (oracle/_ref, the unmodified
headers): BASELINE.json's C1 (seeds 11-15) / C2 / C3 / C5 workloads, every slice.

The reference is driven like DetectPipeline::process_slice with ONE scan worker
(record order: pipeline.hpp:134-139, the parity definition of SURVEY.md §8c);
report_window's fill product and the slide run chunked over the host's threads,
which sea.hpp:23-26 guarantees does not change results. The slices come from
ref_generate_slice, the reference generator's own pieces run in parallel
(pinned byte-identical to generate_trace by tests/test_oracle_golden.py).

Per slice: the records' block digest, the candidate-sink pushes, the ordered
candidate list, the report entries (host, weight, estimate bits, flags), the
retained list and the recorder state (block digests of every indicator / rough
/ linear row in SSEA order, digest.cuh) — each as (n, sha256).

  python tests/golden/make_fullsize.py c2 [--slices 12] [--threads N]
  python tests/golden/make_fullsize.py c1 --seed 11      (120 slices; seeds 11-15)
  python tests/golden/make_fullsize.py crit4 --seed 1    (seeds 1-5; crit6: seeds 21-25)

C2 and C5 need ~5 GiB of host RAM; C3 (64 GiB of linear recorders) needs the
GPU box's host: run it there through gpurun and commit the JSON it writes.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from golden_flow import _lst, _report  # noqa: E402
from oracle.pyoracle import Checker, PlantSpec, SeaConfig  # noqa: E402
from paper_1803_10369_b200 import workloads as WL  # noqa: E402


def sha_blocks(parts):
    h = hashlib.sha256()
    for p in parts:
        h.update(np.ascontiguousarray(p, dtype=np.uint64).tobytes())
    return h.hexdigest()


def state_digest_ref(flow, rows):
    return sha_blocks(flow.state_blocks(i, k) for i in range(rows) for k in (0, 1, 2))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", choices=["c1", "crit4", "crit6", "c2", "c3", "c5"])
    ap.add_argument("--slices", type=int, default=None, help="12 (c2/c3/c5), 120 (c1)")
    ap.add_argument("--seed", type=int, default=11, help="c1 trace seed (11-15)")
    ap.add_argument("--pairs", type=int, default=WL.PAIRS)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    ref = Checker("ref")
    if a.workload == "c1":
        a.slices = a.slices or 120
        cfg, spec, name = WL.c1_sketch(), WL.c1_spec(a.seed, a.slices), f"c1_s{a.seed}"
    elif a.workload in ("crit4", "crit6"):  # acceptance criteria 4 / 6: 3 slices, z = 1, k = 1
        a.slices = 3
        cols, pairs = (65536, 150_000) if a.workload == "crit4" else (1024, 600_000)
        cfg, spec, name = WL.discrete_sketch(cols), WL.discrete_spec(a.seed, pairs), f"{a.workload}_s{a.seed}"
    else:
        a.slices = a.slices or 12
        cfg = WL.sketch_cfg(WL.cols_of(a.workload))
        spec, name = WL.trace_spec(a.pairs, slices=a.slices, workload=a.workload), a.workload
    flow = ref.flow(SeaConfig(**cfg), threads=a.threads)
    out = a.out or os.path.join(HERE, f"fullsize_{name}.json")
    doc = {"workload": name, "cfg": cfg, "spec": spec, "slices": [],
           "source": "oracle/_ref (unmodified reference headers), 1 scan worker, bulk passes chunked"}
    buf = None
    whole = None
    if spec.get("slice_seconds", 1) != 1:  # generate_trace, then SlicePartitioner (trace.hpp:243-281)
        recs_all = ref.generate(PlantSpec(**spec))
        ids = (recs_all[:, 0].astype(np.int64) - int(recs_all[0, 0])) // spec["slice_seconds"]
        whole = [recs_all[ids == k] for k in range(a.slices)]
    for s in range(a.slices):
        t0 = time.time()
        if whole is not None:
            recs = np.ascontiguousarray(whole[s])
        else:
            recs = ref.generate_slice(PlantSpec(**spec), s, a.threads, out=buf)
            buf = recs if buf is None else buf
        rec = {"records": {"n": int(len(recs)), "sha": sha_blocks([ref.block_sums(recs, a.threads)])}}
        t1 = time.time()
        pushes = flow.scan(recs)
        t2 = time.time()
        rec["pushes"] = _lst(pushes)
        rec["csip"] = _lst(flow.candidates())
        rec["report"] = None
        if s + 1 >= cfg["window"]:
            r = flow.report(s + 1 - cfg["window"])
            rec["report"] = _report(r["host"], r["weight"], r["estimate"], r["has_estimate"], r["is_super"])
        flow.slide()
        rec["retained"] = _lst(flow.candidates())
        t3 = time.time()
        rec["state"] = state_digest_ref(flow, cfg["rows"])
        doc["slices"].append(rec)
        print(f"[{a.workload}] slice {s}: gen {t1 - t0:.1f}s scan {t2 - t1:.1f}s eos {t3 - t2:.1f}s "
              f"state {time.time() - t3:.1f}s pushes {len(pushes)} csip {rec['csip']['n']} "
              f"report {rec['report']['n'] if rec['report'] else '-'} retained {rec['retained']['n']}", flush=True)
        json.dump(doc, open(out, "w"), indent=1)
    print("wrote", out)


if __name__ == "__main__":
    main()
