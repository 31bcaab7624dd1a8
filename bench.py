#!/usr/bin/env python
"""SRLA benchmark: packets/s scanned + end-of-slice latency (BASELINE.json).

Workload (BASELINE.json configs[1], "C2" in SURVEY.md §8d): one B200 per rank,
sketch u=4, v=2^20, g=8, g'=1024, z=4 (u8 recorders), k=10, theta=1024, seed
0x5EA00001; synthetic trace = the reference generator's C2 spec (uniform 4M
sources, Zipf(1.0) 4M destinations, 50 planted super points), 1e8 packets per
slice per GPU, produced byte-identically on the device and resident in HBM
(1.2 GB per slice, > L2, so no flush is needed between steps).

A step = DetectPipeline::process_slice on one slice: scan (K1..K5) + report
(when the window is full) + slide. N > 1: hosts are owner-partitioned
(reduce(3, aip, N)); every rank keeps an independent sketch for its hosts and
the per-slice report is all-gathered over NCCL (the only collective).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "packets/sec scanned (1/2/4/8 B200); end-of-slice estimation latency ms"
ALGO_BYTES_PER_PACKET = 140  # 12 B streamed record + 4 rows x one 32-B sector update


def plant_cards():
    return [int(math.floor(1152.0 * math.pow(16384.0 / 1152.0, i / 49.0) + 0.5)) for i in range(50)]


def sketch_cfg(cols):
    return dict(rows=4, cols=cols, rough_slots=8, linear_slots=1024, recorder_bits=4, window=10, theta=1024,
                seed=0x5EA00001)


def trace_spec(pairs, slices=12, workload="c2"):
    if workload == "c3":  # uniform, ~1e6 candidate super points
        return dict(seed=3, slices=slices, window=10, a_hosts=1 << 20, b_hosts=1 << 24, pairs_per_slice=pairs,
                    skew=0.0, plants=[])
    return dict(seed=1, slices=slices, window=10, a_hosts=4194304, b_hosts=1 << 22, pairs_per_slice=pairs,
                skew=1.0, plants=[(0x0AC80001 + i, c, 0, 0xFFFFFFFF) for i, c in enumerate(plant_cards())])


WORKLOADS = {
    "c2": "C2: u=4 v=2^20 g=8 g'=1024 z=4 k=10 theta=1024 seed=0x5EA00001; trace seed 1, 4M uniform sources, "
          "Zipf(1.0) 4M destinations, 50 plants",
    "c3": "C3: u=4 v=2^24 g=8 g'=1024 z=4 k=10 theta=1024 seed=0x5EA00001 (64 GiB linear table, epoch stamps); "
          "trace seed 3, 1M uniform sources, 16M uniform destinations (~1e6 candidates)",
}


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, local_rank, period_ms=100):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        idx = str(local_rank)
        if vis:
            parts = vis.split(",")
            if local_rank < len(parts):
                idx = parts[local_rank].strip()
        self.lines = []
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={idx}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", str(period_ms)],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for name, v in zip(self.NAMES, f[2:6]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- rooflines

def ncu_traffic(workload):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of each kernel
    for this workload, from the committed ncu --set full summary
    (profiles/ncu_summary.json, tools/ncu_summary.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return {}
    wl = json.load(open(p)).get("workloads", {}).get(workload, {})
    return {k: v for k, v in wl.items()}


def kernel_rooflines(tm, step_ms_total, cfg, peak, peak_src, packets, steps, workload):
    """Per-kernel algorithmic bytes / device time (CUDA events on the engine
    stream around every launch, summed over the timed steps).

    K1 k_scan_bin: 12 B record + rows x 4 B bin entry per packet (the direct
      k_scan: 12 B + rows x one 32-B sector update);
    k_split: 4 B coarse entry read + 2 B fine entry written per mark;
    apply (k_slice_apply_bulk / k_slice_stamp): 2 B fine entry per mark +
      every streamed table slice read and written;
    gather (k_union_linear): candidates x rows x g' x W.
    The scan-path figure is SURVEY.md §8d's 140 B per packet (12 B record +
    4 random 32-B sector updates) over K1 + split + apply time."""
    binned = tm["split_kernel_launches"] > 0 or tm["apply_kernel_launches"] > 0
    rows = cfg.rows
    traffic = ncu_traffic(workload)
    ks = {
        "k_scan_bin" if binned else "k_scan": (
            tm["scan_kernel_ms"], tm["scan_kernel_launches"],
            tm["scan_kernel_records"] * ((12 + 4 * rows) if binned else (12 + 32 * rows))),
        "k_split": (tm["split_kernel_ms"], tm["split_kernel_launches"], tm["split_entries"] * 6),
        "k_slice_apply": (tm["apply_kernel_ms"], tm["apply_kernel_launches"],
                          tm["apply_entries"] * 2 + tm["apply_stream_bytes"]),
        "k_union_linear": (tm["gather_kernel_ms"], tm["gather_kernel_launches"], tm["gather_bytes"]),
    }
    kernels = {}
    for name, (kms, n, byts) in ks.items():
        if n == 0 or kms <= 0:
            continue
        ach = byts / (kms * 1e-3) / 1e9
        nc = traffic.get(name) or {}
        ncu = {k: nc[k] for k in ("dram_pct", "sm_pct", "warps_active_pct", "warp_inst") if k in nc} or None
        if ncu and nc.get("ms"):
            # instruction-issue roofline: warp instructions per second against
            # 148 SMs x 4 schedulers x 1 warp-instruction per clock at the max SM clock
            ncu["issue_frac"] = nc["warp_inst"] / (nc["ms"] * 1e-3) / (148 * 4 * 1.965e9)
        kernels[name] = {"ms_per_launch": kms / n, "launches": n, "algorithmic_bytes_per_launch": byts / n,
                         "achieved": ach, "frac": ach / peak, "share_of_step": kms / step_ms_total,
                         "traffic": nc.get("dram_bytes_per_launch"), "ncu": ncu}
    dom = max(kernels, key=lambda k: kernels[k]["share_of_step"])
    d = kernels[dom]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": d["achieved"], "peak": peak, "unit": "GB/s",
                "frac": d["frac"], "traffic": d["traffic"], "peak_source": peak_src,
                "issue_frac": (d["ncu"] or {}).get("issue_frac"),
                "algorithmic_bytes_per_launch": d["algorithmic_bytes_per_launch"],
                "ms_per_launch": d["ms_per_launch"], "share_of_step": d["share_of_step"]}
    path_ms = sum(ks[k][0] for k in ks if k != "k_union_linear")
    path = None
    if path_ms > 0:
        ach = packets * ALGO_BYTES_PER_PACKET / (path_ms * 1e-3) / 1e9
        path = {"kernels": [k for k in ks if k != "k_union_linear"], "algorithmic_bytes_per_packet":
                ALGO_BYTES_PER_PACKET, "ms_per_step": path_ms / steps, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak}
    return roofline, kernels, path


# ---------------------------------------------------------------- CPU reference (checker only)

def cpu_reference(sample_recs, cols, threads, slice_id):
    """Time the reference's own DetectPipeline (oracle/_ref = the unmodified
    headers; the C restatement if _ref is absent) on a bounded sample.
    Returns scan rate and end-of-slice ms (report_window + slide)."""
    from oracle.pyoracle import LIBS, Checker, SeaConfig, build
    kind = "reference"
    if not os.path.exists(LIBS["ref"]):
        kind = "port"
        if not os.path.exists(LIBS["orc"]):
            build()
    chk = Checker("ref" if kind == "reference" else "orc")
    pipe = chk.pipeline(SeaConfig(**sketch_cfg(cols)), workers=threads)
    t0 = time.perf_counter()
    pipe.process_slice(slice_id, sample_recs, True)
    total_ms = (time.perf_counter() - t0) * 1e3
    scan_ms = pipe.scan_ms
    return {"kind": kind, "scan_rate": len(sample_recs) / (scan_ms / 1e3), "scan_ms": scan_ms,
            "eos_ms": total_ms - scan_ms, "threads": threads if kind == "reference" else 1}


def sample_records(n, device):
    """First n background packets (plus the plants) of C2 slice 0 — an exact
    prefix of the benchmark's own slice 0 (same generator draws)."""
    import numpy as np
    from paper_1803_10369_b200.srla import DeviceTraceGenerator, PlantSpec
    gen = DeviceTraceGenerator(PlantSpec(**trace_spec(n, slices=1)), device=device)
    return gen.slice_tensor(0).cpu().numpy().view(np.uint32).copy()


def run_reference_arm(args):
    rank, world, local = env_rank()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    samp_n = args.cpu_sample
    recs = sample_records(samp_n, local)
    full = args.packets
    per_step = []
    res = None
    for i in range(args.warmup + args.steps):
        res = cpu_reference(recs, args.cols or (1 << 20), threads, slice_id=9)
        ms_full = full / res["scan_rate"] * 1e3 + res["eos_ms"]
        if i >= args.warmup:
            per_step.append((ms_full, res))
    ms = statistics.mean(p[0] for p in per_step)
    value = full / (ms / 1e3)
    eos = [p[1]["eos_ms"] for p in per_step]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "packets/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "C2: u=4 v=2^20 g=8 g'=1024 z=4 k=10 theta=1024; 1e8 packets/slice",
                   "packets_per_slice": full, "parallelism": "cpu threads"},
        "end_of_slice_ms": {"median": statistics.median(eos), "p99": max(eos)},
        "cpu_baseline": {"value": value, "unit": "packets/s", "cores": res["threads"], "kind": res["kind"],
                         "sample": f"each step: DetectPipeline<u8>::process_slice (workers={res['threads']}) on the "
                                   f"first {len(recs)} packets of C2 slice 0 at v=2^20 with a report due; "
                                   f"value = 1e8 / (1e8 / measured scan rate + measured report+slide time)"},
        "e2e": {"value": value, "unit": "packets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- the engine

def run_engine(args):
    import numpy as np
    import torch

    from paper_1803_10369_b200 import srla

    rank, world, local = env_rank()
    # one process per GPU; SRLA_BENCH_BACKEND=gloo lets several ranks share a
    # GPU to exercise the N > 1 path on a one-GPU box (timings then contend)
    backend = os.environ.get("SRLA_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    comm_dev = torch.device("cuda", local) if backend == "nccl" else torch.device("cpu")
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cols = args.cols if args.cols else (1 << 24 if args.workload == "c3" else 1 << 20)
    cfg = srla.SeaConfig(**sketch_cfg(cols))
    n_per_gpu = args.packets
    spec = trace_spec(n_per_gpu * world, workload=args.workload)
    gen = srla.DeviceTraceGenerator(srla.PlantSpec(**spec), device=local)

    # stage the trace in HBM: one owned slice per generator slice
    nres = min(spec["slices"], args.resident)
    slices = []
    for s in range(nres):
        full = gen.slice_tensor(s)
        if world > 1:
            own = torch.empty_like(full)
            m = srla.partition_records(full.data_ptr(), full.shape[0], cfg.seed, world, rank, own.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream)
            slices.append(own[:m].clone())
            del own
        else:
            slices.append(full)
        del full
    torch.cuda.synchronize()

    eng = srla.EstimatorArray(cfg, device=local)
    st = torch.cuda.ExternalStream(eng.stream_handle())
    rep_cap = 1 << 21

    def pinned_entries(n):  # DMA-able report buffer: the engine maps entries straight into it
        return torch.empty(n * srla.ENTRY_DTYPE.itemsize, dtype=torch.uint8, pin_memory=True).numpy().view(
            srla.ENTRY_DTYPE)

    rep_buf = pinned_entries(rep_cap)

    from paper_1803_10369_b200.shard import allgather_report_entries as _allgather_dev

    def allgather_report(entries):  # merged on the device (N > 1)
        return entries if world == 1 else _allgather_dev(entries, dist, comm_dev)

    def step(sid):
        eng.scan(slices[sid % nres])
        n, nr = _end_slice(eng, sid, rep_buf)
        if world > 1:
            if args.handoff == "compact":  # (host, weight) words + this shard's Eq. 9 table, merged on the device
                from paper_1803_10369_b200.shard import allgather_report_compact
                h = torch.from_numpy(comp_hosts[:n].view(np.int32)).to(comm_dev, non_blocking=True)
                w = torch.from_numpy(comp_w[:n].view(np.int32)).to(comm_dev, non_blocking=True)
                mask = 0xFFFFFFFF
                return allgather_report_compact(h.to(torch.int64) & mask, w.to(torch.int64) & mask,
                                                torch.from_numpy(comp_est).to(comm_dev),
                                                torch.from_numpy(comp_flags).to(comm_dev), dist), n
            return allgather_report(rep_buf[:n]), n
        return None, n

    import ctypes as C

    L = cfg.linear_slots + 1
    comp_hosts = torch.empty(rep_cap * 4, dtype=torch.uint8, pin_memory=True).numpy().view(np.uint32)
    comp_w = torch.empty(rep_cap * 4, dtype=torch.uint8, pin_memory=True).numpy().view(np.uint32)
    comp_est, comp_flags = np.empty(L, np.float64), np.empty(L, np.uint8)

    def _end_slice(e, sid, buf):
        if args.handoff == "compact":  # hosts + weights (8 B/entry) + the window's Eq. 9 table
            n, nr = e.end_slice_compact(sid, comp_hosts, comp_w, comp_est, comp_flags)
            return n, nr
        n, nr = C.c_uint64(), C.c_uint64()
        srla._check(srla._lib.srla_end_slice(e._h, sid, 1, C.c_void_p(buf.ctypes.data), len(buf), C.byref(n),
                                             C.byref(nr)))
        return n.value, nr.value

    # Overlapped pipeline (C2 default): srla_end_slice_async(s) returns at once and
    # srla_scan_batch(s+1) bins its packets (K1) into the second bin set while
    # slice s's end-of-slice still runs, then joins it; the report of slice s is
    # collected with srla_end_slice_wait. Same work per step, pipelined.
    abufs = [pinned_entries(rep_cap) for _ in range(2)] if args.overlap else None
    pend = {"slot": None}

    def collect():
        if pend["slot"] is None:
            return None
        n, _ = eng.end_slice_wait()
        rep = abufs[pend["slot"]][:n]
        pend["slot"] = None
        if world > 1:
            allgather_report(rep)
        return n

    def step_overlapped(sid):
        eng.scan(slices[sid % nres])  # joins the pending end-of-slice after its K1
        n = collect()
        eng.end_slice_async(sid, abufs[sid % 2])
        pend["slot"] = sid % 2
        return n

    sid = 0
    prefill = max(0, cfg.window - 1 - args.warmup)
    for _ in range(prefill + args.warmup):
        if args.overlap:
            step_overlapped(sid)
        else:
            step(sid)
        sid += 1
    if args.overlap:
        collect()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    eng.synchronize()

    eng.timing_reset()
    tm0 = {k: v for k, v in eng.timing().items() if k in ("alloc_ms", "allocs")}  # process-wide counters
    st0 = eng.stats()
    clocks = Clocks(local, args.clock_ms)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(st)
    eos_dev, eos_wall, entries = [], [], []

    def eos_sample(n):
        tm = eng.timing()
        eos_dev.append(tm["last_end_slice_device_ms"])
        eos_wall.append(tm["last_end_slice_wall_ms"])
        entries.append(n)

    for _ in range(args.steps):
        if args.overlap:
            n = step_overlapped(sid)
            if n is not None:
                eos_sample(n)
        else:
            _, n = step(sid)
            eos_sample(n)
        sid += 1
    if args.overlap:
        eos_sample(collect())
    t_end.record(st)
    t_end.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = t_start.elapsed_time(t_end)
    tm = eng.timing()
    st1 = eng.stats()
    pk = torch.tensor([float(st1["packets"] - st0["packets"]), ms], dtype=torch.float64, device=comm_dev)
    if dist:
        tot = pk[:1].clone()
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        mx = pk[1:].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        packets, ms = tot.item(), mx.item()
    else:
        packets = pk[0].item()
    value = packets / (ms / 1e3)

    peak, peak_src = measured_peaks()
    roofline, kernels, path = kernel_rooflines(tm, ms, cfg, peak, peak_src, tm["scan_kernel_records"], args.steps,
                                              args.workload)

    # end to end through the public API with host buffers (pinned), H2D inside:
    # scan_batch(host) + end_slice_async/wait, so a slice's host->device copies
    # overlap the previous slice's end-of-slice work
    e2e = None
    if not args.no_e2e:
        nh = min(2, nres)
        host = [slices[i].cpu().pin_memory().numpy().view(np.uint32) for i in range(nh)]
        h2d = sum(h.nbytes for h in host) / nh
        bufs = [pinned_entries(rep_cap) for _ in range(2)]
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        d2h = 0
        t0 = time.perf_counter()
        pending = None
        for i in range(args.steps):
            eng.scan(host[(sid + i) % nh])
            if pending is not None:
                n, _ = eng.end_slice_wait()
                allgather_report(bufs[pending][:n])
                d2h += n * srla.ENTRY_DTYPE.itemsize
            eng.end_slice_async(sid + i, bufs[i % 2])
            pending = i % 2
        n, _ = eng.end_slice_wait()
        allgather_report(bufs[pending][:n])
        d2h += n * srla.ENTRY_DTYPE.itemsize
        sid += args.steps
        eng.synchronize()
        if dist:
            dist.barrier()
        el = time.perf_counter() - t0
        if dist:
            t = torch.tensor([el], dtype=torch.float64, device=comm_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = t.item()
        e2e = {"value": packets / el, "unit": "packets/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h / args.steps),
               "api": "srla_scan_batch(host, pinned) + srla_end_slice_async/wait"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "c2":
        recs = sample_records(args.cpu_sample, local)
        threads = os.cpu_count() or 1
        r = cpu_reference(recs, cols, threads, slice_id=9)
        ms_full = n_per_gpu / r["scan_rate"] * 1e3 + r["eos_ms"]
        cpu = {"value": n_per_gpu / (ms_full / 1e3), "unit": "packets/s", "cores": r["threads"], "kind": r["kind"],
               "sample": f"DetectPipeline<u8>::process_slice (workers={r['threads']}) on the first {len(recs)} "
                         f"packets of C2 slice 0 at v=2^20 with a report due: scan {r['scan_rate']:.4g} pkt/s, "
                         f"report+slide {r['eos_ms']:.1f} ms; value = 1e8/(1e8/scan rate + report+slide)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "packets/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (reference generator C2 spec, device port)",
            "config": {"workload": WORKLOADS[args.workload],
                       "packets_per_slice_per_gpu": n_per_gpu, "resident_slices": nres,
                       "report_handoff": "srla_end_slice_async/wait: 24-byte srla_entry per entry (pinned), "
                                         "next slice's K1 overlapped" if args.overlap else
                       "srla_end_slice_compact: host+weight per entry and the Eq. 9 table"
                       if args.handoff == "compact" else "srla_end_slice: 24-byte srla_entry per entry",
                       "l2": "inputs larger than L2 (1.2 GB per slice); no flush",
                       "parallelism": f"owner-partitioned x{world}" if world > 1 else "1 GPU"},
            "end_of_slice_ms": {"device_median": statistics.median(eos_dev),
                                "device_p99": sorted(eos_dev)[min(len(eos_dev) - 1, int(0.99 * len(eos_dev)))],
                                "device_max": max(eos_dev), "samples": len(eos_dev),
                                "wall_median": statistics.median(eos_wall), "report_entries_median":
                                    statistics.median(entries)},
            "roofline": roofline,
            "kernels": kernels,
            "roofline_scan_path": path,
            "breakdown_ms_per_step": {k: (tm[k] - tm0.get(k, 0)) / args.steps for k in
                                      ("scan_kernel_ms", "order_wall_ms", "report_wall_ms", "slide_wall_ms",
                                       "sync_wait_ms", "syncs", "alloc_ms", "allocs")},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "overlapped_chunks": int(st1["overlapped_chunks"] - st0["overlapped_chunks"]),
            "gpu_launches": int(st1["kernel_launches"] - st0["kernel_launches"]),
            "library_launches": int(st1["library_launches"] - st0["library_launches"]),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--packets", type=int, default=100_000_000, help="packets per slice per GPU")
    ap.add_argument("--cols", type=int, default=0, help="sketch columns (default: the workload's)")
    ap.add_argument("--workload", default="c2", choices=["c2", "c3"])
    ap.add_argument("--resident", type=int, default=0, help="distinct slices staged in HBM (default 12; c3: 10)")
    ap.add_argument("--cpu-sample", type=int, default=20_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--clock-ms", type=int, default=100, help="nvidia-smi clock sampling period in the timed region")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--overlap", action="store_true",
                    help="pipeline slice s+1's K1 under slice s's asynchronous end-of-slice (SRLA_OVERLAP=1; "
                         "measured slower on C2, kept as an option)")
    ap.add_argument("--handoff", default="compact", choices=["compact", "entries"],
                    help="report hand-off of the device-resident steps (e2e always returns srla_entry)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.overlap:
        os.environ["SRLA_OVERLAP"] = "1"
    if not args.resident:
        args.resident = 10 if args.workload == "c3" else 12
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_engine(args)


if __name__ == "__main__":
    sys.exit(main())
