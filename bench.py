#!/usr/bin/env python
"""SRLA benchmark: packets/s scanned + end-of-slice latency (BASELINE.json).

Headline workload (BASELINE.json configs[1], "C2" in SURVEY.md §8d): one B200
per rank, sketch u=4, v=2^20, g=8, g'=1024, z=4 (u8 recorders), k=10,
theta=1024, seed 0x5EA00001; synthetic trace = the reference generator's C2
spec (uniform 4M sources, Zipf(1.0) 4M destinations, 50 planted super points),
1e8 packets per slice per GPU, produced byte-identically on the device and
resident in HBM (1.2 GB per slice, > L2, so no flush is needed between steps).

A step = DetectPipeline::process_slice on one slice: scan (K1..K5) + report
(when the window is full) + slide. The line also carries a `c3` record
(configs[2]: v=2^24, ~1e6 candidates): the end-of-slice latency target.

N > 1 (weak scaling, configs[3]'s shape): hosts are owner-partitioned
(reduce(3, aip, N)); every rank keeps an independent sketch for its hosts and
the per-slice report is all-gathered (the only collective). `--gpus N` without
a torchrun environment launches the N ranks itself; with fewer GPUs than
ranks they share GPUs over gloo (functional, contended timings).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1803_10369_b200 import workloads as WL  # noqa: E402  (data only: no CUDA)

METRIC = "packets/sec scanned (1/2/4/8 B200); end-of-slice estimation latency ms"
ALGO_BYTES_PER_PACKET = 140  # 12 B streamed record + 4 rows x one 32-B sector update


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def random_access_peak():
    """BASELINE.md §3's HBM random-access roofline R: random 1-byte stores
    into a 4 GiB table, counted at one 32-B sector each (tools/membench.cu,
    profiles/r01_membench.json)."""
    p = os.path.join(ROOT, "profiles", "r01_membench.json")
    if not os.path.exists(p):
        return None
    return json.load(open(p))["st8_4096MB_Gops"] * 32.0


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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
    if tm.get("serial_kernel_launches"):
        kernels["k_serial"] = {"ms_per_launch": tm["serial_kernel_ms"] / tm["serial_kernel_launches"],
                               "launches": tm["serial_kernel_launches"],
                               "share_of_step": tm["serial_kernel_ms"] / step_ms_total,
                               "flagged_hosts": tm["flagged_hosts"]}
    dom = max((k for k in kernels if "achieved" in kernels[k]), key=lambda k: kernels[k]["share_of_step"])
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

def reference_checker():
    """oracle/_ref (the unmodified reference headers) when present, else the C restatement."""
    from oracle.pyoracle import LIBS, Checker, build
    if os.path.exists(LIBS["ref"]):
        return Checker("ref"), "reference"
    if not os.path.exists(LIBS["orc"]):
        build()
    return Checker("orc"), "port"


def reference_steady(chk, cols, slices, threads, prefill, warmup, steps):
    """The reference's own DetectPipeline<u8> (workers = threads) over full
    slices: `prefill` slices to fill the window, then warmup + timed steps of
    process_slice (scan + report_window + slide), cycling over `slices`."""
    from oracle.pyoracle import SeaConfig
    pipe = chk.pipeline(SeaConfig(**WL.sketch_cfg(cols)), workers=threads)
    sid = 0
    for _ in range(prefill + warmup):
        pipe.process_slice(sid, slices[sid % len(slices)], True)
        sid += 1
    per, eos, packets, cands = [], [], 0, []
    for _ in range(steps):
        recs = slices[sid % len(slices)]
        s0 = pipe.scan_ms
        t0 = time.perf_counter()
        rep = pipe.process_slice(sid, recs, True)
        ms = (time.perf_counter() - t0) * 1e3
        per.append(ms)
        eos.append(ms - (pipe.scan_ms - s0))
        packets += len(recs)
        cands.append(0 if rep is None else len(rep["host"]))
        sid += 1
    total = sum(per)
    return {"value": packets / (total / 1e3), "ms_per_step": total / steps, "eos_median": statistics.median(eos),
            "eos_p99": max(eos), "report_entries_median": statistics.median(cands), "packets": packets}


def run_reference_arm(args):
    """--impl reference: the reference's CPU implementation of the path on
    this box's host cores, same workload / metric / steps as the engine arm.
    Input = the reference generator's own slices (ref_generate_slice)."""
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    from oracle.pyoracle import PlantSpec
    chk, kind = reference_checker()
    threads = os.cpu_count() or 1
    spec = WL.trace_spec(args.packets, slices=args.resident, workload="c2")
    t0 = time.perf_counter()
    if kind == "reference":
        slices = [chk.generate_slice(PlantSpec(**spec), s, threads) for s in range(args.resident)]
    else:
        whole = chk.generate(PlantSpec(**spec))
        n0 = len(whole) // args.resident
        slices = [whole[i * n0:(i + 1) * n0] for i in range(args.resident)]
    gen_s = time.perf_counter() - t0
    prefill = 9
    r = reference_steady(chk, 1 << 20, slices, threads, prefill, args.warmup, args.steps)
    n = max(1, world) if world > 1 else args.gpus
    sample = (f"each step: DetectPipeline<u8>::process_slice (workers={threads}, unpinned) on one full "
              f"{args.packets:.0e}-packet C2 slice at steady state ({prefill} prefill + {args.warmup} warmup slices, "
              f"~{r['report_entries_median']:.0f} candidates per report); slices from ref_generate_slice "
              f"({gen_s:.0f} s, not timed); CPU {cpu_model()}, {threads} logical cores")
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": "packets/s", "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic (reference generator C2 spec)",
        "config": {"workload": WL.DESCRIPTIONS["c2"], "packets_per_slice": args.packets,
                   "resident_slices": args.resident, "parallelism": f"{threads} CPU threads (rank 0 only)"},
        "same_config": kind == "reference",
        "end_of_slice_ms": {"median": r["eos_median"], "p99": r["eos_p99"]},
        "cpu_baseline": {"value": r["value"], "unit": "packets/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": r["value"], "unit": "packets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- the engine

class Workload:
    """Slices staged in HBM + an engine for one workload on this rank."""

    def __init__(self, name, args, rank, world, local):
        import torch

        from paper_1803_10369_b200 import srla
        self.name, self.srla = name, srla
        cols = args.cols if args.cols else WL.cols_of(name)
        self.cfg = srla.SeaConfig(**WL.sketch_cfg(cols))
        self.spec = WL.trace_spec(args.packets * world, slices=12, workload=name)
        gen = srla.DeviceTraceGenerator(srla.PlantSpec(**self.spec), device=local)
        self.nres = min(self.spec["slices"], args.resident if name == "c2" else 10)
        self.slices = []
        for s in range(self.nres):
            full = gen.slice_tensor(s)
            if world > 1:
                own = torch.empty_like(full)
                m = srla.partition_records(full.data_ptr(), full.shape[0], self.cfg.seed, world, rank,
                                           own.data_ptr(), torch.cuda.current_stream().cuda_stream)
                self.slices.append(own[:m].clone())
                del own
            else:
                self.slices.append(full)
            del full
        torch.cuda.synchronize()
        self.eng = srla.EstimatorArray(self.cfg, device=local)
        self.rep_cap = 1 << 21
        self.L = self.cfg.linear_slots + 1


def run_engine(args):
    import ctypes as C

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

    w = Workload(args.workload, args, rank, world, local)
    eng, cfg, slices, nres = w.eng, w.cfg, w.slices, w.nres
    shard = None
    if world > 1:
        # the C ABI's sharded pipeline: the rank's engine + the report
        # all-gather merged by host on the device (srla_shard_*), over the
        # library's NCCL communicator (or gloo when ranks share a GPU)
        from paper_1803_10369_b200.shard import OWNED, EngineShard, GlooTransport, NcclTransport
        del w.eng, eng
        transport = NcclTransport(dist, local) if backend == "nccl" else GlooTransport(dist)
        shard = EngineShard(cfg, transport, device=local)
        shard.reserve(w.rep_cap * world)
        eng = shard.engine
    st = torch.cuda.ExternalStream(eng.stream_handle())

    def pinned(nbytes):
        return torch.empty(nbytes, dtype=torch.uint8, pin_memory=True).numpy()

    def pinned_entries(n):  # DMA-able report buffer: the engine maps entries straight into it
        return pinned(n * srla.ENTRY_DTYPE.itemsize).view(srla.ENTRY_DTYPE)

    comp_hosts = pinned(w.rep_cap * 4).view(np.uint32)
    comp_w = pinned(w.rep_cap * 4).view(np.uint32)
    comp_est, comp_flags = np.empty(w.L, np.float64), np.empty(w.L, np.uint8)
    rep_buf = pinned_entries(w.rep_cap)

    def end_slice(sid):
        if args.handoff == "compact":  # hosts + weights (8 B/entry) + the window's Eq. 9 table
            return eng.end_slice_compact(sid, comp_hosts, comp_w, comp_est, comp_flags)
        n, nr = C.c_uint64(), C.c_uint64()
        srla._check(srla._lib.srla_end_slice(eng._h, sid, 1, C.c_void_p(rep_buf.ctypes.data), len(rep_buf),
                                             C.byref(n), C.byref(nr)))
        return n.value, nr.value

    def step(sid):
        if shard is not None:  # scan + end-of-slice + merged report, one collective call
            rep, _ = shard.process_slice(sid, slices[sid % nres], mode=OWNED)
            return 0 if rep is None else len(rep)
        eng.scan(slices[sid % nres])
        n, _ = end_slice(sid)
        return n

    sid = 0
    prefill = max(0, cfg.window - 1 - args.warmup)
    for _ in range(prefill + args.warmup):
        step(sid)
        sid += 1
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
    for _ in range(args.steps):
        n = step(sid)
        tm = eng.timing()
        eos_dev.append(tm["last_end_slice_device_ms"])
        eos_wall.append(tm["last_end_slice_wall_ms"])
        entries.append(n)
        sid += 1
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
    R = random_access_peak()
    rand = None
    if R:
        ach = value / max(1, world) * ALGO_BYTES_PER_PACKET / 1e9
        rand = {"R": R, "unit": "GB/s", "achieved_per_gpu": ach, "frac": ach / R,
                "definition": "packets/s per GPU x 140 B (12 B record + 4 random 32-B sector updates) over R = "
                              "measured random 1-byte stores into a 4 GiB table x 32 B (tools/membench.cu, "
                              "profiles/r01_membench.json); > 1 because the engine bins the marks and streams "
                              "the table instead of updating sectors at random"}

    # end to end through the public API with host buffers (pinned), H2D inside:
    # scan_batch(host) + end_slice_async/wait, so a slice's host->device copies
    # overlap the previous slice's end-of-slice work
    e2e = None
    if not args.no_e2e:
        nh = min(2, nres)
        host = [slices[i].cpu().pin_memory().numpy().view(np.uint32) for i in range(nh)]
        h2d = sum(h.nbytes for h in host) / nh
        bufs = [pinned_entries(w.rep_cap) for _ in range(2)]
        # untimed warm-up steps through the same path (the host staging buffers
        # and the first slices' allocations happen here, not in the timed region)
        for i in range(args.warmup):
            if shard is not None:
                shard.process_slice(sid + i, host[(sid + i) % nh], mode=OWNED)
            else:
                eng.scan(host[(sid + i) % nh])
                eng.end_slice_async(sid + i, bufs[0])
                eng.end_slice_wait()
        sid += args.warmup
        eng.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        d2h = 0
        t0 = time.perf_counter()
        if shard is not None:  # srla_shard_process_slice with host records: H2D, scan, merged report D2H
            for i in range(args.steps):
                rep, _ = shard.process_slice(sid + i, host[(sid + i) % nh], mode=OWNED)
                d2h += 0 if rep is None else rep.nbytes
        else:
            pending = None
            for i in range(args.steps):
                eng.scan(host[(sid + i) % nh])
                if pending is not None:
                    n, _ = eng.end_slice_wait()
                    d2h += n * srla.ENTRY_DTYPE.itemsize
                eng.end_slice_async(sid + i, bufs[i % 2])
                pending = i % 2
            n, _ = eng.end_slice_wait()
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
               "api": "srla_shard_process_slice(host records)" if shard is not None else
               "srla_scan_batch(host, pinned) + srla_end_slice_async/wait"}
        # the ceiling of this path: plain pinned host->device copies of the same
        # slice on this box (best of 3), against the copies inside the e2e loop
        src = torch.from_numpy(host[0].reshape(-1).view(np.uint8))
        dst = torch.empty(src.numel(), dtype=torch.uint8, device=torch.device("cuda", local))
        best = 0.0
        for _ in range(3):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            best = max(best, src.numel() / (time.perf_counter() - t1) / 1e9)
        del dst
        achieved = h2d * args.steps / el / 1e9  # this rank's copies (each rank moves its own slices)
        e2e["h2d"] = {"achieved_gbs_per_gpu": achieved, "pinned_copy_peak_gbs": best, "frac": achieved / best,
                      "definition": "e2e H2D bytes / e2e time, over plain pinned H2D copies of one slice (best of 3)"}
        del host

    # the reference's own entry point through the drop-in headers (C++):
    # DetectPipeline<uint8_t>::process_slice with host records, in its own process
    e2e_dropin = None
    dropin = os.path.join(ROOT, "paper_1803_10369_b200", "lib", "bench_dropin")
    if rank == 0 and world == 1 and not args.no_e2e and args.workload == "c2" and os.path.exists(dropin):
        try:
            r = subprocess.run([dropin, str(args.steps), str(args.warmup), str(args.packets)], capture_output=True,
                               text=True, timeout=900)
            e2e_dropin = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else \
                {"error": (r.stderr or r.stdout)[-300:]}
        except Exception as ex:  # noqa: BLE001 (reported, not fatal)
            e2e_dropin = {"error": str(ex)[:300]}

    # the reference on this box's host cores, steady state on the same slices
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "c2":
        chk, kind = reference_checker()
        threads = os.cpu_count() or 1
        host = [s.cpu().numpy().view(np.uint32) for s in slices]
        r = reference_steady(chk, cfg.cols, host, threads, prefill=9, warmup=0, steps=args.cpu_steps)
        cpu = {"value": r["value"], "unit": "packets/s", "cores": threads, "kind": kind,
               "sample": f"DetectPipeline<u8>::process_slice (workers={threads}, unpinned; {cpu_model()}) on "
                         f"{args.cpu_steps} full C2 slices at steady state after a 9-slice prefill "
                         f"(~{r['report_entries_median']:.0f} candidates per report), end-of-slice "
                         f"{r['eos_median']:.0f} ms median"}
        del host

    del slices, w.slices
    torch.cuda.empty_cache()
    c3 = None
    if world == 1 and args.workload == "c2" and not args.no_c3:
        del eng, w
        torch.cuda.empty_cache()
        c3 = run_c3(args, local, peak, peak_src)
    if shard is not None:
        shard.close()
        transport.close() if hasattr(transport, "close") else None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "packets/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (reference generator spec, device port)",
            "config": {"workload": WL.DESCRIPTIONS[args.workload],
                       "packets_per_slice_per_gpu": args.packets, "resident_slices": nres,
                       "report_handoff": "srla_end_slice_compact: host+weight per entry and the Eq. 9 table"
                       if args.handoff == "compact" else "srla_end_slice: 24-byte srla_entry per entry",
                       "l2": "inputs larger than L2 (1.2 GB per slice); no flush",
                       "parallelism": f"owner-partitioned x{world}: srla_shard_* (records arrive owner-sharded; "
                                      f"report all-gather over {'NCCL' if backend == 'nccl' else 'gloo, ranks sharing a GPU'})"
                       if world > 1 else "1 GPU"},
            "end_of_slice_ms": {"device_median": statistics.median(eos_dev),
                                "device_p99": sorted(eos_dev)[min(len(eos_dev) - 1, int(0.99 * len(eos_dev)))],
                                "device_max": max(eos_dev), "samples": len(eos_dev),
                                "wall_median": statistics.median(eos_wall), "report_entries_median":
                                    statistics.median(entries)},
            "roofline": roofline,
            "kernels": kernels,
            "roofline_scan_path": path,
            "random_access_roofline": rand,
            "breakdown_ms_per_step": {k: (tm[k] - tm0.get(k, 0)) / args.steps for k in
                                      ("scan_kernel_ms", "order_wall_ms", "report_wall_ms", "slide_wall_ms",
                                       "sync_wait_ms", "syncs", "alloc_ms", "allocs", "serial_kernel_ms")},
            "flagged_hosts_per_step": tm["flagged_hosts"] / args.steps,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_dropin": e2e_dropin,
            "c3": c3,
            "gpu_launches": int(st1["kernel_launches"] - st0["kernel_launches"]),
            "library_launches": int(st1["library_launches"] - st0["library_launches"]),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def run_c3(args, local, peak, peak_src):
    """configs[2] (v = 2^24, ~1e6 candidates): the end-of-slice latency target.
    k - 1 prefill slices, W warm-up steps, then K timed process_slice steps."""
    import numpy as np
    import torch

    class A:  # the C3 slice shape at the same packets per slice
        packets, cols, resident = args.packets, 0, 10

    w = Workload("c3", A, 0, 1, local)
    eng, cfg = w.eng, w.cfg
    st = torch.cuda.ExternalStream(eng.stream_handle())
    hosts = torch.empty(w.rep_cap * 4, dtype=torch.uint8, pin_memory=True).numpy().view(np.uint32)
    wts = torch.empty(w.rep_cap * 4, dtype=torch.uint8, pin_memory=True).numpy().view(np.uint32)
    est, flags = np.empty(w.L, np.float64), np.empty(w.L, np.uint8)
    sid = 0
    for _ in range(cfg.window - 1 + args.warmup):
        eng.scan(w.slices[sid % w.nres])
        eng.end_slice_compact(sid, hosts, wts, est, flags)
        sid += 1
    eng.synchronize()
    eng.timing_reset()
    st0 = eng.stats()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(st)
    eos_dev, eos_wall, entries = [], [], []
    for _ in range(args.steps):
        eng.scan(w.slices[sid % w.nres])
        n, _ = eng.end_slice_compact(sid, hosts, wts, est, flags)
        tm = eng.timing()
        eos_dev.append(tm["last_end_slice_device_ms"])
        eos_wall.append(tm["last_end_slice_wall_ms"])
        entries.append(n)
        sid += 1
    t1.record(st)
    t1.synchronize()
    ms = t0.elapsed_time(t1)
    tm, st1 = eng.timing(), eng.stats()
    packets = st1["packets"] - st0["packets"]
    roofline, kernels, path = kernel_rooflines(tm, ms, cfg, peak, peak_src, tm["scan_kernel_records"], args.steps,
                                              "c3")
    q = sorted(eos_dev)
    out = {"workload": WL.DESCRIPTIONS["c3"], "value": packets / (ms / 1e3), "unit": "packets/s",
           "ms_per_step": ms / args.steps,
           "end_of_slice_ms": {"device_median": statistics.median(eos_dev),
                               "device_p99": q[min(len(q) - 1, int(0.99 * len(q)))], "device_max": q[-1],
                               "wall_median": statistics.median(eos_wall), "samples": len(q),
                               "target_ms": 1.0},
           "report_entries_median": statistics.median(entries), "roofline": roofline, "kernels": kernels,
           "flagged_hosts_per_step": tm["flagged_hosts"] / args.steps,
           "gpu_launches": int(st1["kernel_launches"] - st0["kernel_launches"])}
    del eng, w
    torch.cuda.empty_cache()
    return out


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args):
    """`--gpus N` outside torchrun: launch N ranks (one process per GPU) the
    way the driver does; ranks share GPUs over gloo when fewer are present."""
    env = dict(os.environ)
    try:
        import torch
        ndev = torch.cuda.device_count()
    except Exception:
        ndev = 0
    if ndev < args.gpus:
        env["SRLA_BENCH_BACKEND"] = "gloo"
        print(f"[bench] {args.gpus} ranks on {ndev} GPU(s): ranks share GPUs over gloo", file=sys.stderr)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--packets", type=int, default=WL.PAIRS, help="packets per slice per GPU")
    ap.add_argument("--cols", type=int, default=0, help="sketch columns (default: the workload's)")
    ap.add_argument("--workload", default="c2", choices=["c2", "c3", "c5"])
    ap.add_argument("--resident", type=int, default=12, help="distinct slices staged in HBM")
    ap.add_argument("--cpu-steps", type=int, default=2, help="timed steady-state slices of the cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 end-of-slice record")
    ap.add_argument("--clock-ms", type=int, default=100, help="nvidia-smi clock sampling period in the timed region")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--handoff", default="compact", choices=["compact", "entries"],
                    help="report hand-off of the device-resident steps (e2e always returns srla_entry)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    return run_engine(args)


if __name__ == "__main__":
    sys.exit(main())
