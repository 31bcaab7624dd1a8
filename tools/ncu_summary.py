"""Fold ncu --set full captures into profiles/ncu_summary.json.

  python tools/ncu_summary.py <workload> <report.ncu-rep> [...]

Per kernel (bench.py's names): DRAM bytes read + written per launch, duration,
DRAM/SM throughput. bench.py reads dram_bytes_per_launch as roofline.traffic."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_table import rows  # noqa: E402

NAMES = [("k_scan_bin", "k_scan_bin"), ("k_split", "k_split"), ("k_slice_apply", "k_slice_apply"),
         ("k_slice_stamp", "k_slice_apply"), ("k_stamp_warp", "k_slice_apply"), ("k_union_linear", "k_union_linear"), ("k_scan<", "k_scan")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TSCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def main(workload, reps):
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_summary.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    out.setdefault("how", "ncu --set full --clock-control none (cold-cache, serialised replay) of one bench.py run "
                          "per workload; dram_bytes_per_launch = dram__bytes_read.sum + dram__bytes_write.sum")
    wl = out.setdefault("workloads", {}).setdefault(workload, {})
    for rep in reps:
        for d, u in rows(rep):
            kname = d["Kernel Name"]
            key = next((k for pat, k in NAMES if pat in kname), None)
            if key is None:
                continue
            b = float(d["dram__bytes_read.sum"]) * SCALE[u["dram__bytes_read.sum"]] + \
                float(d["dram__bytes_write.sum"]) * SCALE[u["dram__bytes_write.sum"]]
            ms = float(d["gpu__time_duration.sum"]) * TSCALE[u["gpu__time_duration.sum"]]
            ent = wl.setdefault(key, {"launches": []})
            ent["launches"].append({"kernel": kname.split("(")[0], "dram_bytes": b, "ms": ms,
                                    "dram_pct": float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]),
                                    "sm_pct": float(d["sm__throughput.avg.pct_of_peak_sustained_elapsed"]),
                                    "warp_inst": float(d["smsp__inst_executed.sum"]),
                                    "warps_active_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"]),
                                    "source": os.path.basename(rep)})
    for ent in wl.values():
        ls = ent["launches"]
        ent["dram_bytes_per_launch"] = sum(x["dram_bytes"] for x in ls) / len(ls)
        for key in ("dram_pct", "sm_pct", "warp_inst", "warps_active_pct", "ms"):
            ent[key] = sum(x[key] for x in ls) / len(ls)
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps({k: v["dram_bytes_per_launch"] for k, v in wl.items()}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
