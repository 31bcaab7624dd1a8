"""Summarise bench JSON lines: value, step, EOS, per-kernel shares."""
import json
import sys

for f in sys.argv[1:]:
    for l in open(f):
        if not l.startswith("{"):
            continue
        d = json.loads(l)
        if "value" not in d:
            print(f, d)
            continue
        e = d.get("end_of_slice_ms", {})
        print(f"{f}: {d['value']:.4g} pkt/s  {d['ms_per_step']:.3f} ms/step  EOS med {e.get('device_median', e.get('median', 0)):.3f} p99 {e.get('device_p99', e.get('p99', 0)):.3f}"
              f"  e2e {d['e2e']['value'] if d.get('e2e') else None}")
        for k, v in (d.get("kernels") or {}).items():
            print(f"    {k:16s} {v['ms_per_launch']:.3f} ms x{v['launches']}  frac {v.get('frac', 0):.3f} share {v['share_of_step']:.3f}")
        if d.get("breakdown_ms_per_step"):
            print("    breakdown", {k: round(v, 3) for k, v in d["breakdown_ms_per_step"].items()})
