"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v = float(d["Metric Value"].replace(",", ""))
            u = d["Metric Unit"]
            us = v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v
            out.append((int(d["ID"]), d["Kernel Name"].split("(")[0].replace("void ", "")[:70], us))
    return out


def main(path, first=None, last=None):
    data = load(path)
    if first is not None:
        data = [d for d in data if first <= d[0] <= last]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for _, n, us in data:
        agg[n][0] += 1
        agg[n][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':70s} {'n':>5s} {'total ms':>9s} {'avg us':>9s} share")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:70s} {v[0]:5d} {v[1] / 1e3:9.3f} {v[1] / v[0]:9.1f} {v[1] / tot:.3f}")
    print(f"total {tot / 1e3:.3f} ms over {len(data)} launches")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], *(int(x) for x in a[1:3])) if len(a) >= 3 else main(a[0])
