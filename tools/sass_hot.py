"""Hot spots of a per-SASS ncu source export (.sass.csv[.gz]): executed
instructions and stall samples by address window, plus the top instructions."""
import csv
import gzip
import sys


def load(path):
    f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    rows = list(csv.reader(f))
    hdr = rows[1]
    data = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break
        if len(r) >= len(hdr):
            data.append(r)
    return hdr, data


def main(path, win=50, top=30):
    hdr, data = load(path)
    iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[iE]) for r in data) or 1
    totw = sum(int(r[iW]) for r in data) or 1
    print(f"{len(data)} SASS, {tot} warp-instr, {totw} samples")
    for k in range(0, len(data), win):
        seg = data[k:k + win]
        e = sum(int(r[iE]) for r in seg) / tot
        w = sum(int(r[iW]) for r in seg) / totw
        if e > 0.01 or w > 0.01:
            print(f"{k:5d} exec {e:.3f} stall {w:.3f}  {seg[0][iS][:50]}")
    print("top stalls:")
    for i in sorted(sorted(range(len(data)), key=lambda i: -int(data[i][iW]))[:top]):
        print(f"{i:5d} {int(data[i][iE]):>11d} {int(data[i][iW]) / totw:.3f} {data[i][iS][:70]}")


if __name__ == "__main__":
    main(sys.argv[1], *(int(x) for x in sys.argv[2:]))
