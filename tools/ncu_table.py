"""Print key ncu --set full metrics per captured launch (reads an .ncu-rep)."""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "smsp__inst_executed.sum",
        "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum"]


def rows(rep):
    """rep: an .ncu-rep, or its `--page raw --csv` export (.raw.csv)."""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for x in r[2:]:
        d = dict(zip(hdr, x))
        yield d, dict(zip(hdr, units))


if __name__ == "__main__":
    for d, u in rows(sys.argv[1]):
        print(d["Kernel Name"][:60])
        for w in WANT:
            if w in d:
                print(f"   {w:60s} {d[w]:>16s} {u.get(w, '')}")
