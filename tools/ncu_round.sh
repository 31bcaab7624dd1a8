#!/bin/bash
# ncu evidence for the current build: launch lists + one --set full capture per hot kernel.
# Reports are exported to CSV on the box (raw page + per-SASS source page) and the
# .ncu-rep files dropped unless KEEP_REP=1 (gpurun brings back <= 64 MiB).
# Usage: tools/ncu_round.sh tag [c2|c3|both]
O=gpurun_out/$1; mkdir -p $O
W=${2:-both}
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
cap() {  # workload kernel
  local f=$O/full_$1_${2//[^a-z_]/}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 4 -c 1 -o $f $B --workload $1 > $f.log 2>&1
  ncu -i $f.ncu-rep --page raw --csv > $f.raw.csv 2>/dev/null
  ncu -i $f.ncu-rep --page source --csv --print-source sass > $f.sass.csv 2>/dev/null
  gzip -f $f.sass.csv
  [ "$KEEP_REP" = "1" ] || rm -f $f.ncu-rep
}
if [ "$W" != "c3" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv $B > $O/launches_c2.log 2>&1
  for k in k_scan_bin "^k_split$" k_slice_apply_nib k_union_linear_nib; do cap c2 "$k"; done
fi
if [ "$W" != "c2" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv $B --workload c3 > $O/launches_c3.log 2>&1
  for k in k_scan_bin "^k_split$" k_stamp_warp k_union_linear_epoch; do cap c3 "$k"; done
fi
ls -la $O
