O=gpurun_out/q16; mkdir -p $O
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench.jsonl 2>&1
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
for k in k_slice_apply_nib k_union_linear_nib k_scan_bin; do
  f=$O/full_c2_$k
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o $f $B > $f.log 2>&1
  ncu -i $f.ncu-rep --page raw --csv > $f.raw.csv 2>/dev/null
  ncu -i $f.ncu-rep --page source --csv --print-source sass > $f.sass.csv 2>/dev/null; gzip -f $f.sass.csv; rm -f $f.ncu-rep
done
