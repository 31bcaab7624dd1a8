O=gpurun_out/q25; mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --workload c3"
for k in k_slice_stamp; do
  f=$O/full_c3_$k
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o $f $B > $f.log 2>&1
  ncu -i $f.ncu-rep --page raw --csv > $f.raw.csv 2>/dev/null
  ncu -i $f.ncu-rep --page source --csv --print-source sass > $f.sass.csv 2>/dev/null; gzip -f $f.sass.csv; rm -f $f.ncu-rep
done
