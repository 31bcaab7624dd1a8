O=gpurun_out/r2src; mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
for k in k_scan_bin "^k_split$"; do
  f=$O/src_c2_${k//[^a-z_]/}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -o $f $B > $f.log 2>&1
  ncu -i $f.ncu-rep --page source --csv --print-source cuda > $f.cuda.csv 2>$f.err
  rm -f $f.ncu-rep
done
ls -la $O
