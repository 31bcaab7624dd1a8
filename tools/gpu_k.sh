mkdir -p gpurun_out/ncu /tmp/ncu
SRLA_STAMP_CELLS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_stamp_cells -s 3 -c 1 -o /tmp/ncu/cells python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu cells rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_scan_bin -s 5 -c 1 -o /tmp/ncu/k1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c3 > /dev/null 2>&1; echo "ncu k1 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_split -s 5 -c 1 -o /tmp/ncu/split python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c3 > /dev/null 2>&1; echo "ncu split rc=$?"
for k in cells k1 split; do
  ncu -i /tmp/ncu/$k.ncu-rep --page details --csv > gpurun_out/ncu/r2k_${k}_details.csv 2>/dev/null
  ncu -i /tmp/ncu/$k.ncu-rep --page raw --csv > gpurun_out/ncu/r2k_${k}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/$k.ncu-rep --page source --csv --print-source cuda > gpurun_out/ncu/r2k_${k}_source.csv 2>/dev/null
done
ls -la gpurun_out/ncu; du -sh gpurun_out
