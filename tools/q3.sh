O=gpurun_out/q3; mkdir -p $O
SRLA_TRACE=1 timeout 600 python bench.py --steps 4 --no-e2e --no-cpu-baseline > $O/trace_c2.jsonl 2> $O/trace_c2.err
timeout 600 python bench.py --no-cpu-baseline > $O/bench.jsonl 2> $O/bench.err
SRLA_EPOCH=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_c2_epoch.jsonl 2> $O/bench_c2_epoch.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_split|k_slice_stamp|k_scan_bin' -s 12 -c 3 \
   -o $O/prof_c3scan python bench.py --workload c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/prof_c3scan.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_split|k_scan_bin' -s 6 -c 2 \
   -o $O/prof_c2scan python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/prof_c2scan.log 2>&1
