O=gpurun_out/c3a; mkdir -p $O
SRLA_TRACE=1 timeout 600 python bench.py --workload c3 --steps 4 --no-e2e --no-cpu-baseline > $O/trace.jsonl 2> $O/trace.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python bench.py --workload c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_union_linear_epoch|k_retain|k_cset_insert|k_sweep|k_age' -s 20 -c 6 \
   -o $O/prof_eos python bench.py --workload c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/prof_eos.log 2>&1
ls -la $O
