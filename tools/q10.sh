O=gpurun_out/q10; mkdir -p $O
SRLA_EOS_TRACE=1 timeout 900 python bench.py --workload c3 --no-cpu-baseline --no-e2e --steps 8 > $O/c3_trace.jsonl 2> $O/c3_trace.err
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline > $O/bench_$i.jsonl 2>&1; done
