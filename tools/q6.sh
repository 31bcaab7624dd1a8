O=gpurun_out/q6; mkdir -p $O
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/bench1.jsonl 2> $O/bench1.err
SRLA_TRACE=1 timeout 600 python bench.py --steps 6 --no-e2e --no-cpu-baseline > $O/trace_c2.jsonl 2> $O/trace_c2.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/bench2.jsonl 2> $O/bench2.err
