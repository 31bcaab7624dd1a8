O=gpurun_out/q4; mkdir -p $O
bash tools/quick.sh q4
SRLA_TRACE=1 timeout 600 python bench.py --steps 3 --no-e2e --no-cpu-baseline > $O/trace_c2.jsonl 2> $O/trace_c2.err
