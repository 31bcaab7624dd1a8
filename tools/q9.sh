O=gpurun_out/q9; mkdir -p $O
bash tools/quick.sh q9
SRLA_FINE_KB=64 timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_fine64.jsonl 2>&1
SRLA_FINE_KB=16 timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_fine16.jsonl 2>&1
