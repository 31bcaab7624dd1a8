O=gpurun_out/q20; mkdir -p $O
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_gate.jsonl 2>&1
SRLA_K1_EARLY=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench_early.jsonl 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --overlap off > $O/bench_off.jsonl 2>&1
