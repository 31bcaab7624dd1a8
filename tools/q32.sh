O=gpurun_out/q32; mkdir -p $O
for w in 1 2 8; do SRLA_SPLIT_WAVES=$w timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/bench_w$w.jsonl 2>&1; done
SRLA_EARLY_SPLIT=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/bench_off.jsonl 2>&1
