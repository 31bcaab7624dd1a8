O=gpurun_out/q29; mkdir -p $O
for w in 3 6 8; do SRLA_APPLY_WAVES=$w timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 > $O/bench_w$w.jsonl 2>&1; done
