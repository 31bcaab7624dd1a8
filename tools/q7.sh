O=gpurun_out/q7; mkdir -p $O
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c100_$i.jsonl 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 --clock-ms 1000 > $O/bench_c1000_$i.jsonl 2>&1
done
