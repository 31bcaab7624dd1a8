O=gpurun_out/q8; mkdir -p $O
for i in 1 2 3 4; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 > $O/bench_$i.jsonl 2>&1
done
