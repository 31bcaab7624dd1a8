O=gpurun_out/q5; mkdir -p $O
bash tools/quick.sh q5
for sm in 1024 100000; do
SRLA_SPARSE_MAX=$sm timeout 900 python bench.py --workload c3 --no-cpu-baseline --no-e2e --steps 10 > $O/bench_c3_sparse$sm.jsonl 2>&1
done
