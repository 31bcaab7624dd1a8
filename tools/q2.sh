O=gpurun_out/q2; mkdir -p $O
free -g > $O/free.txt
bash tools/quick.sh q2
SRLA_SPARSE_MAX=0 timeout 900 python bench.py --workload c3 --no-cpu-baseline --no-e2e > $O/bench_c3_dense.jsonl 2>&1
