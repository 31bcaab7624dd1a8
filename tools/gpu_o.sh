B="--steps 20 --warmup 3 --no-c3 --no-cpu-baseline --no-e2e"
for r in 4 8; do for w in 8 16 32; do
  SRLA_REGION_MB=$r SRLA_SPLIT_WAVES=$w timeout 300 python bench.py $B > gpurun_out/r2o_r${r}_w${w}.jsonl 2>&1
done; done
SRLA_REGION_MB=8 SRLA_SPLIT_WAVES=8 timeout 300 python bench.py --workload c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2o_c3_r8_w8.jsonl 2>&1
timeout 300 python bench.py --workload c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2o_c3_default.jsonl 2>&1
python tools/show.py gpurun_out/r2o_*.jsonl | grep pkt
