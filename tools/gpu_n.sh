B="--steps 20 --warmup 3 --no-c3 --no-cpu-baseline --no-e2e"
for r in 8 16; do for w in 4 8; do for o in fast legacy; do
  SRLA_REGION_MB=$r SRLA_SPLIT_WAVES=$w SRLA_ORDER=$o timeout 300 python bench.py $B > gpurun_out/r2n_r${r}_w${w}_$o.jsonl 2>&1
done; done; done
python tools/show.py gpurun_out/r2n_*.jsonl | grep pkt
