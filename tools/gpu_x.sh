O=gpurun_out/r02c; mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-c3"
for w in c2 c3; do
  f=$O/full_${w}_k_split
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_split$' -s 4 -c 1 -o $f $B --workload $w > $f.log 2>&1
  ncu -i $f.ncu-rep --page raw --csv > $f.raw.csv 2>/dev/null
  ncu -i $f.ncu-rep --page source --csv --print-source sass > $f.sass.csv 2>/dev/null; gzip -f $f.sass.csv; rm -f $f.ncu-rep
done
SRLA_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench_n2_gloo.jsonl 2> $O/bench_n2_gloo.err
timeout 600 python -m pytest tests/test_multi_engine_gpu.py tests/test_parity_gpu.py -q -k "shards or contract or nccl" 2>&1 | tail -3
ls -la $O
