B="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for r in 16 32 64; do SRLA_REGION_MB=$r timeout 300 python bench.py --workload c3 $B > gpurun_out/r2r_c3_r$r.jsonl 2>&1; done
timeout 300 python bench.py $B --no-c3 > gpurun_out/r2r_c2.jsonl 2>&1
python tools/show.py gpurun_out/r2r_*.jsonl
timeout 600 python -m pytest tests/test_fullsize_parity_gpu.py tests/test_parity_gpu.py -q -x -k "fullsize or binned or epoch" 2>&1 | tail -3
