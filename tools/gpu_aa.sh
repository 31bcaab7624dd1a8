B="--steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 python bench.py $B --no-c3 > gpurun_out/r2aa_c2.jsonl 2>&1; python tools/show.py gpurun_out/r2aa_c2.jsonl | head -4
timeout 300 python bench.py --workload c3 $B > gpurun_out/r2aa_c3.jsonl 2>&1; python tools/show.py gpurun_out/r2aa_c3.jsonl | head -4
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_parity_gpu.py -q -x 2>&1 | tail -2
