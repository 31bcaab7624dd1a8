B="--steps 20 --warmup 3 --no-c3 --no-cpu-baseline --no-e2e"
timeout 120 python -m pytest tests/test_parity_gpu.py -q -x -k "binned and contended" 2>&1 | tail -2
for v in 1 0 1; do SRLA_FUSED=$v timeout 200 python bench.py $B > gpurun_out/r2t_fused$v.jsonl 2>&1; python tools/show.py gpurun_out/r2t_fused$v.jsonl 2>/dev/null | head -7; done
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_parity_gpu.py tests/test_dropin.py -q -x 2>&1 | tail -3
