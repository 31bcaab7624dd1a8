B="--workload c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
for v in 1 0 1; do SRLA_GATHER_TMA=$v timeout 300 python bench.py $B > gpurun_out/r2v_tma$v.jsonl 2>&1; python tools/show.py gpurun_out/r2v_tma$v.jsonl 2>/dev/null | head -6; done
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_parity_gpu.py -q -x -k "epoch or c3 or binned" 2>&1 | tail -3
