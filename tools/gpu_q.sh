B="--steps 20 --warmup 3 --no-c3 --no-cpu-baseline --no-e2e"
for v in 1 0 1 0; do SRLA_K1_PACK=$v timeout 300 python bench.py $B > gpurun_out/r2q_pack$v.jsonl 2>&1; python tools/show.py gpurun_out/r2q_pack$v.jsonl | head -2; done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2q_gpu.log 2>&1; echo "gpu rc=$?"; tail -8 gpurun_out/r2q_gpu.log
