B="--steps 20 --warmup 3 --no-c3 --no-cpu-baseline --no-e2e"
for v in 256 512 1024 256; do SRLA_APPLY_THREADS=$v timeout 200 python bench.py $B > gpurun_out/r2u_at$v.jsonl 2>&1; python tools/show.py gpurun_out/r2u_at$v.jsonl 2>/dev/null | head -5; done
