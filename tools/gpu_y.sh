python -c "import torch; print(torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream,'priority_range') else 'n/a')"
B="--steps 20 --warmup 3 --no-c3 --no-cpu-baseline --no-e2e"
for v in 1 0 1 0; do SRLA_SPLIT_PRIO=$v timeout 200 python bench.py $B > gpurun_out/r2y_p$v.jsonl 2>&1; python tools/show.py gpurun_out/r2y_p$v.jsonl 2>/dev/null | head -4; done
for v in 1 0; do SRLA_SPLIT_PRIO=$v timeout 200 python bench.py --workload c3 $B > gpurun_out/r2y_c3_p$v.jsonl 2>&1; python tools/show.py gpurun_out/r2y_c3_p$v.jsonl 2>/dev/null | head -1; done
