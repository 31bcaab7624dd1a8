for v in "SRLA_STAMP_CELLS=1 SRLA_ORDER=fast" "SRLA_STAMP_CELLS=0 SRLA_ORDER=fast" "SRLA_STAMP_CELLS=1 SRLA_ORDER=legacy"; do
  echo "== $v"; env $v timeout 300 python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2j.jsonl 2>&1
  python tools/show.py gpurun_out/r2j.jsonl
done
timeout 300 python -m pytest tests/test_fullsize_parity_gpu.py -x -q -k c3 2>&1 | tail -2
