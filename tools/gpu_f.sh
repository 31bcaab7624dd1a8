python -m pytest tests/test_fullsize_parity_gpu.py -k c3 -x -q 2>&1 | tail -3
python -m pytest tests/test_parity_gpu.py -x -q -k "epoch or binned" 2>&1 | tail -3
for v in 1 0; do SRLA_STAMP_CELLS=$v python bench.py --workload c3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2f_c3_cells$v.jsonl 2>&1; done
python tools/show.py gpurun_out/r2f_c3_cells1.jsonl gpurun_out/r2f_c3_cells0.jsonl
