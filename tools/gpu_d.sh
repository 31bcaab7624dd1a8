set -x
python -m pytest tests/test_multi_engine_gpu.py -x -q 2>&1 | tail -30
SRLA_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/r2d_bench_n2.jsonl 2> gpurun_out/r2d_bench_n2.err; tail -5 gpurun_out/r2d_bench_n2.err
