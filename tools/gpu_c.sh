set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2c_gpu.log 2>&1; tail -3 gpurun_out/r2c_gpu.log
( time python bench.py --steps 20 --warmup 5 ) > gpurun_out/r2c_bench.jsonl 2> gpurun_out/r2c_bench.err; tail -3 gpurun_out/r2c_bench.err
( time python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/r2c_ref.jsonl 2> gpurun_out/r2c_ref.err; tail -3 gpurun_out/r2c_ref.err
