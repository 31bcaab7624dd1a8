for v in 1 0; do SRLA_EARLY_SPLIT=$v python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-c3 > gpurun_out/r2e_split$v.jsonl 2>&1; done
python tools/show.py gpurun_out/r2e_split1.jsonl gpurun_out/r2e_split0.jsonl
SRLA_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2e_n2.jsonl 2> gpurun_out/r2e_n2.err; tail -3 gpurun_out/r2e_n2.err
