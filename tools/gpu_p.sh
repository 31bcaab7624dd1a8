timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2p_gpu.log 2>&1; echo "gpu rc=$?"; tail -15 gpurun_out/r2p_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2p_bench.jsonl 2> gpurun_out/r2p_bench.err; echo "bench rc=$?"
python tools/show.py gpurun_out/r2p_bench.jsonl
python -c "import json;d=json.loads(open('gpurun_out/r2p_bench.jsonl').read().strip().splitlines()[-1]);print(d['e2e_dropin']);print(d['e2e']['value'])"
