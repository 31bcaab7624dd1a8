timeout 900 python -m pytest tests -m gpu -x -q -k "not fullsize" > gpurun_out/r2g_gpu.log 2>&1; echo "gpu rc=$?"; tail -15 gpurun_out/r2g_gpu.log
timeout 300 python -m pytest tests/test_fullsize_parity_gpu.py -x -q > gpurun_out/r2g_full.log 2>&1; echo "full rc=$?"; tail -5 gpurun_out/r2g_full.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_bench.jsonl 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
python tools/show.py gpurun_out/r2g_bench.jsonl
python - <<'PY'
import json; d=json.loads(open('gpurun_out/r2g_bench.jsonl').read().strip().splitlines()[-1]); c=d['c3']
print('c3', c['value'], c['ms_per_step'], c['end_of_slice_ms'])
for k,v in c['kernels'].items(): print('  c3', k, round(v['ms_per_launch'],3), v.get('frac'), v.get('share_of_step'))
PY
