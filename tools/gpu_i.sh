timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2i_bench.jsonl 2> gpurun_out/r2i_bench.err; echo "bench rc=$?"
python tools/show.py gpurun_out/r2i_bench.jsonl
python - <<'PY'
import json; d=json.loads(open('gpurun_out/r2i_bench.jsonl').read().strip().splitlines()[-1]); c=d['c3']
print('c3', c['value'], c['ms_per_step'], c['end_of_slice_ms']['device_median'], 'flagged/step', d['flagged_hosts_per_step'])
for k,v in c['kernels'].items(): print('  c3', k, round(v['ms_per_launch'],3), v.get('frac'), v.get('share_of_step'))
PY
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_gpu.log 2>&1; echo "gpu rc=$?"; tail -15 gpurun_out/r2i_gpu.log
