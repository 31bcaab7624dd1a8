for o in legacy fast; do SRLA_ORDER=$o timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-c3 --no-e2e > gpurun_out/r2h_$o.jsonl 2>&1; done
python tools/show.py gpurun_out/r2h_legacy.jsonl gpurun_out/r2h_fast.jsonl
SRLA_ORDER=fast timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2h_launches_fast.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-c3 --no-e2e > /dev/null 2>&1; echo ncu rc=$?
