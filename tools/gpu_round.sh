#!/bin/bash
# One GPU call: parity tests, smoke, bench (both arms), launch list, ncu full captures.
# Usage: tools/gpu_round.sh [tag]   (outputs under gpurun_out/<tag>/)
TAG=${1:-run}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.jsonl 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 > $O/bench_ref.jsonl 2> $O/bench_ref.err
timeout 900 python bench.py --workload c3 --no-cpu-baseline > $O/bench_c3.jsonl 2> $O/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
   python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_scan_bin|k_split|k_slice_apply' -s 30 -c 3 \
   -o /tmp/prof_scan python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/prof_scan.log 2>&1
ncu -i /tmp/prof_scan.ncu-rep --page raw --csv > $O/prof_scan.raw.csv 2>/dev/null   # gpurun brings back <= 64 MiB
ls -la $O
