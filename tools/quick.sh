#!/bin/bash
# quick GPU check: parity tests + C2/C3 bench lines.  Usage: tools/quick.sh tag [pytest-args]
TAG=${1:-q}; shift
O=gpurun_out/$TAG; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q "$@" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench.jsonl 2> $O/bench.err
timeout 900 python bench.py --workload c3 --no-cpu-baseline > $O/bench_c3.jsonl 2> $O/bench_c3.err
tail -3 $O/pytest_gpu.log
