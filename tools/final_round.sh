#!/bin/bash
# Round-end evidence: default bench (both arms), C3 bench, launch lists and ncu captures.
TAG=${1:-final}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1; lscpu > $O/lscpu.txt 2>&1
timeout 900 python bench.py > $O/bench.jsonl 2> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.jsonl 2> $O/bench_ref.err
timeout 900 python bench.py --workload c3 > $O/bench_c3.jsonl 2> $O/bench_c3.err
bash tools/ncu_round.sh $TAG/ncu
