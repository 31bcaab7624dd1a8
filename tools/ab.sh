#!/bin/bash
# A/B a knob on the GPU box: one bench line per setting.
#   tools/ab.sh <tag> <ENV_VAR> <value>... [-- extra bench.py args]
# e.g. tools/ab.sh r1 SRLA_REGION_MB 8 16 32 -- --workload c2 --steps 10
# Knobs (engine.cu): SRLA_REGION_MB, SRLA_FINE_KB, SRLA_SPLIT_WAVES, SRLA_EARLY_SPLIT,
# SRLA_RETAIN_LATE, SRLA_SPLIT_THREADS, SRLA_STAMP_SPARSE, SRLA_STAMP_BLOCKS, SRLA_APPLY_BLOCKS, SRLA_EPOCH, SRLA_NIBBLE, SRLA_OVERLAP, SRLA_DIRECT_MARKS.
TAG=$1; VAR=$2; shift 2
VALS=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do VALS+=("$1"); shift; done
[ "$1" == "--" ] && shift
O=gpurun_out/$TAG; mkdir -p $O
for v in "${VALS[@]}"; do
  env $VAR=$v timeout 900 python bench.py --no-cpu-baseline --no-e2e "$@" > $O/bench_${VAR}_$v.jsonl 2>&1
done
python tools/show.py $O/*.jsonl
