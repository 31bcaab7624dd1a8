O=gpurun_out/q12; mkdir -p $O
bash tools/quick.sh q12
SRLA_EOS_TRACE=1 timeout 900 python bench.py --workload c3 --no-cpu-baseline --no-e2e --steps 4 2>&1 | grep "srla eos" | tail -3 > $O/eos_trace.txt
