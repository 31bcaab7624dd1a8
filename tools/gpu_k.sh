mkdir -p gpurun_out/ncu
SRLA_STAMP_CELLS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_stamp_cells -s 3 -c 1 -o gpurun_out/ncu/r2k_cells python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu cells rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_scan_bin -s 5 -c 1 -o gpurun_out/ncu/r2k_k1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c3 > /dev/null 2>&1; echo "ncu k1 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_split -s 5 -c 1 -o gpurun_out/ncu/r2k_split python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c3 > /dev/null 2>&1; echo "ncu split rc=$?"
ls -la gpurun_out/ncu
