bash tools/gpu_round.sh r02a
bash tools/ncu_round.sh r02a both
du -sh gpurun_out/r02a
