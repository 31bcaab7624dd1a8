bash tools/gpu_round.sh r02b
bash tools/ncu_round.sh r02b both
rm -f gpurun_out/r02b/*.ncu-rep
du -sh gpurun_out/r02b
