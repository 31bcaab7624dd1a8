B="--steps 10 --warmup 3 --no-c3"
bash tools/ab.sh r2m_fine SRLA_FINE_KB 16 32 64 -- $B 2>&1 | grep -v "^ "
bash tools/ab.sh r2m_region SRLA_REGION_MB 8 32 -- $B 2>&1 | grep -v "^ "
bash tools/ab.sh r2m_waves SRLA_SPLIT_WAVES 1 4 -- $B 2>&1 | grep -v "^ "
