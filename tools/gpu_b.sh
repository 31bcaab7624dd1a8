set -x
python -m pytest tests/test_parity_gpu.py -k state_blocks -x -q 2>&1 | tail -5
python -m pytest tests/test_fullsize_parity_gpu.py -k "c2 or c5" -x -q -s 2>&1 | tail -15
python tests/golden/make_fullsize.py c3 --threads 16 --out gpurun_out/fullsize_c3.json > gpurun_out/fullsize_c3.log 2>&1
tail -3 gpurun_out/fullsize_c3.log
cp gpurun_out/fullsize_c3.json tests/golden/fullsize_c3.json && python -m pytest tests/test_fullsize_parity_gpu.py -k "c3" -x -q -s 2>&1 | tail -8
