timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/x26.txt
bash tools/run_ab.sh x26 "rowmax" "fwd 32768 32 128 1" "fwd 32768 32 128 0" "fwd 131072 32 128 1"
