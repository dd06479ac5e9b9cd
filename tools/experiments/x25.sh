timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q 2>&1 | tail -1 > gpurun_out/x25.txt
bash tools/run_ab.sh x25 "nch1 nch2" "fwd 32768 32 128 1" "fwd 32768 32 128 0" "fwd 131072 32 128 1"
