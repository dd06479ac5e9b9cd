timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/x10_pytest.txt
bash tools/run_ab.sh x10 "" "bwd 32768 32 128 1" "bwd 32768 32 128 0" "bwd 131072 32 128 1"
