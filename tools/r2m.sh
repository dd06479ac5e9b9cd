timeout 600 python -m pytest tests/test_gpu_tile.py tests/test_dropin.py -m gpu -x -q > gpurun_out/r2m_pytest.txt 2>&1
bash tools/run_ab.sh r2m "base_prev base" "fwd 32768 32 128 1" "fwd 131072 32 128 1" "fwd 32768 32 128 0"
