A2D_LIB_PATH=xlib/lib_dqred.so timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q -k backward 2>&1 | tail -2 > gpurun_out/x16_pytest.txt
bash tools/run_ab.sh x16 "dqred" "bwd 32768 32 128 1" "bwd 32768 32 128 0" "bwd 131072 32 128 1"
