A2D_LIB_PATH=xlib/lib_dq4.so timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q -k backward 2>&1 | tail -1 > gpurun_out/x30.txt
A2D_LIB_PATH=xlib/lib_dq8.so timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q -k backward 2>&1 | tail -1 >> gpurun_out/x30.txt
for r in 1 2; do
bash tools/run_ab.sh x30 "dq4 dq8" "bwd 32768 32 128 1" "bwd 32768 32 128 0"
done
