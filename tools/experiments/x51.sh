timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q -k backward 2>&1 | tail -1 > gpurun_out/x51.txt
A2D_LIB_PATH=xlib/lib_direct.so timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q -k "backward or full_size or grouped" 2>&1 | tail -1 >> gpurun_out/x51.txt
for r in 1 2; do
bash tools/run_ab.sh x51 "direct" "bwd 32768 32 128 1" "bwd 131072 32 128 1"
done
