timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q -k "forward" 2>&1 | tail -1 > gpurun_out/x49.txt
A2D_LIB_PATH=xlib/lib_split.so timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q -k "forward" 2>&1 | tail -1 >> gpurun_out/x49.txt
for r in 1 2; do
bash tools/run_ab.sh x49 "split" "fwd 32768 32 128 1" "fwd 32768 32 128 0"
done
