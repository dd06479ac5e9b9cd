A2D_LIB_PATH=xlib/lib_cs2.so timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q -k "forward" 2>&1 | tail -1 > gpurun_out/x39.txt
for r in 1 2; do
bash tools/run_ab.sh x39 "cs2" "fwd 32768 32 128 1" "fwd 32768 32 128 0"
done
