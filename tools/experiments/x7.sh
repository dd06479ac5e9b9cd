timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q 2>&1 | tail -2 > gpurun_out/x7_pytest.txt
A2D_LIB_PATH=xlib/lib_trace.so timeout 120 python tools/trace_fwd2.py 32768 32 0 > gpurun_out/x7_trace.txt 2>&1
bash tools/run_ab.sh x7 "nosm" "fwd 32768 32 128 1" "fwd 32768 32 128 0" "fwd 131072 32 128 1"
