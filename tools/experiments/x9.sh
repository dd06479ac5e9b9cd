timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/x9_pytest.txt
A2D_LIB_PATH=xlib/lib_trace.so timeout 120 python tools/trace_fwd2.py 32768 32 0 > gpurun_out/x9_trace.txt 2>&1
bash tools/run_ab.sh x9 "noseq" "fwd 32768 32 128 1" "fwd 32768 32 128 0" "fwd 131072 32 128 1" "fwd 32768 32 64 1"
