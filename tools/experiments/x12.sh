timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/x12_pytest.txt
A2D_LIB_PATH=xlib/lib_TRACE.so timeout 120 python tools/trace_bwd.py 32768 32 1 2>&1 | tail -18 > gpurun_out/x12_trace.txt
bash tools/run_ab.sh x12 "" "bwd 32768 32 128 1" "bwd 32768 32 128 0" "bwd 131072 32 128 1"
