for v in trnosm trnotma trnosmnotma; do echo "=== $v" >> gpurun_out/x6_trace.txt; A2D_LIB_PATH=xlib/lib_$v.so timeout 120 python tools/trace_fwd2.py 32768 32 0 2>&1 | tail -16 >> gpurun_out/x6_trace.txt; done
bash tools/run_ab.sh x6 "notma nosm" "fwd 32768 32 128 0"
