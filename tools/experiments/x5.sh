for v in trace trnoexp trallmufu trhalf trspin; do echo "=== $v" >> gpurun_out/x5_trace.txt; A2D_LIB_PATH=xlib/lib_$v.so timeout 120 python tools/trace_fwd2.py 32768 32 0 2>&1 | tail -16 >> gpurun_out/x5_trace.txt; done
bash tools/run_ab.sh x5 "allmufu half poly3 spin" "fwd 32768 32 128 0"
