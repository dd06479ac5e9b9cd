for bh in 2 1; do
  timeout 120 python tools/perf_tile.py bwd 9472 $bh 128 0 >> gpurun_out/x23.txt 2>&1
  A2D_LIB_PATH=xlib/lib_nodq.so timeout 120 python tools/perf_tile.py bwd 9472 $bh 128 0 | sed 's/^/nodq /' >> gpurun_out/x23.txt 2>&1
done
