timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd2_kernel -s 1 -c 1 -o gpurun_out/r1f_fwd python tools/perf_tile.py fwd 32768 32 128 1 > gpurun_out/r1f_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd128_kernel -s 1 -c 1 -o gpurun_out/r1f_bwd python tools/perf_tile.py bwd 32768 32 128 1 >> gpurun_out/r1f_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:bwd128_kernel -s 1 -c 1 -o gpurun_out/r1f_bwd128k python tools/perf_tile.py bwd 131072 32 128 1 >> gpurun_out/r1f_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:fwd2_kernel -s 1 -c 1 -o gpurun_out/r1f_fwd128k python tools/perf_tile.py fwd 131072 32 128 1 >> gpurun_out/r1f_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:lse_merge_kernel -c 1 -o gpurun_out/r1f_merge python tools/perf_merge.py >> gpurun_out/r1f_ncu.log 2>&1
