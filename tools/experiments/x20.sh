timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/x20_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/x20_smoke.txt
timeout 900 ncu --set full --clock-control none -k regex:bwd128_kernel -s 1 -c 1 -o gpurun_out/x20_bwd128k python tools/perf_tile.py bwd 131072 32 128 1 > gpurun_out/x20_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:fwd2_kernel -s 1 -c 1 -o gpurun_out/x20_fwd128k python tools/perf_tile.py fwd 131072 32 128 1 >> gpurun_out/x20_ncu.log 2>&1
