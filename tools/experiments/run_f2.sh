set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_tile.py -m gpu -x -q > $OUT/f2_pytest.txt 2>&1; echo "rc=$?" >> $OUT/f2_pytest.txt
for c in 1 0; do
 timeout 120 python tools/perf_tile.py fwd 32768 32 128 $c >> $OUT/f2_perf.txt 2>&1
 A2D_FWD_V1=1 timeout 120 python tools/perf_tile.py fwd 32768 32 128 $c | sed 's/^/v1 /' >> $OUT/f2_perf.txt 2>&1
done
timeout 120 python tools/perf_tile.py fwd 131072 32 128 1 >> $OUT/f2_perf.txt 2>&1
timeout 120 python tools/perf_tile.py fwd 32768 32 64 1 >> $OUT/f2_perf.txt 2>&1
A2D_FWD_V1=1 timeout 120 python tools/perf_tile.py fwd 32768 32 64 1 | sed 's/^/v1 /' >> $OUT/f2_perf.txt 2>&1
