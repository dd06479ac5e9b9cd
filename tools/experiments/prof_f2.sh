set -u
OUT=gpurun_out; mkdir -p $OUT
TAG=${1:-f2}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd2_kernel -s 1 -c 1 \
    -o $OUT/${TAG}_fwd2 python tools/perf_tile.py fwd 32768 32 128 1 > $OUT/${TAG}_ncu_fwd2.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:bwd128_kernel -s 1 -c 1 \
    -o $OUT/${TAG}_bwd_128k python tools/perf_tile.py bwd 131072 32 128 1 > $OUT/${TAG}_ncu_bwd128k.log 2>&1
echo done
