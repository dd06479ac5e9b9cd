#!/usr/bin/env bash
# One gpurun call: GPU parity tests, smoke, bench line, ncu launch list and
# full captures of the two tile kernels.  Usage (from the repo root, on the box):
#   bash tools/gpu_check.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/${TAG}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
echo "smoke rc=$?" >> $OUT/${TAG}_smoke.txt
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?" >> $OUT/${TAG}_bench.err
timeout 300 python tools/perf_tile.py all 32768 32 128 1 > $OUT/${TAG}_perf_c2.txt 2>&1
timeout 300 python tools/perf_tile.py all 131072 32 128 1 >> $OUT/${TAG}_perf_c2.txt 2>&1
timeout 300 python tools/perf_tile.py all 32768 32 128 0 >> $OUT/${TAG}_perf_c2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
  > $OUT/${TAG}_launches_bench.log 2>&1
if [ "${NCU_FULL:-1}" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd2_kernel -s 1 -c 1 \
    -o $OUT/${TAG}_fwd python tools/perf_tile.py fwd 32768 32 128 1 > $OUT/${TAG}_ncu_fwd.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd128_kernel -s 1 -c 1 \
    -o $OUT/${TAG}_bwd python tools/perf_tile.py bwd 32768 32 128 1 > $OUT/${TAG}_ncu_bwd.log 2>&1
  timeout 600 ncu --set full --clock-control none -k regex:lse_merge_kernel -c 1 \
    -o $OUT/${TAG}_merge python tools/perf_merge.py > $OUT/${TAG}_ncu_merge.log 2>&1
fi
echo done
