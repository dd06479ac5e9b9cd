#!/usr/bin/env bash
# One gpurun call: GPU parity tests, smoke, bench line, tile timings, ncu
# launch list and full captures of the tile kernels.  Usage (repo root, on the box):
#   bash tools/gpu_check.sh TAG            (NCU_FULL=0 skips the full captures)
set -u
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_smi.txt 2>&1
nproc >> $OUT/${TAG}_smi.txt; lscpu | grep "Model name" >> $OUT/${TAG}_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/${TAG}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
echo "smoke rc=$?" >> $OUT/${TAG}_smoke.txt
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?" >> $OUT/${TAG}_bench.err
timeout 300 python tools/perf_tile.py all 32768 32 128 1 > $OUT/${TAG}_perf.txt 2>&1
timeout 300 python tools/perf_tile.py all 131072 32 128 1 >> $OUT/${TAG}_perf.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
  > $OUT/${TAG}_launches_bench.log 2>&1
if [ "${NCU_FULL:-1}" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd2_kernel -s 1 -c 1 \
    -o $OUT/${TAG}_fwd python tools/perf_tile.py fwd 32768 32 128 1 > $OUT/${TAG}_ncu_fwd.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:bwd -s 1 -c 1 \
    -o $OUT/${TAG}_bwd python tools/perf_tile.py bwd 32768 32 128 1 > $OUT/${TAG}_ncu_bwd.log 2>&1
fi
echo done
