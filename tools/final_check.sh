#!/usr/bin/env bash
# Round evidence run (one gpurun call): GPU tests, smoke, the bench contract
# line at the metric config and the SURVEY configs on one GPU, the ncu launch
# list of the bench, full ncu captures of both tile kernels at the bench
# config (-> profiles/traffic.json) and of the LSE merge at the 2x4 merge size,
# and the per-tensor parity report.   Usage: bash tools/final_check.sh TAG
set -u
TAG=${1:-r2}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/${TAG}_smi.txt 2>&1
nproc >> $OUT/${TAG}_smi.txt; lscpu | grep "Model name" >> $OUT/${TAG}_smi.txt
timeout 1200 python -m pytest tests -m gpu -q > $OUT/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/${TAG}_smoke.txt
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/${TAG}_bench_ref.json 2>> $OUT/${TAG}_bench.err
timeout 600 python bench.py --seq-len 32768 --no-cpu > $OUT/${TAG}_bench_c2.json 2>> $OUT/${TAG}_bench.err
timeout 900 python bench.py --seq-len 524288 --heads 16 --fwd-only --non-causal --no-cpu --steps 3 > $OUT/${TAG}_bench_c5_1gpu.json 2>> $OUT/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
  > $OUT/${TAG}_launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fwd2_kernel -s 1 -c 1 \
  -o $OUT/${TAG}_fwd128k python tools/perf_tile.py fwd 131072 32 128 1 > $OUT/${TAG}_ncu_fwd.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bwd128_kernel -s 1 -c 1 \
  -o $OUT/${TAG}_bwd128k python tools/perf_tile.py bwd 131072 32 128 1 > $OUT/${TAG}_ncu_bwd.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:lse_merge_kernel -c 1 \
  -o $OUT/${TAG}_merge python tools/perf_merge.py 4 524288 128 > $OUT/${TAG}_ncu_merge.log 2>&1
timeout 1500 python tools/parity_report.py --out $OUT/${TAG}_parity.json > $OUT/${TAG}_parity.log 2>&1
echo done
