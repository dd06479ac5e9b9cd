# Round-end evidence run: GPU tests, smoke, the bench contract line, extra
# SURVEY configs on one GPU, ncu launch list.  Usage: bash tools/final_check.sh TAG
set -u
TAG=${1:-r1e}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/${TAG}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/${TAG}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/${TAG}_smoke.txt
timeout 600 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
timeout 300 python bench.py --seq-len 32768 --no-cpu > $OUT/${TAG}_bench_c2.json 2>> $OUT/${TAG}_bench.err
timeout 600 python bench.py --seq-len 524288 --heads 16 --fwd-only --non-causal --no-cpu --steps 3 > $OUT/${TAG}_bench_c5_1gpu.json 2>> $OUT/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
  > $OUT/${TAG}_launches_bench.log 2>&1
echo done
