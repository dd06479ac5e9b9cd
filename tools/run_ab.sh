# A/B tile timings across xlib variants: bash tools/run_ab.sh TAG "variants" "perf args..."
set -u
TAG=$1; VARS=$2; shift 2
OUT=gpurun_out; mkdir -p $OUT
for a in "$@"; do
  timeout 120 python tools/perf_tile.py $a 2>&1 | sed "s/^/main  /" >> $OUT/${TAG}_ab.txt
  for v in $VARS; do
    A2D_LIB_PATH=xlib/lib_$v.so timeout 120 python tools/perf_tile.py $a 2>&1 | sed "s/^/$v  /" >> $OUT/${TAG}_ab.txt
  done
done
