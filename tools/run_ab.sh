#!/usr/bin/env bash
# A/B tile timings of xlib2/ variants (tools/mk_variant.py), interleaved
# rounds so clock drift hits every variant alike.
#   bash tools/run_ab.sh TAG "base v1 v2" "bwd 32768 32 128 1" ["fwd 32768 32 128 1" ...]
set -u
TAG=$1; VARS=$2; shift 2
OUT=gpurun_out; mkdir -p $OUT
for round in 1 2; do
  for a in "$@"; do
    for v in $VARS; do
      A2D_LIB_PATH=xlib2/lib_$v.so timeout 180 python tools/perf_tile.py $a 2>&1 | tail -1 | sed "s/^/r$round $v  /" >> $OUT/${TAG}_ab.txt
    done
  done
done
