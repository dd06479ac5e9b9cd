nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 500 > gpurun_out/r2o_clocks.csv &
SMI=$!
export A2D_PERF_ITERS=20
bash tools/run_ab.sh r2o "base bwdsleep" "bwd 131072 32 128 1"
bash tools/run_ab.sh r2o "base fwdsleep" "fwd 131072 32 128 1"
kill $SMI
