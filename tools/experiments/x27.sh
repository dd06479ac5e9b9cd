bash tools/run_ab.sh x27 "poly3 poly18 allmufu" "fwd 32768 32 128 1" "fwd 32768 32 128 0"
