bash tools/run_ab.sh x13 "nodq" "bwd 32768 32 128 1" "bwd 32768 32 128 0"
