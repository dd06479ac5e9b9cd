bash tools/run_ab.sh x21 "norot" "bwd 32768 32 128 1" "bwd 131072 32 128 1"
