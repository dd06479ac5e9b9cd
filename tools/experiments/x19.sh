bash tools/run_ab.sh x19 "sleepall" "all 32768 32 128 1" "all 131072 32 128 1"
