for r in 1 2; do
bash tools/run_ab.sh x29 "bpoly0 bpoly18" "bwd 32768 32 128 1" "bwd 32768 32 128 0"
done
