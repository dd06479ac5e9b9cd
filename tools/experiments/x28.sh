for r in 1 2 3; do
bash tools/run_ab.sh x28 "poly18" "fwd 32768 32 128 1" "fwd 65536 32 128 0"
done
