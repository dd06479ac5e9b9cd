for r in 1 2; do
bash tools/run_ab.sh x54 "kst2" "fwd 32768 32 128 1" "fwd 131072 32 128 1"
done
