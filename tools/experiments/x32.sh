for r in 1 2; do
bash tools/run_ab.sh x32 "halfdq nodq" "bwd 32768 32 128 1" "bwd 131072 32 128 1"
done
