set -x
for n in 129 300 1000; do timeout 60 python tools/check_variant.py $n 3 128 >> gpurun_out/r2f_check.txt 2>&1; done
timeout 60 python tools/check_variant.py 1000 2 96 >> gpurun_out/r2f_check.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_pytest.txt 2>&1
bash tools/run_ab.sh r2f "base fwd1" "fwd 32768 32 128 1" "fwd 131072 32 128 1" "fwd 32768 32 128 0"
