for v in base red2; do A2D_LIB_PATH=xlib2/lib_$v.so timeout 120 python tools/check_variant.py 1000 3 128 >> gpurun_out/r2i_check_$v.txt 2>&1; A2D_LIB_PATH=xlib2/lib_$v.so timeout 120 python tools/check_variant.py 300 2 64 >> gpurun_out/r2i_check_$v.txt 2>&1; done
bash tools/run_ab.sh r2i "base_prev base" "fwd 32768 32 128 1" "fwd 131072 32 128 1"
bash tools/run_ab.sh r2i "base red1 red2 red3" "bwd 32768 32 128 1" "bwd 131072 32 128 1"
