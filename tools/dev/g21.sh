KSEL=4 timeout 900 python tools/tune_packed.py
for a in "c5 700" "c5 900" "l5big 0" "l5big 1000"; do timeout 300 python tools/prof_general.py $a --time; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "table_kernel or randomised_new or config5" 2>&1 | tail -2
for lib in build_variants/packed_P1.so build_variants/packed_P2.so; do PCA_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python -m pytest tests/test_gpu_packed.py -q -x 2>&1 | tail -1; done
