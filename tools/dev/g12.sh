timeout 600 python -m pytest tests/test_gpu_debug.py -q > gpurun_out/r02_guard.log 2>&1; echo "guard rc=$?"; tail -2 gpurun_out/r02_guard.log
PCA_B200_LIB_OVERRIDE=$PWD/build_variants/libpca_b200_debug.so timeout 1700 python -m pytest tests -m gpu -q > gpurun_out/r02_debug_build_pytest.log 2>&1; echo "debug rc=$?"; tail -3 gpurun_out/r02_debug_build_pytest.log
