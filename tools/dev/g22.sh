KSEL=2 timeout 900 python tools/tune_packed.py
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02e_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02e_pytest.log
timeout 300 python tools/time_binary.py
