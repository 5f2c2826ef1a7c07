set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "table_kernel or lockstep_random or config2 or multi_sweep or strips or l1_l2 or randomised or config5" > gpurun_out/r02_pytest_tab.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r02_pytest_tab.log
for k in 0 1; do for a in "c5 700" "c5 900" "l5big 0" "l5big 1000"; do timeout 300 python tools/prof_general.py $a --time --kernel $k; done; done > gpurun_out/r02_tab_times.log 2>&1
cat gpurun_out/r02_tab_times.log | grep us
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -c 1 -o gpurun_out/r02_tab_c5_900 python tools/prof_general.py c5 900 > gpurun_out/r02_ncu_tab.log 2>&1; echo ncu=$?
