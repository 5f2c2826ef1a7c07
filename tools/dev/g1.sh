set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu_a.log 2>&1; echo pytest=$?
for a in "c5 900" "l5big 0" "l5big 1000"; do timeout 300 python tools/prof_general.py $a --time; done > gpurun_out/r02_gen_times.log 2>&1
for a in "c5 900" "l5big 0" "l5big 1000"; do set -- $a; timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -c 1 -o gpurun_out/r02_gen_$1_$2 python tools/prof_general.py $1 $2 > gpurun_out/r02_ncu_gen_$1_$2.log 2>&1; echo ncu $1 $2 rc=$?; done
