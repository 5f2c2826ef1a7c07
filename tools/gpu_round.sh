#!/bin/bash
# One gpurun session: GPU tests, the bench line, then (only if the same command exited 0)
# the ncu launch list and one --set full capture of the sweep kernel.
#   tools/gpu_round.sh [tag] [pytest-args...]
TAG=${1:-run}; shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x "$@" > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?"
tail -4 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench=$?"; tail -1 gpurun_out/bench_$TAG.log | cut -c1-1500
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"  # the bench step (200 sweeps)
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu1_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_binary -s 3 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu2_$TAG.log 2>&1
echo "ncu=$?"
