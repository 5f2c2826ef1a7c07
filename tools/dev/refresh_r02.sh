# refresh every round-2 number after the wave-sizing change: suite, smoke, variants + bench,
# launch list, per-config times, PCA vs Gibbs, time courses
TAG=${1:-r02x}
timeout 1700 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/${TAG}_pytest.log
cp gpurun_out/parity_report.json gpurun_out/${TAG}_parity_report.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke=$?"; tail -1 gpurun_out/${TAG}_smoke.log
bash tools/dev/variants_r02.sh $TAG
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench=$?"; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-200
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-variants"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1; echo "ncu1=$?"
ncu --set full --clock-control none --import-source on -k regex:sweep_packed -s 3 -c 1 -o gpurun_out/${TAG}_packed_full $CMD > gpurun_out/${TAG}_ncu2.log 2>&1; echo "ncu2=$?"
ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:sweep_packed -c 12 --csv --log-file gpurun_out/${TAG}_dram_multi.csv $CMD > gpurun_out/${TAG}_ncu3.log 2>&1; echo "ncu3=$?"
timeout 900 python tools/perf_configs.py > gpurun_out/${TAG}_perf_configs.jsonl 2>&1; echo "perf=$?"
timeout 900 python tools/pca_vs_gibbs.py > gpurun_out/${TAG}_pca_vs_gibbs.log 2>&1; echo "pvg=$?"; cp gpurun_out/pca_vs_gibbs.json gpurun_out/${TAG}_pca_vs_gibbs.json
timeout 600 python tools/sweep_time_course.py 5 128 512 512 1000 50 > gpurun_out/${TAG}_time_course_c5.json 2>&1; echo "tc=$?"
