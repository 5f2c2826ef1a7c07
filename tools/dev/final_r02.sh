# round-2 closing run: GPU suite, smoke, variant instruction captures (-> profiles/ on the box
# so the bench line reads them), bench line, launch list, packed + table ncu captures, DRAM
TAG=${1:-r02z}
timeout 1700 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/${TAG}_pytest.log
cp gpurun_out/parity_report.json gpurun_out/${TAG}_parity_report.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke=$?"; tail -1 gpurun_out/${TAG}_smoke.log
bash tools/dev/variants_r02.sh $TAG
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench=$?"; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-300
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-variants"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1; echo "ncu1=$?"
ncu --set full --clock-control none --import-source on -k regex:sweep_packed -s 3 -c 1 -o gpurun_out/${TAG}_packed_full $CMD > gpurun_out/${TAG}_ncu2.log 2>&1; echo "ncu2=$?"
ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:sweep_packed -c 12 --csv --log-file gpurun_out/${TAG}_dram_multi.csv $CMD > gpurun_out/${TAG}_ncu3.log 2>&1; echo "ncu3=$?"
for a in "c5 900" "c5 500"; do set -- $a; timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -c 1 -o gpurun_out/${TAG}_tab_$1_$2 python tools/prof_general.py $1 $2 > gpurun_out/${TAG}_ncu_tab_$1_$2.log 2>&1; echo "ncu tab $1 $2 rc=$?"; done
