# copy a closing run's outputs (tag) into profiles/ (dev)
T=${1:?tag}
set -e
tail -1 gpurun_out/${T}_bench.log | python -m json.tool > profiles/r02_bench.json
cp gpurun_out/${T}_ncu_full_variant_c5_summary.json profiles/r02_ncu_full_variant_c5_summary.json
cp gpurun_out/${T}_ncu_full_variant_c3_l5_summary.json profiles/r02_ncu_full_variant_c3_l5_summary.json
cp gpurun_out/${T}_parity_report.json profiles/r02_parity_report.json
cp gpurun_out/${T}_launches.csv profiles/r02_launches.csv
python tools/launch_summary.py gpurun_out/${T}_launches.csv > profiles/r02_launches_summary.txt
python tools/ncu_summary.py gpurun_out/${T}_packed_full.ncu-rep --json profiles/r02_ncu_full_sweep_packed_summary.json --H 8192 --sites 67108864 > /dev/null
python tools/ncu_lines.py gpurun_out/${T}_packed_full.ncu-rep --top 40 --out profiles/r02_ncu_lines_sweep_packed.txt > /dev/null
python tools/ncu_dram_multi.py gpurun_out/${T}_dram_multi.csv --out profiles/r02_dram_multilaunch_sweep_packed.json --H 8192 --sites 67108864 > /dev/null
[ -f gpurun_out/${T}_perf_configs.jsonl ] && grep '^{' gpurun_out/${T}_perf_configs.jsonl > profiles/r02_perf_configs.jsonl
[ -f gpurun_out/${T}_pca_vs_gibbs.json ] && cp gpurun_out/${T}_pca_vs_gibbs.json profiles/r02_pca_vs_gibbs.json
[ -f gpurun_out/${T}_time_course_c5.json ] && cp gpurun_out/${T}_time_course_c5.json profiles/r02_time_course_c5.json
echo collected $T
