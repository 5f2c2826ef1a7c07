# all-launch instruction captures of the two multi-level variants, their summaries into
# profiles/ (so the bench line that follows reads them), then the bench line
TAG=${1:-r02z}
for v in c5 c3_l5; do
  python bench.py --variant-only $v > gpurun_out/${TAG}_var_${v}_plain.log 2>&1 && \
  timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:sweep_ --csv \
      --log-file gpurun_out/${TAG}_var_${v}.csv python bench.py --variant-only $v > gpurun_out/${TAG}_var_${v}_ncu.log 2>&1
  echo "var $v rc=$?"
  python tools/ncu_variant_summary.py gpurun_out/${TAG}_var_${v}.csv $v profiles/r02_ncu_full_variant_${v}_summary.json && \
    cp profiles/r02_ncu_full_variant_${v}_summary.json gpurun_out/${TAG}_ncu_full_variant_${v}_summary.json
done
