# A/B the table kernel: us per sweep at C5 t=700 (no counting) / t=900 (counting) and 8192^2
# l=5 t=0 / t=1000, for each library given (default: the in-tree build)
libs=${@:-paper_2507_14869_b200/libpca_b200.so}
for rep in 1 2; do
for lib in $libs; do
  for a in "c5 700" "c5 900" "l5big 0" "l5big 1000"; do
    echo "$lib $(PCA_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python tools/prof_general.py $a --time)"
  done
done
done
