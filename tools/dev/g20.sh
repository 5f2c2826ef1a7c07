for lib in build_variants/tab_B.so build_variants/tab_C.so build_variants/tab_D.so paper_2507_14869_b200/libpca_b200.so; do
  for a in "c5 700" "c5 900" "l5big 0" "l5big 1000"; do echo "$lib $(PCA_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python tools/prof_general.py $a --time)"; done
done
