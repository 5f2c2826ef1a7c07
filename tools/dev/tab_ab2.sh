# A/B the table kernel including the noisy first sweeps (dev)
for rep in 1 2; do
for lib in "$@"; do
  for a in "c5 5" "c5 700" "c5 900" "l5big 0" "l5big 1000"; do
    echo "$lib $(PCA_B200_LIB_OVERRIDE=$PWD/$lib timeout 300 python tools/prof_general.py $a --time)"
  done
done
done
