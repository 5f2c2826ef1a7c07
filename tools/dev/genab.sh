#!/bin/bash
# A/B of general-kernel builds: C5 time course + other level counts
for lib in ${LIBS:-build_variants/base.so build_variants/new.so}; do echo $lib
PCA_B200_LIB_OVERRIDE=$PWD/$lib python tools/sweep_time_course.py 5 128 512 512 1000 250
PCA_B200_LIB_OVERRIDE=$PWD/$lib python tools/sweep_time_course.py 3 64 512 512 400 200
PCA_B200_LIB_OVERRIDE=$PWD/$lib python tools/sweep_time_course.py 9 1 2048 2048 200 100
done
