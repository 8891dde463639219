#!/usr/bin/env bash
# Round-2 profiling pass A: build kernels (launch list + --set full of the
# hierarchy and sort kernels), C3 radius count kernel, CUB sort bar.
set -u
OUT=gpurun_out
mkdir -p $OUT
tools/cub_vs_onesweep 20 > $OUT/r02_cub_vs_onesweep.json 2> $OUT/r02_cub.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/r02_build_launches.csv python tools/prof_build.py 10000000 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"hierarchy_|onesweep_kernel|histogram" -s 6 -c 7 \
    -o $OUT/r02_build python tools/prof_build.py 10000000 3 > $OUT/r02_ncu_build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"spatial_kernel" -s 0 -c 2 \
    -o $OUT/r02_c3_radius python tools/prof_knn.py 10000000 1 10 sphere radius > $OUT/r02_ncu_c3.log 2>&1
echo done
