#!/usr/bin/env bash
# C3 radius 2P: launch list + --set full of the count kernel and the spill copy.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_c3_launches.csv python tools/prof_knn.py 10000000 2 10 sphere radius > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"spatial_kernel|spill_copy|compact_warp" -s 3 -c 3 \
    -o $OUT/${TAG}_c3_full python tools/prof_knn.py 10000000 2 10 sphere radius > $OUT/${TAG}_c3.log 2>&1
echo done
