#!/usr/bin/env bash
# Profiling pass for one round (run on the GPU box through gpurun):
#   bash tools/profile_round.sh r01
# Writes gpurun_out/<tag>_*: the bench JSON, the ncu launch list of a short
# bench run, and --set full captures of the kNN, radius-count, hierarchy and
# one-sweep kernels.  Summarise here with tools/ncu_summary.py into profiles/.
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/${TAG}_gpu.csv
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv python bench.py --profile --steps 2 --warmup 1 \
    > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_kernel -s 1 -c 1 \
    -o $OUT/${TAG}_knn python bench.py --profile --steps 2 --warmup 1 > $OUT/${TAG}_ncu_knn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"spatial_kernel|hierarchy_|onesweep_kernel|internal_rows" -s 4 -c 9 \
    -o $OUT/${TAG}_other python tools/prof_radius.py > $OUT/${TAG}_ncu_other.log 2>&1
echo done
