#!/usr/bin/env bash
# Round-2 evidence pass (GPU box): bench line, launch list, ncu --set full of
# the top kernels, compute-sanitizer over every kernel family.
#   bash tools/profile_r02.sh [tag]   -> gpurun_out/<tag>_*
# Summarise here: python tools/summarize_round.py <tag>
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/${TAG}_gpu.csv
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv python bench.py --profile --steps 2 --warmup 1 \
    > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:knn_kernel -s 1 -c 1 \
    -o $OUT/${TAG}_knn python tools/prof_knn.py 10000000 2 10 cube knn > $OUT/${TAG}_ncu_knn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"hierarchy_|onesweep_kernel|morton_kernel|scene_reduce" -s 9 -c 9 \
    -o $OUT/${TAG}_build python tools/prof_build.py 10000000 2 > $OUT/${TAG}_ncu_build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spatial_kernel -s 0 -c 1 \
    -o $OUT/${TAG}_c2_radius python tools/prof_knn.py 10000000 1 10 cube radius > $OUT/${TAG}_ncu_c2r.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spatial_kernel -s 0 -c 1 \
    -o $OUT/${TAG}_c3_radius python tools/prof_knn.py 10000000 1 10 sphere radius > $OUT/${TAG}_ncu_c3r.log 2>&1
# compute-sanitizer is closed on some GPU pools: SANITIZE=0 skips it
[ "${SANITIZE:-1}" = 1 ] && for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool" >> $OUT/${TAG}_sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_smoke.py \
      >> $OUT/${TAG}_sanitizer.txt 2>&1
done
echo done
