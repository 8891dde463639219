#!/usr/bin/env bash
# Build-kernel check on the GPU box: parity tests of the build, build timing
# at 1e7 / 1e8, launch list and --set full of the hierarchy kernels.
set -u
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02c}
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > $OUT/${TAG}_gputest.txt 2>&1
for n in 10000000 100000000; do
  timeout 300 python tools/prof_knn.py $n 9 10 cube build >> $OUT/${TAG}_build.txt 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_build_launches.csv python tools/prof_build.py 10000000 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"hierarchy_" -s 2 -c 2 \
    -o $OUT/${TAG}_hier python tools/prof_build.py 10000000 2 > $OUT/${TAG}_ncu_hier.log 2>&1
echo done
