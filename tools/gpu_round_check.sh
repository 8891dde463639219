set -u
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/r02b_gpu.csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/r02b_gputest.txt 2>&1
timeout 600 python bench.py > $OUT/r02b_bench.json 2> $OUT/r02b_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/r02b_launches.csv python bench.py --profile --steps 2 --warmup 1 > /dev/null 2>&1
echo done
