#!/usr/bin/env bash
# A/B build timing at 1e7 (and 1e8) for library variants:
#   bash tools/ab_build.sh "default old t256" [n]
names=$1; n=${2:-10000000}
for rep in 1 2; do
  for v in $names; do
    if [ "$v" = default ]; then lib=""; else lib=paper_1908_11807_b200/_lib/variants/$v.so; fi
    echo -n "[$v] "
    LBVH_LIB=$lib timeout 300 python tools/prof_knn.py $n 9 10 cube build 2>&1 | tail -1
  done
done
