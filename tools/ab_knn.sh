#!/usr/bin/env bash
# A/B kNN timing (C2 filled and hollow-sphere sources) for library variants:
#   bash tools/ab_knn.sh "default old" [n] [k]
names=$1; n=${2:-10000000}; k=${3:-10}
for rep in 1 2; do
  for v in $names; do
    if [ "$v" = default ]; then lib=""; else lib=paper_1908_11807_b200/_lib/variants/$v.so; fi
    for src in cube sphere; do
      echo -n "[$v] "
      LBVH_LIB=$lib timeout 300 python tools/prof_knn.py $n 3 $k $src knn 2>&1 | tail -1
    done
  done
done
