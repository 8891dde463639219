#!/usr/bin/env bash
# A/B timing of compile-time variants built with
#   python -c "from paper_1908_11807_b200 import _build; _build.build_variant(NAME, [DEFINES])"
# usage: bash tools/ab_lib.sh "name1 name2 ..." -- <args for tools/prof_knn.py>
# "default" = the in-tree library.  Each variant runs twice, interleaved.
names=$1; shift; [ "${1:-}" = "--" ] && shift
for rep in 1 2; do
  for v in $names; do
    if [ "$v" = default ]; then lib=""; else lib=paper_1908_11807_b200/_lib/variants/$v.so; fi
    echo -n "[$v] "
    LBVH_LIB=$lib timeout 300 python tools/prof_knn.py "$@" 2>&1 | tail -1
  done
done
