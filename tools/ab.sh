#!/usr/bin/env bash
# A/B timing of env-switch variants: bash tools/ab.sh "<ENV=.. ENV2=..>" "<...>" -- args for prof_knn.py
# Each variant runs in its own process (the library reads switches once).
variants=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do variants+=("$1"); shift; done
[ "${1:-}" = "--" ] && shift
for v in "${variants[@]}"; do
  echo -n "[$v] "
  env $v timeout 300 python tools/prof_knn.py "$@" 2>&1 | tail -1
done
