#!/bin/bash
# same-box A/B of library builds in ablib/ (alternating, 3 rounds)
# usage: scripts/ab_lib.sh [config] lib1 lib2 ...
cfg=${CFG:-paper}
for round in 1 2 3; do
  for l in "$@"; do
    echo -n "$l "; ATTNSM_LIB=$PWD/ablib/$l.so timeout 100 python scripts/quick_time.py $cfg | tail -1
  done
done
