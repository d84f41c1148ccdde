#!/bin/bash
# On the GPU box: launch list + one full ncu capture of the vocab GEMMs.
# usage: scripts/profile.sh <tag> [config]
set -u
TAG=${1:-r01}
CFG=${2:-paper}
OUT=gpurun_out
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
# every attnsm launch of one step after 3 warm-up steps (cold-cache, serialised)
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:attnsm \
  -s 200 -c 60 --csv --log-file $OUT/launches_${TAG}.csv \
  python scripts/profile_step.py $CFG > $OUT/launches_${TAG}.log 2>&1
# full set on the vocab forward + first vocab-backward chunk launches of step 2
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:gemm_tc \
  -s 40 -c 4 -o $OUT/prof_${TAG} -f python scripts/profile_step.py $CFG > $OUT/prof_${TAG}.log 2>&1
echo profile done
