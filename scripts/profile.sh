#!/bin/bash
# On the GPU box: launch list of one step + one full ncu capture of the
# vocab-forward and one vocab-backward chunk launch.
# usage: scripts/profile.sh <tag> [config]
set -u
TAG=${1:-r01}
CFG=${2:-paper}
OUT=gpurun_out
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
LPS=$(python scripts/profile_step.py $CFG 2>/dev/null | awk '/launches per step/ {print $4}')
echo "launches per step: $LPS"
# every stage launch of step 4 (after 3 warm-up steps), cold-cache, serialised
timeout 600 $NCU --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"gemm_tc|lse_reduce|dz_kernel|lens_kernel|dlogits_from" \
  -s $((3 * LPS)) -c $LPS --csv --log-file $OUT/launches_${TAG}.csv \
  python scripts/profile_step.py $CFG > $OUT/launches_${TAG}.log 2>&1
# full set: vocab_fwd, chunk 0's dlogits and chunk 0's vocab-backward launch
# of the second step (the kernels matching the regex: all but lse_reduce, dz,
# lengths upload)
TCPS=$((LPS - 3))
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"gemm_tc|dlogits_from" \
  -s $((TCPS + 3)) -c 3 -o $OUT/prof_${TAG} -f python scripts/profile_step.py $CFG > $OUT/prof_${TAG}.log 2>&1
echo profile done
