#!/bin/bash
# Path Sorting evidence for the default (wavefront) mapping, run under gpurun on one GPU:
# event-timed iterations and the warp execution efficiency of every iteration kernel on
# the unsorted (path-major) vs the B-sorted store.  Usage: scripts/sorting_evidence.sh TAG PATHS
set -u
mkdir -p gpurun_out
TAG=${1:-r13}
P=${2:-3e7}
B="python bench.py --paths $P --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$B --no-sort > gpurun_out/sortev_unsorted_$TAG.log 2>&1
$B > gpurun_out/sortev_sorted_$TAG.log 2>&1
M=smsp__thread_inst_executed_per_inst_executed.ratio,gpu__time_duration.sum,smsp__inst_executed.sum
C="python bench.py --paths $P --steps 1 --warmup 2 --no-cpu-baseline --no-e2e"
for s in sorted unsorted; do
  F=""; [ $s = unsorted ] && F="--no-sort"
  ncu --metrics $M --clock-control none --csv -k regex:"k_prefix|k_le_forward|k_le_gradient|k_path_gradient" \
      --log-file gpurun_out/sortev_warp_${s}_$TAG.csv $C $F > /dev/null 2>&1
done
echo sorting evidence done
