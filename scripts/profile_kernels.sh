#!/bin/bash
# End-of-change profiling at the bench config (run under gpurun, one GPU):
#   plain run -> launch list of the same command -> one --set full capture per hot kernel
# (ncu fully replays only the first matching kernel of a process at these memory sizes,
# SKIP = matching launches to skip, W = warm-up steps;
# so each kernel gets its own process).  Usage: scripts/profile_kernels.sh TAG [PATHS]
set -u
mkdir -p gpurun_out
TAG=${1:-r7}
P=${2:-1e8}
CMD="python bench.py --paths $P --steps 1 --warmup ${W:-1} --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
for k in ${KERNELS:-k_le_gradient_ms k_le_forward k_path_gradient k_prefix}; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-1} -c 1 \
      -o gpurun_out/prof_${TAG}_$k $CMD > gpurun_out/ncu_full_${TAG}_$k.log 2>&1
done
echo profile done
