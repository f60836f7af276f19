#!/bin/bash
# Profiling recipe (run under gpurun): plain run, launch list, full capture of K4/K5,
# and warp-execution efficiency of the unsorted vs B-sorted store.
set -u
mkdir -p gpurun_out
TAG=${1:-r1}
P=${2:-1e6}
CMD="python bench.py --paths $P --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_gradient" -s 2 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
M=smsp__thread_inst_executed_per_inst_executed.ratio,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__warps_active.avg.pct_of_peak_sustained_active
$CMD --no-sort > gpurun_out/plain_unsorted_$TAG.log 2>&1 && \
ncu --metrics $M --clock-control none --csv -k regex:"k_forward|k_gradient" -s 2 -c 2 --log-file gpurun_out/warp_eff_unsorted_$TAG.csv $CMD --no-sort > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv -k regex:"k_forward|k_gradient" -s 2 -c 2 --log-file gpurun_out/warp_eff_sorted_$TAG.csv $CMD > /dev/null 2>&1
echo profile done
