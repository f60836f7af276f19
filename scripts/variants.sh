#!/bin/bash
# Timing sweep of kernel mappings (no profiler).  Usage: scripts/variants.sh PATHS "variant1" "variant2" ...
P=${1:-1e7}; shift
mkdir -p gpurun_out
for v in "$@"; do
  tag=$(echo "$v" | tr -d ' -')
  timeout 900 python bench.py --paths $P --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $v > gpurun_out/var_${P}_$tag.log 2>&1
  python scripts/summarize_bench.py "gpurun_out/var_${P}_$tag.log" "$tag"
done
