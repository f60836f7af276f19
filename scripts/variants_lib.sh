#!/bin/bash
# A/B timing of experiment builds (no profiler).  Usage:
#   scripts/variants_lib.sh PATHS "bench flags" tag1 tag2 ...   (variants/libpathrec_<tag>.so)
P=${1:-1e7}; F=$2; shift 2
mkdir -p gpurun_out
for t in "$@"; do
  PRC_LIB=$PWD/variants/libpathrec_$t.so timeout 900 python bench.py --paths $P --steps 3 --warmup 3 \
      --no-cpu-baseline --no-e2e $F > gpurun_out/varlib_${P}_$t.log 2>&1
  python scripts/summarize_bench.py "gpurun_out/varlib_${P}_$t.log" "$t"
done
