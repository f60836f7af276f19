mkdir -p gpurun_out
bash scripts/variants_lib.sh 1e8 "" base rot > gpurun_out/s9_ab.txt 2>&1
bash scripts/variants.sh 1e8 "--spread 16" "--spread 32" "--spread 128" >> gpurun_out/s9_ab.txt 2>&1
for c in 4 16 64; do timeout 300 python bench.py --config a --grad-copies $c --no-cpu-baseline --no-e2e > gpurun_out/s9_a_c$c.log 2>&1; python scripts/summarize_bench.py gpurun_out/s9_a_c$c.log a_copies$c >> gpurun_out/s9_ab.txt; done
echo done
