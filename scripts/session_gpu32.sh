mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s32_pytest.log 2>&1; echo pytest=$? >> gpurun_out/s32_pytest.log
bash scripts/variants_lib.sh 1e7 "--config d" base scache > gpurun_out/s32_ab.txt 2>&1
bash scripts/variants_lib.sh 1e8 "" base scache >> gpurun_out/s32_ab.txt 2>&1
for c in 8 16 32 64; do
  timeout 300 python bench.py --config a --no-e2e --no-cpu-baseline --grad-copies $c > gpurun_out/s32_a_$c.log 2>&1
  python scripts/summarize_bench.py gpurun_out/s32_a_$c.log a_copies$c >> gpurun_out/s32_ab.txt
done
echo done
