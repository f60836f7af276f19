mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s5_pytest.log 2>&1; echo pytest=$? >> gpurun_out/s5_pytest.log
bash scripts/variants_lib.sh 1e8 "" base rep2 rep4 > gpurun_out/s5_ab.txt 2>&1
timeout 900 python bench.py --config e --steps 3 --warmup 3 --no-e2e > gpurun_out/s5_bench_e.log 2>&1
echo done
