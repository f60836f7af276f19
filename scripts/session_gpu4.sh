mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4_pytest.log 2>&1; echo pytest=$? >> gpurun_out/s4_pytest.log
timeout 600 python bench.py > gpurun_out/s4_bench_b.log 2>&1
for p in 1.25e7 2.5e7 5e7; do timeout 300 python bench.py --paths $p --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s4_shard_$p.log 2>&1; done
timeout 900 python bench.py --config e --steps 3 --warmup 3 --no-e2e > gpurun_out/s4_bench_e.log 2>&1
KERNELS=k_le_gradient_ms timeout 1500 bash scripts/profile_kernels.sh r11 1e8 > gpurun_out/s4_profile.log 2>&1
echo done
