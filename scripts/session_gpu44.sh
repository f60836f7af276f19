mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s44_pytest.log 2>&1; echo pytest=$? >> gpurun_out/s44_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s44_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s44_bench_b.log 2>&1
timeout 600 python bench.py --config c --steps 3 --warmup 3 --no-e2e > gpurun_out/s44_bench_c.log 2>&1
timeout 600 python bench.py --config a --no-e2e > gpurun_out/s44_bench_a.log 2>&1
timeout 600 python bench.py --config d --no-e2e > gpurun_out/s44_bench_d.log 2>&1
export W=2
SKIP=1 KERNELS="k_le_forward" timeout 1800 bash scripts/profile_kernels.sh r15b 1e8 > gpurun_out/s44_profile.log 2>&1
echo done
