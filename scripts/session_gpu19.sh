mkdir -p gpurun_out
export W=2
SKIP=1 KERNELS="k_le_gradient_ms k_path_gradient" timeout 2400 bash scripts/profile_kernels.sh r12 1e8 > gpurun_out/s19_profile.log 2>&1
for k in k_le_forward k_prefix; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_r12_$k python bench.py --paths 1e8 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_r12_$k.log 2>&1
done
timeout 600 python bench.py > gpurun_out/s19_bench_b.log 2>&1
timeout 600 python bench.py --config c --steps 3 --warmup 3 --no-e2e > gpurun_out/s19_bench_c.log 2>&1
timeout 900 python bench.py --config e --steps 3 --warmup 3 --no-e2e > gpurun_out/s19_bench_e.log 2>&1
timeout 300 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/s19_ref.log 2>&1
echo done
