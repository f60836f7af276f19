mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s50_smoke.log 2>&1
export W=2
KERNELS="" timeout 900 bash scripts/profile_kernels.sh r15c 1e8 > gpurun_out/s50_profile.log 2>&1
echo done
