mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s41_pytest.log 2>&1; echo pytest=$? >> gpurun_out/s41_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s41_smoke.log 2>&1
bash scripts/variants_lib.sh 1e8 "" fwd256 new fwd256 new > gpurun_out/s41_ab.txt 2>&1
bash scripts/variants_lib.sh 1e8 "--config c" fwd256 new >> gpurun_out/s41_ab.txt 2>&1
bash scripts/variants_lib.sh 1e7 "--config d" fwd256 new >> gpurun_out/s41_ab.txt 2>&1
bash scripts/variants_lib.sh 1e6 "--config a" fwd256 new >> gpurun_out/s41_ab.txt 2>&1
timeout 600 python bench.py > gpurun_out/s41_bench_b.log 2>&1
echo done
