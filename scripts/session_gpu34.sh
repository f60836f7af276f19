mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s34_pytest.log 2>&1; echo pytest=$? >> gpurun_out/s34_pytest.log
bash scripts/variants_lib.sh 1e7 "--config d" scache3 > gpurun_out/s34_ab.txt 2>&1
for p in 1 2; do
  timeout 300 python bench.py --config d --no-e2e --no-cpu-baseline --packet $p > gpurun_out/s34_d_p$p.log 2>&1
  python scripts/summarize_bench.py gpurun_out/s34_d_p$p.log d_packet$p >> gpurun_out/s34_ab.txt
done
bash scripts/variants_lib.sh 1e8 "" scache3 >> gpurun_out/s34_ab.txt 2>&1
echo done
