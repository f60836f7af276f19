mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s48_pytest.log 2>&1; echo pytest=$? >> gpurun_out/s48_pytest.log
bash scripts/variants_lib.sh 1e8 "" pg5 pg6 pg7 > gpurun_out/s48_ab.txt 2>&1
bash scripts/variants_lib.sh 1e8 "--config c" pg5 pg6 >> gpurun_out/s48_ab.txt 2>&1
bash scripts/variants_lib.sh 1e7 "--config d" pg5 pg6 >> gpurun_out/s48_ab.txt 2>&1
bash scripts/variants_lib.sh 1e6 "--config a" pg5 pg6 >> gpurun_out/s48_ab.txt 2>&1
timeout 600 python bench.py > gpurun_out/s48_bench_b.log 2>&1
echo done
