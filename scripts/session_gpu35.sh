mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s35_pytest.log 2>&1; echo pytest=$? >> gpurun_out/s35_pytest.log
bash scripts/variants_lib.sh 1e7 "--config d" scache3 scache4 base > gpurun_out/s35_ab.txt 2>&1
bash scripts/variants_lib.sh 1e8 "" base scache4 base scache4 >> gpurun_out/s35_ab.txt 2>&1
echo done
