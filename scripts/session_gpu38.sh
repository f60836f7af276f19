mkdir -p gpurun_out
bash scripts/variants_lib.sh 1e8 "" base stream base stream > gpurun_out/s38_ab.txt 2>&1
bash scripts/variants_lib.sh 1e8 "--grad-copies 4" base stream >> gpurun_out/s38_ab.txt 2>&1
bash scripts/variants_lib.sh 1e8 "--config c" base stream >> gpurun_out/s38_ab.txt 2>&1
bash scripts/variants_lib.sh 1e7 "--config d" base stream >> gpurun_out/s38_ab.txt 2>&1
echo done
