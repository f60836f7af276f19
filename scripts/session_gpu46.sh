mkdir -p gpurun_out
bash scripts/variants_lib.sh 1e8 "" new cw new cw > gpurun_out/s46_ab.txt 2>&1
bash scripts/variants_lib.sh 1e8 "--grad-copies 4" new cw >> gpurun_out/s46_ab.txt 2>&1
bash scripts/variants_lib.sh 1e8 "--config c" new cw >> gpurun_out/s46_ab.txt 2>&1
echo done
