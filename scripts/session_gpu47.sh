mkdir -p gpurun_out
bash scripts/variants_lib.sh 1e8 "" new pg6 pg8 pf4 new pg6 pg8 pf4 > gpurun_out/s47_ab.txt 2>&1
echo done
