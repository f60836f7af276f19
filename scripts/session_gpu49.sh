mkdir -p gpurun_out
bash scripts/variants_lib.sh 1e8 "" new pf6 pf10 pf12 new pf6 pf10 pf12 > gpurun_out/s49_ab.txt 2>&1
echo done
