mkdir -p gpurun_out
bash scripts/variants_lib.sh 1e8 "" base l1max base l1max > gpurun_out/s37_ab.txt 2>&1
bash scripts/variants_lib.sh 1e8 "--config c" base l1max >> gpurun_out/s37_ab.txt 2>&1
bash scripts/variants_lib.sh 1e6 "--config a" base l1max >> gpurun_out/s37_ab.txt 2>&1
echo done
