mkdir -p gpurun_out
bash scripts/variants_lib.sh 1e8 "" new f64 f96 new f64 f96 > gpurun_out/s45_ab.txt 2>&1
echo done
