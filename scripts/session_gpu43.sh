mkdir -p gpurun_out
bash scripts/variants_lib.sh 1e8 "" new gp64 g32 p32 new gp64 g32 p32 > gpurun_out/s43_ab.txt 2>&1
bash scripts/variants_lib.sh 1e8 "--config c" new gp64 >> gpurun_out/s43_ab.txt 2>&1
bash scripts/variants_lib.sh 1e7 "--config d" new gp64 >> gpurun_out/s43_ab.txt 2>&1
bash scripts/variants_lib.sh 1e6 "--config a" new gp64 >> gpurun_out/s43_ab.txt 2>&1
echo done
