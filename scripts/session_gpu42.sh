mkdir -p gpurun_out
bash scripts/variants_lib.sh 1e8 "" new g64 g256 p64 p256 new g64 p64 > gpurun_out/s42_ab.txt 2>&1
echo done
