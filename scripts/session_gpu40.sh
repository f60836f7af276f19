mkdir -p gpurun_out
bash scripts/variants_lib.sh 1e8 "" base wf128 wf512 wf128m7 base wf128 > gpurun_out/s40_ab.txt 2>&1
echo done
