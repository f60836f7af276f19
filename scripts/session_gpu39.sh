mkdir -p gpurun_out
timeout 1200 python bench.py --config e --steps 3 --warmup 3 --no-e2e > gpurun_out/s39_bench_e.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/s39_torchrun1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 1 --warmup 1 > gpurun_out/s39_torchrun1_ref.log 2>&1
echo done
