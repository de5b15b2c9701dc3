#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu > gpurun_out/torchrun.log 2>&1
echo "rc=$?" >> gpurun_out/torchrun.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ref_small.log 2>&1
echo "rc=$?" >> gpurun_out/ref_small.log
