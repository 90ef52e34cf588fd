#!/bin/bash
# Full GPU suite with the ranks of the multi-rank cases spread over 4 real GPUs (NVLink peers), then N = 2 bench.
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests_4gpu.log 2>&1; echo tests rc=$? | tee -a gpurun_out/gputests_4gpu.log
CUDA_VISIBLE_DEVICES=0,1 timeout 700 $TR --nproc-per-node 2 --master-port 29581 bench.py --gpus 2 --steps 10 --warmup 3 --zeropp --mics > gpurun_out/bench_n2c.log 2>&1; echo n2 rc=$?
