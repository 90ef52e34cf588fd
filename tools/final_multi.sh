#!/bin/bash
# Round-2 closing run on 4 GPUs: N = 2 and N = 4 bench lines (GPT-2 1.3B, ZeRO++ / MiCS beside) and the reference arm.
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0,1 timeout 700 $TR --nproc-per-node 2 --master-port 29651 bench.py --gpus 2 --steps 10 --warmup 3 --zeropp --mics > gpurun_out/fin_n2.log 2>&1; echo n2 rc=$?
timeout 800 $TR --nproc-per-node 4 --master-port 29652 bench.py --gpus 4 --steps 10 --warmup 3 --zeropp --mics > gpurun_out/fin_n4.log 2>&1; echo n4 rc=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR --nproc-per-node 2 --master-port 29653 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/fin_ref_n2.log 2>&1; echo ref2 rc=$?
timeout 300 $TR --nproc-per-node 4 --master-port 29654 bench.py --impl reference --gpus 4 --steps 3 --warmup 3 > gpurun_out/fin_ref_n4.log 2>&1; echo ref4 rc=$?
