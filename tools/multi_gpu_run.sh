#!/bin/bash
# N = 2 / 4 bench lines (GPT-2 1.3B with ZeRO++ and MiCS beside FCDP), the N = 4 reference arm and config C4.
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 700 $TR --nproc-per-node 2 --master-port 29551 bench.py --gpus 2 --steps 10 --warmup 3 --zeropp --mics > gpurun_out/bench_n2.log 2>&1; echo n2 rc=$?
timeout 800 $TR --nproc-per-node 4 --master-port 29552 bench.py --gpus 4 --steps 10 --warmup 3 --zeropp --mics > gpurun_out/bench_n4.log 2>&1; echo n4 rc=$?
timeout 300 $TR --nproc-per-node 4 --master-port 29553 bench.py --impl reference --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_ref_n4.log 2>&1; echo ref4 rc=$?
timeout 1200 $TR --nproc-per-node 4 --master-port 29562 bench.py --gpus 4 --preset llama13b --strategy fcdp --batch 0 --steps 3 --warmup 3 --zero3-steps 2 --tau-variant 0 --no-e2e > gpurun_out/c4_n4.log 2>&1; echo c4_n4 rc=$?
