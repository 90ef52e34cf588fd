#!/bin/bash
# NIC bandwidth profiles (Fig. 10) at 2x1, then N = 4 bench lines (GPT-2 1.3B, C3) after the driving-model kernels.
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0,1 timeout 600 $TR --nproc-per-node 2 --master-port 29571 tools/nic_profile.py --preset gpt2-1.3b --strategies zero3,fcdp > gpurun_out/nicprof_gpt2.json 2> gpurun_out/nicprof_gpt2.log; echo nic1 rc=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29572 tools/nic_profile.py --preset llama7b-lora16 --batch 2 --strategies zero3,fcdp,fcdp-comm > gpurun_out/nicprof_c3.json 2> gpurun_out/nicprof_c3.log; echo nic2 rc=$?
timeout 800 $TR --nproc-per-node 4 --master-port 29573 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_n4b.log 2>&1; echo n4 rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29574 bench.py --gpus 4 --preset llama7b-lora16 --strategy fcdp-comm --batch 2 --steps 4 --warmup 3 --zero3-steps 2 --no-e2e > gpurun_out/c3_n4b.log 2>&1; echo c3n4 rc=$?
