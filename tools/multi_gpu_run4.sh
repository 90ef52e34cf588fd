#!/bin/bash
# Functional check of the N = 8 (2x4) bench flow with 2 ranks per GPU on a 4-GPU box (throughput not meaningful),
# the reference arm at N = 8, and the two colsum ncu captures.
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out
timeout 1200 $TR --nproc-per-node 8 --master-port 29591 bench.py --gpus 8 --steps 3 --warmup 3 --zero3-steps 2 > gpurun_out/bench_n8_shared.log 2>&1; echo n8 rc=$?
timeout 600 $TR --nproc-per-node 8 --master-port 29592 bench.py --impl reference --gpus 8 --steps 2 --warmup 1 > gpurun_out/bench_ref_n8.log 2>&1; echo ref8 rc=$?
CMD="python bench.py --steps 2 --warmup 1 --no-zero3 --no-cpu-baseline --no-e2e --tau-variant -1 --watchdog 900"
CUDA_VISIBLE_DEVICES=0 ncu --set full --clock-control none --import-source on -k regex:colsum_partial_kernel -s 41 -c 1 -o gpurun_out/prof_gelu_bwd $CMD > gpurun_out/ncu_full_gelu_bwd.log 2>&1; echo ncu1 rc=$?
CUDA_VISIBLE_DEVICES=0 ncu --set full --clock-control none --import-source on -k regex:colsum_partial_kernel -s 40 -c 1 -o gpurun_out/prof_bias_grad $CMD > gpurun_out/ncu_full_bias_grad.log 2>&1; echo ncu2 rc=$?
