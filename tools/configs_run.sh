#!/bin/bash
# BASELINE configs C3 (Llama-7B LoRA, FCDP-Comm) and C4 (Llama-13B, ZeRO-3 max batch) on 1 and 4 GPUs.
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out
timeout 600 python bench.py --preset llama7b-lora16 --strategy fcdp-comm --batch 2 --steps 4 --warmup 3 --zero3-steps 2 --no-cpu-baseline --no-e2e > gpurun_out/c3_n1.log 2>&1; echo c3_n1 rc=$?
timeout 900 $TR --nproc-per-node 4 --master-port 29561 bench.py --gpus 4 --preset llama7b-lora16 --strategy fcdp-comm --batch 2 --steps 4 --warmup 3 --zero3-steps 2 --no-e2e > gpurun_out/c3_n4.log 2>&1; echo c3_n4 rc=$?
timeout 1200 $TR --nproc-per-node 4 --master-port 29562 bench.py --gpus 4 --preset llama13b --strategy fcdp --batch 0 --steps 3 --warmup 3 --zero3-steps 2 --tau-variant 0 --no-e2e > gpurun_out/c4_n4.log 2>&1; echo c4_n4 rc=$?
