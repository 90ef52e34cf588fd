#!/bin/bash
# Config C5 refresh at the round-2 HEAD on 4 GPUs (2x2): inter-node bandwidth sweep, FCDP vs ZeRO-3 (GPT-2 1.3B)
# and FCDP-Comm vs ZeRO-3 (Llama-7B LoRA r=16).
mkdir -p gpurun_out
python tools/sweep.py --gpus 4 --topologies 2x2 --preset-model gpt2-1.3b --batch 8 --strategies fcdp,zero3 \
  --presets ib100-rdma-measured,eth100g-theoretical,ib100-ipoib-measured,eth10g-measured \
  --out gpurun_out/sweep_gpt2_r02.jsonl --per-run-timeout 400 > gpurun_out/sweep_gpt2.log 2>&1
python tools/sweep.py --gpus 4 --topologies 2x2 --preset-model llama7b-lora16 --batch 2 --strategies fcdp-comm \
  --presets ib100-rdma-measured,eth100g-theoretical,ib100-ipoib-measured,eth10g-measured,eth1g-measured \
  --out gpurun_out/sweep_c3_r02.jsonl --per-run-timeout 500 > gpurun_out/sweep_c3.log 2>&1
python tools/sweep.py --gpus 4 --topologies 2x2 --preset-model llama7b-lora16 --batch 2 --strategies zero3 \
  --presets ib100-rdma-measured,eth10g-measured \
  --out gpurun_out/sweep_c3_r02.jsonl --per-run-timeout 600 >> gpurun_out/sweep_c3.log 2>&1
echo sweep-done
