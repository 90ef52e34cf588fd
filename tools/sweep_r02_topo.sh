#!/bin/bash
# Config C5, topology axis at the round-2 HEAD on 4 GPUs: 1x4 and 4x1 emulated nodes (2x2 in tools/sweep_r02.sh),
# FCDP vs ZeRO-3 (GPT-2 1.3B) at two inter-node bandwidths; NIC profile at 2x2.
mkdir -p gpurun_out
python tools/sweep.py --gpus 4 --topologies 1x4,4x1 --preset-model gpt2-1.3b --batch 8 --strategies fcdp,zero3 \
  --presets ib100-rdma-measured,eth10g-measured --out gpurun_out/sweep_topo_r02.jsonl --per-run-timeout 500 \
  > gpurun_out/sweep_topo.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4 --master-port 29681 \
  tools/nic_profile.py --preset gpt2-1.3b --strategies zero3,fcdp > gpurun_out/nicprof_gpt2_2x2.json 2> gpurun_out/nicprof_gpt2_2x2.log
echo done
