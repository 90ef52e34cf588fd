#!/bin/bash
# A/B: the N > 1 reduce-scatter with its full grid vs capped at 1 / 2 CTAs per SM (beside the backward GEMMs).
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out
B="bench.py --steps 8 --warmup 3 --no-zero3 --tau-variant -1 --no-e2e --no-cpu-baseline"
for cap in 0 1 2; do
  CUDA_VISIBLE_DEVICES=0,1 FCDP_RS_CTAS_PER_SM=$cap timeout 400 $TR --nproc-per-node 2 --master-port 2960$cap $B --gpus 2 > gpurun_out/rscap_n2_$cap.log 2>&1
  FCDP_RS_CTAS_PER_SM=$cap timeout 400 $TR --nproc-per-node 4 --master-port 2961$cap $B --gpus 4 > gpurun_out/rscap_n4_$cap.log 2>&1
done
