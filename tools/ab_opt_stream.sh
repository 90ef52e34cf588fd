#!/bin/bash
# A/B (historical): the G = 1 fused RS + AdamW on the high-priority RS stream vs serialised on the compute stream
# (now the default; FCDP_OPT_STREAM=rs selects the side stream).
mkdir -p gpurun_out
B="python bench.py --steps 15 --warmup 3 --no-cpu-baseline --no-zero3 --tau-variant -1 --no-e2e"
for i in 1 2; do
  FCDP_OPT_STREAM=rs timeout 300 $B > gpurun_out/ab_side_$i.log 2>&1
  FCDP_OPT_STREAM=compute timeout 300 $B > gpurun_out/ab_comp_$i.log 2>&1
done
