#!/bin/bash
# A/B/C: the G = 1 fused RS + AdamW (a) on the compute stream (default), (b) on the high-priority RS stream
# capped at 1 CTA per SM so each SM keeps room for a GEMM CTA beside it, (c) the same on the low-priority stream.
mkdir -p gpurun_out
B="python bench.py --steps 15 --warmup 3 --no-cpu-baseline --no-zero3 --tau-variant -1 --no-e2e"
for i in 1 2; do
  timeout 300 $B > gpurun_out/bg_comp_$i.log 2>&1
  FCDP_OPT_STREAM=rs FCDP_OPT_CTAS_PER_SM=1 timeout 300 $B > gpurun_out/bg_rs1_$i.log 2>&1
  FCDP_OPT_PRIO=low FCDP_OPT_CTAS_PER_SM=1 timeout 300 $B > gpurun_out/bg_low1_$i.log 2>&1
  FCDP_OPT_STREAM=rs FCDP_OPT_CTAS_PER_SM=2 timeout 300 $B > gpurun_out/bg_rs2_$i.log 2>&1
done
