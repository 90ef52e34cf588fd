#!/bin/bash
# A/B: FCDP-Cache stores at G = 1, tau = 0: all deferred to the LIFO flush at the forward->backward turn
# (FCDP_STORE_EAGER=0) vs the first ones issued eagerly in forward order (default).
mkdir -p gpurun_out
B="python bench.py --tau 0 --tau-variant -1 --steps 15 --warmup 3 --no-cpu-baseline --no-zero3 --no-e2e"
for i in 1 2; do
  FCDP_STORE_EAGER=0 timeout 300 $B > gpurun_out/eager_off_$i.log 2>&1
  timeout 300 $B > gpurun_out/eager_on_$i.log 2>&1
done
