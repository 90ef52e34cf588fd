#!/bin/bash
# Round-2 ncu evidence (ONE GPU, under gpurun):
#   1. the plain command exits 0 first;
#   2. launch list of the N = 1 bench step (every kernel's device time; cold-cache and serialised, so compare shares);
#   3. --set full of the fused RS + AdamW and of the driving-model kernels inside the bench step, one report each.
set -e
CMD="python bench.py --steps 2 --warmup 1 --no-zero3 --no-cpu-baseline --no-e2e --tau-variant -1 --watchdog 900"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
full() {  # name regex skip count
  ncu --set full --clock-control none --import-source on -k regex:"$2" -s "$3" -c "$4" -o "gpurun_out/prof_$1" $CMD \
      > "gpurun_out/ncu_full_$1.log" 2>&1 || echo "ncu $1 failed"
}
full adam 'adam_grad_kernel' 30 2
full gelu_fwd 'bias_gelu_fwd_kernel' 30 1
# colsum_partial_kernel per GPT-2 block backward: <false> fc2 bias, <true> GELU + fc bias, <false> proj, <false> qkv
full gelu_bwd 'colsum_partial_kernel' 41 1
full bias_grad 'colsum_partial_kernel' 40 1
full xent 'xent_(fwd|bwd)_kernel' 2 2
full ln 'ln_(fwd|bwd_dx)_kernel' 60 2
echo profile-done
