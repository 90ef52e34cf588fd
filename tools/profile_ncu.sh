#!/bin/bash
# ncu evidence for profiles/ (run under gpurun on ONE GPU):
#   1. the plain command must exit 0 first;
#   2. launch list (every kernel, device time, cold-cache/serialised -> compare shares);
#   3. --set full on the engine's kernels (one launch each of the top classes).
set -e
CMD="python bench.py --steps 2 --warmup 1 --no-zero3 --no-cpu-baseline --no-e2e --watchdog 900 ${BENCH_ARGS}"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"adam_kernel|concat_kernel|expand_kernel|rs_dense_kernel|rs_masked_kernel|rs_finalize_kernel|copy_kernel" \
    -s 20 -c 6 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo profile-done
