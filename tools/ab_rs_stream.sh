#!/bin/bash
# A/B: the G > 1 reduce-scatter on its own high-priority stream (default) vs serialised on the compute stream
# (FCDP_RS_STREAM=compute): step time and the RS kernel's live rate at 2x1 and 2x2; engine parity with the option.
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out
FCDP_RS_STREAM=compute timeout 900 python -m pytest tests/test_engine_gpu.py -x -q -p no:cacheprovider -k "parity and (2-1 or 2-2 or 1-2 or 4-1)" > gpurun_out/rsstream_tests.log 2>&1; echo tests rc=$? >> gpurun_out/rsstream_tests.log
B="bench.py --steps 8 --warmup 3 --no-zero3 --tau-variant -1 --no-e2e --no-cpu-baseline"
for i in 1 2; do
  for mode in rs compute; do
    CUDA_VISIBLE_DEVICES=0,1 FCDP_RS_STREAM=$mode timeout 400 $TR --nproc-per-node 2 --master-port 2970$i $B --gpus 2 > gpurun_out/rsstream_n2_${mode}_$i.log 2>&1
    FCDP_RS_STREAM=$mode timeout 400 $TR --nproc-per-node 4 --master-port 2971$i $B --gpus 4 > gpurun_out/rsstream_n4_${mode}_$i.log 2>&1
  done
done
