#!/bin/bash
# store/load interleave (variant 536870912) with and without the L2 prefetch (128 = off)
out=gpurun_out; mkdir -p $out
QG_JIT_VARIANT=575143936 timeout 600 python tools/jit_check.py 20 24 28 > $out/p37_check.txt 2>&1
for v in 38273024 575143936 575144064 575143960 575144088 38273152; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p37.jsonl 2>> $out/p37.err
done
for v in 38273024 575143936 575144064; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 28 qft >> $out/p37.jsonl 2>> $out/p37.err
done
echo done
