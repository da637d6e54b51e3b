#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in 38273024 55050240; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p54.jsonl 2>> $out/p54.err
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 28 qft >> $out/p54.jsonl 2>> $out/p54.err
done
echo done
