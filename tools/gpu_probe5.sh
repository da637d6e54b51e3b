#!/bin/bash
out=gpurun_out; mkdir -p $out
QG_JIT_VARIANT=262144 timeout 600 python tools/jit_check.py 20 24 28 > $out/p5_check.log 2>&1
for v in 262144 262148 264192 262208 0; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p5_variants.jsonl 2>> $out/p5_variants.err
done
QG_JIT_VARIANT=262144 timeout 300 python tools/jit_time.py 28 qft >> $out/p5_variants.jsonl 2>> $out/p5_variants.err
QG_KW="dict(kernel_cfg=6)" QG_JIT_VARIANT=262144 timeout 300 python tools/jit_time.py 32 random >> $out/p5_variants.jsonl 2>> $out/p5_variants.err
cat $out/p4_tests.log | tail -3 > /dev/null
echo done
