#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in 524288 524320 524312; do
  QG_KW="dict(kernel_cfg=9)" QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p8_variants.jsonl 2>> $out/p8_variants.err
done
QG_KW="dict(kernel_cfg=8)" QG_JIT_VARIANT=524288 timeout 300 python tools/jit_time.py 32 random >> $out/p8_variants.jsonl 2>> $out/p8_variants.err
QG_KW="dict(kernel_cfg=9)" QG_JIT_VARIANT=524288 timeout 300 python tools/jit_time.py 28 qft >> $out/p8_variants.jsonl 2>> $out/p8_variants.err
echo done
