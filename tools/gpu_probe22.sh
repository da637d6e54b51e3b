#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 300 python tools/jit_time.py 32 random >> $out/p22_variants.jsonl 2>> $out/p22_variants.err
for v in 13107200 13107224; do
  QG_KW="dict(kernel_cfg=9)" QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p22_variants.jsonl 2>> $out/p22_variants.err
done
QG_JIT_VARIANT=13107200 timeout 300 python tools/jit_time.py 32 random >> $out/p22_variants.jsonl 2>> $out/p22_variants.err
echo done
