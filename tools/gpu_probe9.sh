#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in 524288 1572864 1589248; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p9_variants.jsonl 2>> $out/p9_variants.err
done
for v in 524288 524320 524312; do
  QG_KW="dict(kernel_cfg=1)" QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p9_variants.jsonl 2>> $out/p9_variants.err
done
echo done
