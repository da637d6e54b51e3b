#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in 38273024 172490752 38338560; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p26_variants.jsonl 2>> $out/p26_variants.err
done
echo done
