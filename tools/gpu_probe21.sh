#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in 4718592 4718848 4719104 4719360; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p21_variants.jsonl 2>> $out/p21_variants.err
done
echo done
