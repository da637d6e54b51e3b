#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in 4718592 38273024; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 28 qft >> $out/p25_variants.jsonl 2>> $out/p25_variants.err
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 qft >> $out/p25_variants.jsonl 2>> $out/p25_variants.err
done
QG_JIT_VARIANT=38273024 timeout 600 python tools/jit_check.py 24 28 > $out/p25_check.log 2>&1
echo done
