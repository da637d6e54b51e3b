#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in 38273024 38273048 38273056 38289408; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p31_variants.jsonl 2>> $out/p31_variants.err
done
QG_KW="dict(kernel_cfg=6)" timeout 300 python tools/jit_time.py 32 random >> $out/p31_variants.jsonl 2>> $out/p31_variants.err
QG_KW="dict(kernel_cfg=9)" timeout 300 python tools/jit_time.py 32 random >> $out/p31_variants.jsonl 2>> $out/p31_variants.err
timeout 1200 ncu --set full --clock-control none -k regex:qg_jit_pass -s 30 -c 1 -o $out/p31_jit32 python tools/jit_time.py 32 random > $out/p31_ncu.log 2>&1
echo done
