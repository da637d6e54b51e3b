#!/bin/bash
out=gpurun_out; mkdir -p $out
QG_JIT_VARIANT=4718592 timeout 600 python tools/jit_check.py 24 28 > $out/p18_check_split.log 2>&1
QG_DEV_IOL=2 timeout 600 python tools/jit_check.py 24 28 > $out/p18_check_iol2.log 2>&1
for l in 5 4 3 2; do
for v in 524288 524312 4718592; do
  QG_DEV_IOL=$l QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random | sed "s/^{/{\"iol\": $l, /" >> $out/p18_variants.jsonl 2>> $out/p18_variants.err
done
done
echo done
