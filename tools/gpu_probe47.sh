#!/bin/bash
out=gpurun_out; mkdir -p $out
QG_JIT_VARIANT=38273025 timeout 600 python tools/jit_check.py 24 > $out/p47_check.txt 2>&1
for v in 38273024 38273025 38273153 38273049 38273057; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p47.jsonl 2>> $out/p47.err
done
echo done
