#!/bin/bash
out=gpurun_out; mkdir -p $out
QG_JIT_VARIANT=1649082496 timeout 600 python tools/jit_check.py 24 28 > $out/p46_check.txt 2>&1
QG_JIT_VARIANT=1648885760 timeout 600 python tools/jit_check.py 26 >> $out/p46_check.txt 2>&1
for v in 1649082496 1648885760 1649082368 1112014848 38273024 1649082520 1649082528; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p46.jsonl 2>> $out/p46.err
done
for v in 38273024 1649082496 1648885760; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 28 qft >> $out/p46.jsonl 2>> $out/p46.err
done
echo done
