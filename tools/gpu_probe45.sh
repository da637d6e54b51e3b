#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in 1649082520 1112014872 575340696; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p45.jsonl 2>> $out/p45.err
done
echo done
