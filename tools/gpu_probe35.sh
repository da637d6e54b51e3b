#!/bin/bash
# three CTAs per SM (80-register cap) vs two, full / memory-only / compute-only
out=gpurun_out; mkdir -p $out
for v in 38273024 46661632 46661656 46661664; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p35.jsonl 2>> $out/p35.err
done
echo done
