#!/bin/bash
# store/load interleave x cache policy (131072 plain loads, 65536 plain stores) x prefetch (128 = off)
out=gpurun_out; mkdir -p $out
for v in 575340696 575340672 575340544 575275136 575209600 38273024 38469632 575340704; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p43.jsonl 2>> $out/p43.err
done
for v in 38273024 575340672 575340544; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 28 qft >> $out/p43.jsonl 2>> $out/p43.err
done
echo done
