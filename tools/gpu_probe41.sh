#!/bin/bash
# decomposition probes at the real kernel's occupancy (QG_DEV_OCC=2), il = store/load interleave
out=gpurun_out; mkdir -p $out
for occ in 2 0; do
for v in 38273024 38273048 38273056 575143936 575143960 575144064 575144088 575143968; do
  QG_DEV_OCC=$occ QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random | sed "s/^{/{\"occ\": $occ, /" >> $out/p41.jsonl 2>> $out/p41.err
done
for v in 38273024 575143936 575144064; do
  QG_DEV_OCC=$occ QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 28 qft | sed "s/^{/{\"occ\": $occ, /" >> $out/p41.jsonl 2>> $out/p41.err
done
done
echo done
