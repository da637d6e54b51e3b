#!/bin/bash
out=gpurun_out; mkdir -p $out
for b in 0 1; do
for v in 38273024 38273048; do
  QG_DEV_TILE_LOWBIAS=$b QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random | sed "s/^{/{\"lowbias\": $b, /" >> $out/p32_variants.jsonl 2>> $out/p32_variants.err
done
done
echo done
