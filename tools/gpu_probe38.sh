#!/bin/bash
# cache-policy of the tile loads/stores (.cs vs plain) x store/load interleave; memory-only rows end in 24
out=gpurun_out; mkdir -p $out
for v in 38273048 38404120 38338584 38469656 38404096 38338560 38469632 575340544 575275008 575340568; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p38.jsonl 2>> $out/p38.err
done
QG_DEV_IOL=5 QG_JIT_VARIANT=38273048 timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"iol": 5, /' >> $out/p38.jsonl 2>> $out/p38.err
echo done
