#!/bin/bash
# r02i: variant re-check on the scoped-barrier kernel (interleave, stores through the load mapping, tile searches)
out=gpurun_out; mkdir -p $out
D=38273024
for i in 1 2; do
for v in $D $((D | 536870912)) $((D | 536870912 | 1073741824)); do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/r02i_recheck.jsonl 2>> $out/r02i_recheck.err
done
QG_DEV_TILE_K=8 timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"tile_k": 8, /' >> $out/r02i_recheck.jsonl 2>> $out/r02i_recheck.err
done
echo done
