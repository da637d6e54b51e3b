#!/bin/bash
# r02i: does decoupling the warps at the transposes pay? (timing probes, wrong results)
out=gpurun_out; mkdir -p $out
D=38273024
for v in $D $((D | 67108864)) $((D | 16)) $D $((D | 67108864)); do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/r02i_warpsync.jsonl 2>> $out/r02i_warpsync.err
done
echo done
