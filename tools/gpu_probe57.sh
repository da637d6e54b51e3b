#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in 38273024 38273048 38273056; do
QG_DEV_JIT_CFG0=1 QG_KW="dict(kernel_cfg=2)" QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p57.jsonl 2>> $out/p57.err
done
echo done
