#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in 1648885760 1649082496; do
QG_DEV_JIT_CFG0=1 QG_KW="dict(kernel_cfg=2)" QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p58.jsonl 2>> $out/p58.err
QG_DEV_JIT_CFG0=1 QG_KW="dict(kernel_cfg=1)" QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p58.jsonl 2>> $out/p58.err
done
echo done
