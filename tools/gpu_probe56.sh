#!/bin/bash
out=gpurun_out; mkdir -p $out
QG_DEV_JIT_CFG0=1 timeout 300 python tools/cfg0_check.py > $out/p56_check.txt 2>&1
QG_DEV_JIT_CFG0=1 QG_KW="dict(kernel_cfg=1)" timeout 300 python tools/jit_time.py 32 random >> $out/p56.jsonl 2>> $out/p56.err
QG_DEV_JIT_CFG0=1 QG_KW="dict(kernel_cfg=1)" QG_JIT_VARIANT=38273048 timeout 300 python tools/jit_time.py 32 random >> $out/p56.jsonl 2>> $out/p56.err
QG_DEV_JIT_CFG0=1 QG_KW="dict(kernel_cfg=1)" QG_JIT_VARIANT=38273056 timeout 300 python tools/jit_time.py 32 random >> $out/p56.jsonl 2>> $out/p56.err
QG_DEV_JIT_CFG0=1 QG_KW="dict(kernel_cfg=1)" timeout 300 python tools/jit_time.py 28 qft >> $out/p56.jsonl 2>> $out/p56.err
echo done
