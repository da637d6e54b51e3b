#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in 0 524288; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p7_variants.jsonl 2>> $out/p7_variants.err
  QG_KW="dict(kernel_cfg=7)" QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p7_variants.jsonl 2>> $out/p7_variants.err
done
QG_KW="dict(low_qubits=6)" QG_JIT_VARIANT=524288 timeout 300 python tools/jit_time.py 32 random >> $out/p7_variants.jsonl 2>> $out/p7_variants.err
QG_KW="dict(kernel_cfg=7)" QG_JIT_VARIANT=32 timeout 300 python tools/jit_time.py 32 random >> $out/p7_variants.jsonl 2>> $out/p7_variants.err
QG_KW="dict(kernel_cfg=7)" QG_JIT_VARIANT=24 timeout 300 python tools/jit_time.py 32 random >> $out/p7_variants.jsonl 2>> $out/p7_variants.err
QG_CFGS="[dict(), dict(kernel_cfg=1), dict(kernel_cfg=2)]" QG_PREC=fp64 timeout 600 python tools/probe_cfg.py 30 >> $out/p7_c128.jsonl 2>&1
echo done
