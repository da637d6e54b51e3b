#!/bin/bash
out=gpurun_out; mkdir -p $out
QG_JIT_PC=1 QG_JIT_VARIANT=38273032 timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"pc": 1, /' >> $out/p53.jsonl 2>> $out/p53.err
QG_JIT_VARIANT=38273032 timeout 300 python tools/jit_time.py 32 random >> $out/p53.jsonl 2>> $out/p53.err
QG_JIT_PC=1 timeout 900 ncu --set full --clock-control none -k regex:qg_jit_pass -s 30 -c 1 -o $out/p53_pc python tools/jit_time.py 32 random > $out/p53_ncu.log 2>&1
echo done
