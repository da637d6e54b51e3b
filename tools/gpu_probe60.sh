#!/bin/bash
# TMA producer/consumer (QG_JIT_PC=2): bit-exactness, then time (full / no ops)
out=gpurun_out; mkdir -p $out
QG_JIT_PC=2 timeout 300 python tools/jit_check.py 24 > $out/p60_check.txt 2>&1; echo "rc=$?" >> $out/p60_check.txt
QG_JIT_PC=2 timeout 300 python tools/jit_check.py 28 >> $out/p60_check.txt 2>&1; echo "rc=$?" >> $out/p60_check.txt
QG_JIT_PC=2 timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"pc": 2, /' >> $out/p60.jsonl 2>> $out/p60.err
QG_JIT_PC=2 QG_JIT_VARIANT=38273032 timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"pc": 2, /' >> $out/p60.jsonl 2>> $out/p60.err
timeout 300 python tools/jit_time.py 32 random >> $out/p60.jsonl 2>> $out/p60.err
QG_JIT_PC=2 timeout 900 ncu --set full --clock-control none -k regex:qg_jit_pass -s 30 -c 1 -o $out/p60_tma python tools/jit_time.py 32 random > $out/p60_ncu.log 2>&1
echo done
