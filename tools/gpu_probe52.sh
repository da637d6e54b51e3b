#!/bin/bash
# producer/consumer pass kernels (QG_JIT_PC=1): bit-exactness, then time
out=gpurun_out; mkdir -p $out
QG_JIT_PC=1 timeout 300 python tools/jit_check.py 24 > $out/p52_check.txt 2>&1; echo "rc=$?" >> $out/p52_check.txt
QG_JIT_PC=1 timeout 300 python tools/jit_check.py 28 >> $out/p52_check.txt 2>&1; echo "rc=$?" >> $out/p52_check.txt
QG_JIT_PC=1 timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"pc": 1, /' >> $out/p52.jsonl 2>> $out/p52.err
QG_JIT_PC=1 QG_JIT_VARIANT=38273048 timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"pc": 1, /' >> $out/p52.jsonl 2>> $out/p52.err
QG_JIT_PC=1 QG_JIT_VARIANT=38273056 timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"pc": 1, /' >> $out/p52.jsonl 2>> $out/p52.err
timeout 300 python tools/jit_time.py 32 random >> $out/p52.jsonl 2>> $out/p52.err
echo done
