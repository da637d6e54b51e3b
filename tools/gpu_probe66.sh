#!/bin/bash
# r02i: phase-run merging (JIT variant 16777216) vs the default: time per circuit and accuracy vs the interpreter
out=gpurun_out; mkdir -p $out
D=38273024
for v in $D $((D | 16777216)) $D $((D | 16777216)); do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/r02i_phrun.jsonl 2>> $out/r02i_phrun.err
done
QG_JIT_VARIANT=$((D | 16777216)) timeout 300 python tools/jit_time.py 28 qft >> $out/r02i_phrun.jsonl 2>> $out/r02i_phrun.err
QG_JIT_VARIANT=$D timeout 300 python tools/jit_time.py 28 qft >> $out/r02i_phrun.jsonl 2>> $out/r02i_phrun.err
QG_JIT_VARIANT=$((D | 16777216)) timeout 600 python tools/jit_check.py 22 26 > $out/r02i_phrun_check.log 2>&1
echo done
