#!/bin/bash
# r02 session-3 first GPU call: suite, bench, JIT variant split (compute vs memory), tile-layout bandwidth.
out=gpurun_out; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $out/p1_gpu.txt 2>&1
timeout 900 python bench.py > $out/p1_bench.json 2> $out/p1_bench.err; echo "bench rc=$?" >> $out/p1_bench.err
for v in 0 1 8 16 24 32 40 56 128; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p1_variants.jsonl 2>> $out/p1_variants.err
done
QG_JIT_VARIANT=0 timeout 300 python tools/jit_time.py 28 qft >> $out/p1_variants.jsonl 2>> $out/p1_variants.err
QG_JIT_VARIANT=8 timeout 300 python tools/jit_time.py 28 qft >> $out/p1_variants.jsonl 2>> $out/p1_variants.err
timeout 600 python tools/bw_probe.py > $out/p1_bw.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $out/p1_tests.log 2>&1; echo "pytest rc=$?" >> $out/p1_tests.log
echo done
