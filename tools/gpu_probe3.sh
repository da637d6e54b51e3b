#!/bin/bash
# register double-buffered JIT tiles (1 CTA/SM) vs the 2-CTA kernel
out=gpurun_out; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_tree_sampler.py tests/test_gpu_distributed.py tests/test_bench_suite.py -x -q > $out/p3_tests.log 2>&1; echo "pytest rc=$?" >> $out/p3_tests.log
for v in 0 2048 2080 4096 4128 12288 12292 12320 8192; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p3_variants.jsonl 2>> $out/p3_variants.err
done
for v in 0 12288; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 28 qft >> $out/p3_variants.jsonl 2>> $out/p3_variants.err
done
echo done
