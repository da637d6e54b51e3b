#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in 0 16384 32768 65536 131072 196608 4; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p4_variants.jsonl 2>> $out/p4_variants.err
done
for v in 0 16384 32768; do
  QG_KW="dict(kernel_cfg=6)" QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p4_variants.jsonl 2>> $out/p4_variants.err
done
timeout 600 python -m pytest tests/test_gpu_tree_sampler.py tests/test_gpu_distributed.py tests/test_bench_suite.py -x -q > $out/p4_tests.log 2>&1; echo "pytest rc=$?" >> $out/p4_tests.log
echo done
