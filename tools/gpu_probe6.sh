#!/bin/bash
out=gpurun_out; mkdir -p $out
for lq in 7 8 9; do
for v in 0 262144; do
  QG_KW="dict(low_qubits=$lq)" QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p6_variants.jsonl 2>> $out/p6_variants.err
done
done
timeout 900 python -m pytest tests/test_gpu_tree_sampler.py tests/test_gpu_distributed.py tests/test_gpu_partition.py tests/test_gpu_jit.py -x -q > $out/p6_tests.log 2>&1; echo "pytest rc=$?" >> $out/p6_tests.log
echo done
