#!/bin/bash
out=gpurun_out; mkdir -p $out
for c in 4 3 2; do
for v in 524288 524312; do
  QG_DEV_CLOW=$c QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random | sed "s/^{/{\"clow\": $c, /" >> $out/p10_variants.jsonl 2>> $out/p10_variants.err
done
done
timeout 600 python -m pytest tests/test_gpu_tree_sampler.py -x -q > $out/p10_tests.log 2>&1; echo "pytest rc=$?" >> $out/p10_tests.log
echo done
