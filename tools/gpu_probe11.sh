#!/bin/bash
out=gpurun_out; mkdir -p $out
for v in 524288 2621440; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p11_variants.jsonl 2>> $out/p11_variants.err
done
timeout 1500 python -m pytest tests -m gpu -x -q > $out/p11_tests.log 2>&1; echo "pytest rc=$?" >> $out/p11_tests.log
timeout 900 python bench.py > $out/p11_bench.json 2> $out/p11_bench.err; echo "bench rc=$?" >> $out/p11_bench.err
echo done
