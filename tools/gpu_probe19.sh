#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 600 python tools/jit_check.py 24 28 > $out/p19_check.log 2>&1
for v in 4718592 4718720; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p19_variants.jsonl 2>> $out/p19_variants.err
done
timeout 300 python tools/jit_time.py 28 qft >> $out/p19_variants.jsonl 2>> $out/p19_variants.err
timeout 1800 python -m pytest tests -m gpu -x -q > $out/p19_tests.log 2>&1; echo "pytest rc=$?" >> $out/p19_tests.log
timeout 900 python bench.py > $out/p19_bench.json 2> $out/p19_bench.err; echo "bench rc=$?" >> $out/p19_bench.err
echo done
