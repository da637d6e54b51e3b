#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 900 python bench.py > $out/p30_bench.json 2> $out/p30_bench.err; echo "bench rc=$?" >> $out/p30_bench.err
for v in 38273024 306708480; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p30_variants.jsonl 2>> $out/p30_variants.err
done
timeout 2400 python -m pytest tests -m gpu -x -q > $out/p30_tests.log 2>&1; echo "pytest rc=$?" >> $out/p30_tests.log
timeout 900 python -m paper_2504_03967_b200.bench_suite --workload random --qubits 20..26 --blocks 200 --precision fp32,fp64 --workers 1,2 --reps 3 --csv $out/p30_suite.csv --ext-csv $out/p30_suite_ext.csv --svg $out/p30_suite.svg --check-scaling > $out/p30_suite.log 2>&1; echo "suite rc=$?" >> $out/p30_suite.log
echo done
