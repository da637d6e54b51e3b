#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_large.py -x -q -m gpu > $out/p64_tests.log 2>&1; echo "rc=$?" >> $out/p64_tests.log
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 3 > $out/p64_bench.json 2> $out/p64.err
echo done
