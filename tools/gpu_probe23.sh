#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_parity.py -x -q > $out/p23_tests.log 2>&1; echo "pytest rc=$?" >> $out/p23_tests.log
timeout 900 python bench.py > $out/p23_bench.json 2> $out/p23_bench.err; echo "bench rc=$?" >> $out/p23_bench.err
echo done
