#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 900 python tools/jit_check128.py 24 28 30 > $out/p29_check128.log 2>&1
timeout 900 python -m pytest tests/test_gpu_jit.py -x -q -k "complex128 or bitexact or interp" > $out/p29_tests.log 2>&1; echo "pytest rc=$?" >> $out/p29_tests.log
timeout 600 python tools/jit_check.py 28 > $out/p29_check64.log 2>&1
echo done
