#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_jit.py -x -q > $out/p24_tests.log 2>&1; echo "pytest rc=$?" >> $out/p24_tests.log
timeout 600 python tools/bench_configs.py c2 > $out/p24_cfg_c2.json 2> $out/p24_cfg_c2.err
echo done
