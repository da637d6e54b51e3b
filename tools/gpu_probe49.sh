#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tree_sampler.py -x -q -m gpu > $out/p49_tests.log 2>&1; echo "pytest rc=$?" >> $out/p49_tests.log
timeout 300 python tools/bench_configs.py c1 > $out/p49_c1.json 2> $out/p49_c1.err
echo done
