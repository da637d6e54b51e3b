#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 600 python tools/probe_tree.py > $out/p15_tree.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tree_sampler.py -x -q > $out/p15_tests.log 2>&1; echo "pytest rc=$?" >> $out/p15_tests.log
timeout 900 python tools/bench_configs.py c4 --images 2 > $out/p15_cfg_c4.json 2> $out/p15_cfg_c4.err
echo done
