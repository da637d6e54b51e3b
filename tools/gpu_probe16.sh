#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 600 python -m pytest tests/test_qcrank.py tests/test_gpu_tree_sampler.py -x -q > $out/p16_tests.log 2>&1; echo "pytest rc=$?" >> $out/p16_tests.log
for c in c1 c2; do timeout 600 python tools/bench_configs.py $c > $out/p16_cfg_$c.json 2> $out/p16_cfg_$c.err; done
timeout 900 python tools/bench_configs.py c4 --images 2 > $out/p16_cfg_c4.json 2> $out/p16_cfg_c4.err
timeout 600 python tools/probe_tree.py > $out/p16_tree.log 2>&1
echo done
