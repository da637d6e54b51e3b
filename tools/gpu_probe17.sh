#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 600 python -m pytest tests/test_qcrank.py tests/test_gpu_tree_sampler.py -x -q > $out/p17_tests.log 2>&1; echo "pytest rc=$?" >> $out/p17_tests.log
timeout 600 python tools/bench_configs.py c1 > $out/p17_cfg_c1.json 2> $out/p17_cfg_c1.err
timeout 900 python tools/bench_configs.py c4 --images 2 > $out/p17_cfg_c4.json 2> $out/p17_cfg_c4.err
echo done
