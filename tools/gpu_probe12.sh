#!/bin/bash
out=gpurun_out; mkdir -p $out
for c in c1 c2; do timeout 600 python tools/bench_configs.py $c > $out/p12_cfg_$c.json 2> $out/p12_cfg_$c.err; done
timeout 900 python tools/bench_configs.py c4 --images 2 > $out/p12_cfg_c4.json 2> $out/p12_cfg_c4.err
timeout 900 python -m pytest tests/test_gpu_parity.py -k qft28 -x -q > $out/p12_tests.log 2>&1; echo "pytest rc=$?" >> $out/p12_tests.log
echo done
