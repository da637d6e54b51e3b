#!/bin/bash
# r02o: interpreter real-scale multiply: bit-exact / parity tests, C1 timing
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_jit.py tests/test_gpu_parity.py -x -q -m gpu > $out/r02p_tests.log 2>&1; echo "rc=$?" >> $out/r02p_tests.log
for i in 1 2 3; do timeout 600 python tools/bench_configs.py c1 >> $out/r02p_cfg_c1.jsonl 2>> $out/r02p_cfg_c1.err; done
echo done
