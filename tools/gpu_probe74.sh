#!/bin/bash
# r02k: scaled two-FMA rotations (complex64): parity / bit-exact tests and A/B timing vs the previous library
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_jit.py tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -m gpu > $out/r02k_scaled_tests.log 2>&1; echo "rc=$?" >> $out/r02k_scaled_tests.log
for i in 1 2; do
  timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"lib": "scaled", /' >> $out/r02k_scaled.jsonl 2>> $out/r02k_scaled.err
  QG_LIB_PATH=$PWD/old_lib_ab.so timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"lib": "shears", /' >> $out/r02k_scaled.jsonl 2>> $out/r02k_scaled.err
done
timeout 300 python tools/jit_time.py 28 qft | sed 's/^{/{"lib": "scaled", /' >> $out/r02k_scaled.jsonl 2>> $out/r02k_scaled.err
echo done
