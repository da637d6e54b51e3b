#!/bin/bash
# r02m: real-scale thread-phase fast path: bit-exact / parity tests and A/B timing (complex64 and complex128)
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_jit.py tests/test_gpu_parity.py -x -q -m gpu > $out/r02n_tests.log 2>&1; echo "rc=$?" >> $out/r02n_tests.log
for i in 1 2; do
  timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"lib": "realscale", /' >> $out/r02n_ab.jsonl 2>> $out/r02n_ab.err
  QG_LIB_PATH=$PWD/ref_lib_ab.so timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"lib": "cmul", /' >> $out/r02n_ab.jsonl 2>> $out/r02n_ab.err
done
timeout 900 python bench.py --precision fp64 --no-cpu-baseline --no-e2e > $out/r02n_bench_c128.json 2> $out/r02n_bench_c128.err
QG_LIB_PATH=$PWD/ref_lib_ab.so timeout 900 python bench.py --precision fp64 --no-cpu-baseline --no-e2e > $out/r02n_bench_c128_ref.json 2> $out/r02n_bench_c128_ref.err
echo done
