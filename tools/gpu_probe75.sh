#!/bin/bash
# r02l: scaled rotations for complex128 too: full GPU suite, smoke, complex128 A/B, default bench
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/r02m_gpu_tests.log 2>&1; echo "pytest rc=$?" >> $out/r02m_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/r02m_smoke.log 2>&1; echo "smoke rc=$?" >> $out/r02m_smoke.log
timeout 900 python bench.py --precision fp64 --no-cpu-baseline --no-e2e > $out/r02m_bench_c128.json 2> $out/r02m_bench_c128.err
QG_LIB_PATH=$PWD/old_lib_ab.so timeout 900 python bench.py --precision fp64 --no-cpu-baseline --no-e2e > $out/r02m_bench_c128_shears.json 2> $out/r02m_bench_c128_shears.err
timeout 900 python bench.py > $out/r02m_bench.json 2> $out/r02m_bench.err; echo "bench rc=$?" >> $out/r02m_bench.err
echo done
