#!/bin/bash
# r02q final: complex128 back on shears (C1 latency), complex64 scaled rotations; full suite, smoke, bench, C1, c128
out=gpurun_out; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/r02q_gpu_tests.log 2>&1; echo "pytest rc=$?" >> $out/r02q_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/r02q_smoke.log 2>&1; echo "smoke rc=$?" >> $out/r02q_smoke.log
for i in 1 2 3; do timeout 600 python tools/bench_configs.py c1 >> $out/r02q_cfg_c1.jsonl 2>> $out/r02q_cfg_c1.err; done
timeout 900 python bench.py > $out/r02q_bench.json 2> $out/r02q_bench.err; echo "bench rc=$?" >> $out/r02q_bench.err
timeout 900 python bench.py --precision fp64 --no-cpu-baseline --no-e2e > $out/r02q_bench_c128.json 2> $out/r02q_bench_c128.err
echo done
