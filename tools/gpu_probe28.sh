#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 2400 python -m pytest tests -m gpu -x -q > $out/p28_tests.log 2>&1; echo "pytest rc=$?" >> $out/p28_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/p28_smoke.log 2>&1; echo "smoke rc=$?" >> $out/p28_smoke.log
timeout 900 python bench.py > $out/p28_bench.json 2> $out/p28_bench.err; echo "bench rc=$?" >> $out/p28_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $out/p28_bench_ref.json 2> $out/p28_bench_ref.err
timeout 900 python tools/jit_check128.py 30 > $out/p28_check128.log 2>&1
echo done
