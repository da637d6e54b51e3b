#!/bin/bash
# r02k final: GPU tests, smoke, default bench, reference arm, e2e breakdown (planner early exit)
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/r02k_gpu_tests.log 2>&1; echo "pytest rc=$?" >> $out/r02k_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/r02k_smoke.log 2>&1; echo "smoke rc=$?" >> $out/r02k_smoke.log
timeout 900 python bench.py > $out/r02k_bench.json 2> $out/r02k_bench.err; echo "bench rc=$?" >> $out/r02k_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/r02k_bench_ref.json 2> $out/r02k_bench_ref.err
timeout 600 python tools/e2e_breakdown.py > $out/r02k_e2e_breakdown.jsonl 2>&1
echo done
