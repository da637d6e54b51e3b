#!/bin/bash
# r02i final: GPU tests, smoke, default bench (after the counts helper and the init-before-plan order)
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/r02j_gpu_tests.log 2>&1; echo "pytest rc=$?" >> $out/r02j_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/r02j_smoke.log 2>&1; echo "smoke rc=$?" >> $out/r02j_smoke.log
timeout 900 python bench.py > $out/r02j_bench.json 2> $out/r02j_bench.err; echo "bench rc=$?" >> $out/r02j_bench.err
timeout 600 python tools/e2e_breakdown.py > $out/r02j_e2e_breakdown.jsonl 2>&1
echo done
