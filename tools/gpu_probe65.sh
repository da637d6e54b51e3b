#!/bin/bash
# r02i: re-validate after container re-creation (tests, smoke, bench) + k = 14 tile probes with the tile search
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/r02i_gpu_tests.log 2>&1; echo "pytest rc=$?" >> $out/r02i_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/r02i_smoke.log 2>&1; echo "smoke rc=$?" >> $out/r02i_smoke.log
timeout 900 python bench.py > $out/r02i_bench.json 2> $out/r02i_bench.err; echo "bench rc=$?" >> $out/r02i_bench.err
for cfg in 0 6 8; do QG_KW="dict(kernel_cfg=$cfg)" timeout 300 python tools/jit_time.py 32 random >> $out/r02i_k14.jsonl 2>> $out/r02i_k14.err; done
echo done
