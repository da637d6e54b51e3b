#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + one full capture of the fused kernel.
# usage (under gpurun): bash tools/gpu_round.sh [tag]
tag=${1:-r01}
set -x
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $out/gpu_$tag.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/gpu_tests_$tag.log 2>&1; echo "pytest rc=$?" >> $out/gpu_tests_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> $out/smoke_$tag.log
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench rc=$?" >> $out/bench_$tag.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_$tag.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $out/ncu_bench_$tag.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:qg_jit_pass -s 20 -c 1 -o $out/prof32_$tag \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $out/ncu_full_$tag.log 2>&1
for c in c1 c2 c4; do timeout 600 python tools/bench_configs.py $c > $out/cfg_${c}_$tag.json 2> $out/cfg_${c}_$tag.err; done
echo done
