#!/bin/bash
# 8 independent tile searches per pass (threads) vs 1: planning time, pass time, bench
out=gpurun_out; mkdir -p $out
for K in 1 8; do QG_DEV_TILE_K=$K timeout 300 python tools/plan_time.py >> $out/p55_plan.jsonl 2>> $out/p55.err; done
for K in 1 8; do QG_DEV_TILE_K=$K timeout 300 python tools/jit_time.py 32 random | sed "s/^{/{\"K\": $K, /" >> $out/p55.jsonl 2>> $out/p55.err; done
timeout 900 python bench.py --no-cpu-baseline > $out/p55_bench.json 2>> $out/p55.err
echo done
