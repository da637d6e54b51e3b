#!/bin/bash
# ncu: JIT memory-only pass (interleaved, no prefetch) vs the microbenchmark's s3 on the same tile layout
out=gpurun_out; mkdir -p $out
sed -n 31p tools/bin/tiles32.txt > /tmp/t31.txt
QG_JIT_VARIANT=575144088 timeout 900 ncu --set full --clock-control none -k regex:qg_jit_pass -s 30 -c 1 -o $out/p42_jitmem python tools/jit_time.py 32 random > $out/p42_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:s3 -c 1 -o $out/p42_s3 ./tools/bin/mem_pattern /tmp/t31.txt > $out/p42_ncu2.log 2>&1
echo done
