#!/bin/bash
# interleave + no prefetch on the passes with tile-uniform phase slots (default now) vs off
out=gpurun_out; mkdir -p $out
timeout 300 python tools/jit_check.py 24 28 > $out/p62_check.txt 2>&1
for a in 0 1; do
  if [ $a = 1 ]; then export QG_DEV_NO_UPH_IL=1; fi
  for n in 28 32; do timeout 300 python tools/jit_time.py $n qft | sed "s/^{/{\"no_uph_il\": $a, /" >> $out/p62.jsonl 2>> $out/p62.err; done
  timeout 300 python tools/jit_time.py 32 random | sed "s/^{/{\"no_uph_il\": $a, /" >> $out/p62.jsonl 2>> $out/p62.err
done
unset QG_DEV_NO_UPH_IL
timeout 300 python tools/bench_configs.py c2 > $out/p62_c2.json 2>> $out/p62.err
echo done
