#!/bin/bash
out=gpurun_out; mkdir -p $out
for kc in 9 6 7; do
  QG_KW="dict(kernel_cfg=$kc)" timeout 300 python tools/jit_time.py 32 random >> $out/p20_variants.jsonl 2>> $out/p20_variants.err
done
for v in 4718616 4718624 4751360 5767168; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p20_variants.jsonl 2>> $out/p20_variants.err
done
timeout 1200 ncu --set full --clock-control none -k regex:qg_jit_pass -s 30 -c 1 -o $out/p20_jit32 python tools/jit_time.py 32 random > $out/p20_ncu.log 2>&1
echo done
