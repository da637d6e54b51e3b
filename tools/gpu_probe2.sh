#!/bin/bash
# overlap experiments on the JIT pass + new GPU tests + one ncu capture of a JIT pass
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_tree_sampler.py tests/test_gpu_distributed.py -x -q > $out/p2_tests.log 2>&1; echo "pytest rc=$?" >> $out/p2_tests.log
for v in 4 64 512 1024 256 516 2; do
  QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p2_variants.jsonl 2>> $out/p2_variants.err
done
QG_JIT_STAGGER_NS=20000 QG_JIT_VARIANT=64 timeout 300 python tools/jit_time.py 32 random >> $out/p2_variants.jsonl 2>> $out/p2_variants.err
for v in 0 24 32; do
  QG_KW="dict(kernel_cfg=6)" QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random >> $out/p2_variants.jsonl 2>> $out/p2_variants.err
done
timeout 1200 ncu --set full --clock-control none -k regex:qg_jit_pass -s 30 -c 1 -o $out/p2_jit32 python tools/jit_time.py 32 random > $out/p2_ncu.log 2>&1
echo done
