#!/bin/bash
# r02i: sticky warp bits (planner) + scoped hand-over barriers (JIT): correctness and A/B timing
out=gpurun_out; mkdir -p $out
timeout 900 python tools/jit_check.py 22 26 28 > $out/r02i_sticky_check.log 2>&1
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_parity.py -x -q -m gpu > $out/r02i_sticky_tests.log 2>&1; echo "rc=$?" >> $out/r02i_sticky_tests.log
for i in 1 2; do
  timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"mode": "sticky+scoped", /' >> $out/r02i_sticky.jsonl 2>> $out/r02i_sticky.err
  QG_DEV_CTA_SYNC=1 timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"mode": "sticky+cta", /' >> $out/r02i_sticky.jsonl 2>> $out/r02i_sticky.err
  QG_DEV_STICKY=0 timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"mode": "plain+scoped", /' >> $out/r02i_sticky.jsonl 2>> $out/r02i_sticky.err
  QG_DEV_STICKY=0 QG_DEV_CTA_SYNC=1 timeout 300 python tools/jit_time.py 32 random | sed 's/^{/{"mode": "plain+cta (r02h)", /' >> $out/r02i_sticky.jsonl 2>> $out/r02i_sticky.err
done
timeout 300 python tools/jit_time.py 28 qft | sed 's/^{/{"mode": "sticky+scoped", /' >> $out/r02i_sticky.jsonl 2>> $out/r02i_sticky.err
echo done
