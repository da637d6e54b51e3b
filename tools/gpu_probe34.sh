#!/bin/bash
# 512 B HBM runs (6 fixed low tile qubits) vs 256 B with the tile-search planner
out=gpurun_out; mkdir -p $out
for c in 5 6; do
for v in 38273024 38273048 38273056; do
  QG_DEV_CLOW=$c QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random | sed "s/^{/{\"clow\": $c, /" >> $out/p34.jsonl 2>> $out/p34.err
done
done
QG_BW_CASES=contig0-12,hi8,r256_q18-25,r256_q19-26,r256_q20-27,r256_q21-28,r256_q20-23_28-31,r256_q12-15_24-27,r256_odd13-27,r512_q24-31,r256_q6_q25-31,r256_q7_q25-31,r256_q10_q25-31 timeout 600 python tools/bw_probe.py >> $out/p34_bw.txt 2>&1
echo done
