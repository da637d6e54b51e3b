#!/bin/bash
# shorter HBM runs (3 / 4 fixed low tile qubits: 60 / 65 passes) vs 5 (71)
out=gpurun_out; mkdir -p $out
for c in 4 3; do
for v in 38273024 38273048 575143936; do
  QG_DEV_CLOW=$c QG_JIT_VARIANT=$v timeout 300 python tools/jit_time.py 32 random | sed "s/^{/{\"clow\": $c, /" >> $out/p51.jsonl 2>> $out/p51.err
done
done
echo done
