#!/bin/bash
# r02i: DRAM traffic per launch of the JIT pass for the QFT28 (C2) and complex128 32 q bench workloads
out=gpurun_out; mkdir -p $out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:qg_jit_pass -s 5 -c 1 --csv --log-file $out/r02i_traffic_qft28.csv \
  python bench.py --circuit qft --qubits 28 --steps 1 --warmup 1 --no-e2e > $out/r02i_traffic_qft28.log 2>&1
timeout 1200 ncu --metrics $M --clock-control none -k regex:qg_jit_pass -s 20 -c 1 --csv --log-file $out/r02i_traffic_c128.csv \
  python bench.py --precision fp64 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $out/r02i_traffic_c128.log 2>&1
echo done
