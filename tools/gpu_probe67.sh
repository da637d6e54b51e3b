#!/bin/bash
# r02i: C2 (QFT 28 q, complex64, 1e5 shots e2e) as a bench.py line
out=gpurun_out; mkdir -p $out
timeout 600 python bench.py --circuit qft --qubits 28 --steps 20 --warmup 5 --e2e-steps 5 > $out/r02i_bench_qft28.json 2> $out/r02i_bench_qft28.err; echo "rc=$?" >> $out/r02i_bench_qft28.err
timeout 600 python bench.py --circuit qft --qubits 32 --steps 5 --warmup 3 --no-e2e > $out/r02i_bench_qft32.json 2> $out/r02i_bench_qft32.err; echo "rc=$?" >> $out/r02i_bench_qft32.err
echo done
