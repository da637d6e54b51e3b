#!/bin/bash
out=gpurun_out; mkdir -p $out
timeout 900 python tools/jit_check128.py 20 24 28 30 > $out/p27_check128.log 2>&1
timeout 600 python tools/jit_check.py 24 28 > $out/p27_check64.log 2>&1
echo done
