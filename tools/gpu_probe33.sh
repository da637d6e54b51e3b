#!/bin/bash
# Multi-rank bench path on one GPU: 2 ranks over gloo sharing cuda:0 (the pool has 1 GPU per call).
mkdir -p gpurun_out
QG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --qubits 28 --blocks 200 \
  --steps 2 --warmup 3 > gpurun_out/p33_gloo2.json 2> gpurun_out/p33_gloo2.err
echo "rc=$?"
tail -c 3000 gpurun_out/p33_gloo2.json
