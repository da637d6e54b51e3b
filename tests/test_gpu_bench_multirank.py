"""GPU: bench.py's multi-rank path end to end (the driver's `torchrun --nproc-per-node N
bench.py --gpus N` launch), at world size 2 on the test box's one GPU.

QG_DIST_BACKEND=gloo lets the two ranks share cuda:0 and stage the remap blocks through
host memory; everything else is the NCCL path: per-rank segments, the remap exchange
(partition.remap_dist), per-remap CUDA-event timing, the max-over-ranks reduction and
rank 0's single JSON line."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_gloo():
    env = dict(os.environ, QG_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--qubits", "24", "--blocks", "60", "--steps", "2", "--warmup", "3", "--no-cpu-baseline",
           "--e2e-shots", "1000"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]  # rank 0 alone prints
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["steps"] == 2 and out["warmup"] == 3
    assert out["value"] > 0 and out["ms_per_step"] > 0
    cfg = out["config"]
    assert cfg["parallelism"] == "sv-shard2" and cfg["dist_backend"] == "gloo"
    assert cfg["gates"] == 180 and cfg["remaps"] >= 1
    nvl = out["roofline_nvl"]
    assert nvl is not None and len(nvl["per_remap"]) == cfg["remaps"]
    # one rank's egress per remap: half its 2^23-amplitude complex64 shard
    assert all(r["egress_bytes"] == (1 << 23) * 8 // 2 for r in nvl["per_remap"])
    assert out["e2e"]["value"] > 0 and out["e2e"]["shots"] == 1000
    assert out["gpu_launches"] > 0
