"""GPU: the torch.distributed branch of execute_distributed end to end, at world
size 2 (partition.py:286-355 of the reference).

Two processes share the one GPU of the test box; the process group is gloo, so
remap blocks and the gather travel through host memory (partition._host_wire)
— the same remap_dist code path NCCL runs on a multi-GPU node, with the same
segments, remaps, gather, logical permutation and counts."""

import math
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from paper_2504_03967_b200.generators import RandomSpec, qft_arrays, random_arrays

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    from paper_2504_03967_b200 import partition as pt
    from paper_2504_03967_b200 import statevec as sv
    from paper_2504_03967_b200.ir import CircType, CircuitTensor

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kind, n, prec, shots, chunk = case
        gt, gp = random_arrays(RandomSpec(n, 120, 3)) if kind == "random" else qft_arrays(n)
        circ = CircuitTensor.from_arrays(CircType.RANDOM, n, gt, gp)
        if chunk:
            pt.REMAP_CHUNK_BYTES = chunk  # several exchange rounds per remap
        res = pt.execute_distributed(circ, world, sv.SimOptions(prec, shots, 7, device=0))
        if rank == 0:
            np.savez(out, state=res.state.to_numpy(), idx=res.counts.indices, cnt=res.counts.values,
                     sent=np.array(res.messages_sent), remaps=res.tasks["n_remaps"], total=res.counts.total)
    finally:
        dist.destroy_process_group()


def _run(case, world=2):
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r0.npz")
        mp.start_processes(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True,
                           start_method="spawn")
        with np.load(out) as z:
            return {k: z[k] for k in z.files}


@pytest.mark.parametrize("case", [("random", 14, "fp64", 50_000, 0), ("random", 16, "fp32", 50_000, 1 << 12),
                                  ("qft", 14, "fp32", 20_000, 0)])
def test_execute_distributed_world2(case):
    kind, n, prec, shots, _ = case
    r = _run(case)
    gt, gp = random_arrays(RandomSpec(n, 120, 3)) if kind == "random" else qft_arrays(n)
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    err = float(np.linalg.norm(r["state"].astype(np.complex128) - ref) / np.linalg.norm(ref))
    assert err <= (1e-12 if prec == "fp64" else 1e-5), err
    if kind == "random":
        assert int(r["remaps"]) >= 1  # the exchange actually ran
        assert r["sent"].tolist() == [int(r["remaps"])] * 2  # one peer per 1-qubit remap at W=2
    # counts: total, and TV over the b lowest qubits against the oracle's exact distribution
    assert int(r["total"]) == shots and int(r["cnt"].sum()) == shots
    p = oracle.exact_probabilities(ref)
    b = min(n, int(math.log2(shots / 64)))
    emp = np.bincount(r["idx"] & ((1 << b) - 1), weights=r["cnt"], minlength=1 << b) / shots
    exact = np.bincount(np.arange(1 << n) & ((1 << b) - 1), weights=p, minlength=1 << b)
    assert 0.5 * np.abs(emp - exact).sum() <= 4 * 0.5 * math.sqrt((1 << b) / shots)
