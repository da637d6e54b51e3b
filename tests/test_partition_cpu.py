"""Multi-rank logic on CPU: remap exchange over torch.distributed (gloo, 2 and 4
ranks) equals the in-process remap; partner masks match the reference's plan
(golden vectors); the logical-order gather permutation is exact."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_03967_b200 import partition as pt
from paper_2504_03967_b200.errors import BadWorkerCountError


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, remaps, full, out, chunk_bytes=pt.REMAP_CHUNK_BYTES):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_local = n - (world.bit_length() - 1)
    shard = full[rank << n_local:(rank + 1) << n_local].clone()
    sends = 0
    for gpos, lpos in remaps:
        sends += pt.remap_dist(shard, n_local, gpos, lpos, rank, chunk_bytes=chunk_bytes)
    out[rank] = (shard.numpy().copy(), sends)
    dist.destroy_process_group()


def _run(world, n, remaps, chunk_bytes=pt.REMAP_CHUNK_BYTES):
    g = torch.Generator().manual_seed(7)
    full = torch.complex(torch.randn(1 << n, generator=g, dtype=torch.float64),
                         torch.randn(1 << n, generator=g, dtype=torch.float64))
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n, remaps, full, out, chunk_bytes), nprocs=world, join=True)
    n_local = n - (world.bit_length() - 1)
    shards = [full[r << n_local:(r + 1) << n_local].clone() for r in range(world)]
    for gpos, lpos in remaps:
        pt.remap_local(shards, n_local, gpos, lpos)
    return [out[r] for r in range(world)], shards


@pytest.mark.parametrize("world,n,remaps,chunk_bytes", [
    (2, 6, [([5], [4])], pt.REMAP_CHUNK_BYTES),
    (4, 7, [([6], [4]), ([5, 6], [3, 4]), ([5], [4])], pt.REMAP_CHUNK_BYTES),
    (4, 7, [([5, 6], [3, 4]), ([6], [4])], 48),   # several exchange rounds per block (3 x 16 B chunks)
    # Belady victims below the top local positions: strided blocks, packed per round
    (2, 6, [([5], [2])], pt.REMAP_CHUNK_BYTES),
    (4, 8, [([6, 7], [1, 4]), ([7], [0]), ([6, 7], [5, 2])], pt.REMAP_CHUNK_BYTES),
    (8, 9, [([6, 7, 8], [0, 3, 5]), ([8, 6], [2, 1])], 32),  # and several rounds
])
def test_gloo_remap_equals_local(world, n, remaps, chunk_bytes):
    got, ref = _run(world, n, remaps, chunk_bytes)
    for r in range(world):
        assert np.array_equal(got[r][0], ref[r].numpy())
        assert got[r][1] == sum((1 << len(gp)) - 1 for gp, _ in remaps)


def test_local_remap_is_a_qubit_swap():
    n, world = 6, 4
    n_local = n - 2
    full = torch.arange(1 << n, dtype=torch.float64)
    shards = [full[r << n_local:(r + 1) << n_local].clone() for r in range(world)]
    pt.remap_local(shards, n_local, [4, 5], [2, 3])  # swap physical bits (2,4) and (3,5)
    new = torch.cat(shards).numpy()
    idx = np.arange(1 << n)
    src = idx.copy()
    for a, b in [(2, 4), (3, 5)]:
        ba, bb = (src >> a) & 1, (src >> b) & 1
        src = src ^ ((ba ^ bb) << a) ^ ((ba ^ bb) << b)
    assert np.array_equal(new, full.numpy()[src])


def test_local_remap_arbitrary_positions_is_a_qubit_swap():
    n, world = 7, 4
    n_local = n - 2
    full = torch.arange(1 << n, dtype=torch.float64)
    shards = [full[r << n_local:(r + 1) << n_local].clone() for r in range(world)]
    pt.remap_local(shards, n_local, [6, 5], [1, 3])  # swap physical bits (1,6) and (3,5)
    new = torch.cat(shards).numpy()
    idx = np.arange(1 << n)
    src = idx.copy()
    for a, b in [(1, 6), (3, 5)]:
        ba, bb = (src >> a) & 1, (src >> b) & 1
        src = src ^ ((ba ^ bb) << a) ^ ((ba ^ bb) << b)
    assert np.array_equal(new, full.numpy()[src])


def test_permute_to_logical():
    n = 7
    rng = np.random.default_rng(0)
    perm = rng.permutation(n)
    phys = torch.from_numpy(rng.normal(size=1 << n))
    got = pt._permute_to_logical(phys, n, perm).numpy()
    idx = np.arange(1 << n)
    src = np.zeros_like(idx)
    for q in range(n):
        src |= ((idx >> q) & 1) << int(perm[q])
    assert np.array_equal(got, phys.numpy()[src])


def test_partner_masks_match_reference_plan(golden):
    for j in range(3):
        nq, ng, w = (int(v) for v in golden[f"part{j}_meta"])
        tgt = golden[f"part{j}_type"][:ng, 2]
        masks = [pt.partner_mask(nq, w, int(t)) for t in tgt]
        assert masks == golden[f"part{j}_masks"].tolist()
    assert [pt.partner_mask(4, 4, q) for q in range(4)] == [0, 0, 1, 2]
    with pytest.raises(BadWorkerCountError):
        pt.chunk_length(4, 3)
    with pytest.raises(BadWorkerCountError):
        pt.chunk_length(2, 8)


def _step_worker(rank, world, port, seqs, fps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pt.check_step(seqs[rank], fps[rank], final=(seqs[0] == 99))
        out[rank] = "ok"
    except Exception as e:  # noqa: BLE001
        out[rank] = type(e).__name__
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seqs,fps,want", [
    ([3, 3], [7, 7], "ok"),
    ([3, 4], [7, 7], "ProtocolViolationError"),       # a rank skipped / repeated an exchange
    ([3, 3], [7, 8], "ProtocolViolationError"),       # ranks run different circuits
    ([99, 98], [7, 7], "SequenceMismatchError"),      # final step: partition.py gather seq check
])
def test_check_step_agreement(seqs, fps, want):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_step_worker, args=(2, _free_port(), seqs, fps, out), nprocs=2, join=True)
    assert out[0] == want and out[1] == want


def test_plan_fingerprint():
    gt = np.array([[0, -1, 1], [4, 0, 1]], dtype=np.int32)
    gp = np.array([0.0, 0.0])
    a = pt.plan_fingerprint(gt, gp, 3, 2)
    assert a == pt.plan_fingerprint(gt.copy(), gp.copy(), 3, 2) and 0 <= a < 2**63
    assert a != pt.plan_fingerprint(gt, gp + 1e-9, 3, 2) and a != pt.plan_fingerprint(gt, gp, 3, 4)
