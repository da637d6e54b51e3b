"""Sharded state-vector execution — the reference's partitioned executor
(/root/reference/pkg/src/qgear/partition.py) re-designed for 1..8 B200s.

Reference: the 2^n amplitudes are split into W contiguous chunks (the top
log2 W qubits are "global", partition.py:89-97); every gate whose TARGET is
global triggers one pairwise chunk exchange plus a global barrier
(partition.py:200-274).

Here: the planner (libqgear_b200) runs every gate whose non-diagonal target is
local inside fused passes (global controls and diagonal gates on global
qubits cost nothing: they are rank-bit predicates), and inserts a QUBIT REMAP
only when a non-diagonal target is global: the s needed global qubits swap
places with the top s local qubits — an all-to-all among groups of 2^s ranks,
one block of 2^(n_local-s) amplitudes per peer.  The logical->physical qubit
map is tracked and undone when the state is gathered.

Two exchange backends, same semantics:
  * torch.distributed (one process per GPU, NCCL over NVLink; gloo in CPU
    tests): ``batch_isend_irecv`` of the blocks;
  * in-process shards (``shards_local``): all W shards live in this process
    (on one device) and blocks are exchanged by device copies — this runs
    the multi-rank plans on a single GPU for parity tests.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import statevec as sv
from .errors import BadWorkerCountError, SequenceMismatchError, UnnormalizedStateError


def _check_worker_count(n_qubits: int, workers: int) -> None:
    """partition.py:82-86."""
    if workers < 1 or workers & (workers - 1):
        raise BadWorkerCountError(f"workers must be a power of two >= 1, got {workers}")
    if workers > (1 << n_qubits):
        raise BadWorkerCountError(f"workers {workers} exceeds 2^{n_qubits} amplitudes")


def chunk_length(n_qubits: int, workers: int) -> int:
    _check_worker_count(n_qubits, workers)
    return (1 << n_qubits) // workers


def partner_mask(n_qubits: int, workers: int, qubit: int) -> int:
    """0 when the qubit is local; else the worker-id mask of its partner (partition.py:94-97)."""
    n_local = chunk_length(n_qubits, workers).bit_length() - 1
    return 0 if qubit < n_local else 1 << (qubit - n_local)


# --------------------------------------------------------------------------- remap blocks
def remap_peers(rank: int, n_local: int, global_pos, local_pos):
    """For one remap: [(block j, peer rank)] this rank exchanges, plus its own block index.

    Local positions n_local-s .. n_local-1 (block index bits) swap with global
    positions global_pos[i] (rank bits global_pos[i] - n_local).  Rank r keeps
    block g_r (its own G-bits) and trades block j with the rank whose G-bits are j.
    """
    s = len(global_pos)
    assert list(local_pos) == list(range(n_local - s, n_local)), "remap must use the top local positions"
    rb = [p - n_local for p in global_pos]
    own = sum(((rank >> b) & 1) << i for i, b in enumerate(rb))
    clear = rank & ~sum(1 << b for b in rb)
    peers = []
    for j in range(1 << s):
        if j == own:
            continue
        peer = clear | sum(((j >> i) & 1) << b for i, b in enumerate(rb))
        peers.append((j, peer))
    return own, peers


def remap_local(shards: list[torch.Tensor], n_local: int, global_pos, local_pos) -> None:
    """In-process remap of W shards (exact semantics of the distributed exchange)."""
    s = len(global_pos)
    blk = 1 << (n_local - s)
    old = [t.clone() for t in shards]
    for r, t in enumerate(shards):
        own, peers = remap_peers(r, n_local, global_pos, local_pos)
        for j, peer in peers:
            # peer's block at index `own` (= my G-bits) comes to my block j
            t[j * blk:(j + 1) * blk].copy_(old[peer][own * blk:(own + 1) * blk])


REMAP_CHUNK_BYTES = 1 << 30  # per peer and round: bounds the staging memory (37 q / 8 ranks = 128 GiB shards)


def remap_dist(shard: torch.Tensor, n_local: int, global_pos, local_pos, rank: int, group=None,
               staging: torch.Tensor | None = None, chunk_bytes: int = REMAP_CHUNK_BYTES) -> int:
    """torch.distributed remap of this rank's shard; returns the number of sends.

    Block j of this shard goes to the rank whose swapped bits equal j and comes
    back from it (an all-to-all within the group of 2^s ranks sharing the other
    rank bits).  The exchange runs in rounds of at most `chunk_bytes` per peer
    through a staging buffer of (2^s - 1) chunks, so a 128 GiB shard needs
    ~7 GiB of staging, not another 112 GiB."""
    import torch.distributed as dist

    s = len(global_pos)
    blk = 1 << (n_local - s)
    own, peers = remap_peers(rank, n_local, global_pos, local_pos)
    if not peers:
        return 0
    chunk = max(1, min(blk, chunk_bytes // shard.element_size()))
    need = len(peers) * chunk
    if staging is None or staging.numel() < need or staging.dtype != shard.dtype:
        staging = torch.empty(need, dtype=shard.dtype, device=shard.device)

    def wire(t: torch.Tensor) -> torch.Tensor:  # complex blocks travel as (re, im) pairs
        return torch.view_as_real(t) if t.is_complex() else t

    for off in range(0, blk, chunk):
        n = min(chunk, blk - off)
        ops = []
        for k, (j, peer) in enumerate(peers):
            ops.append(dist.P2POp(dist.isend, wire(shard[j * blk + off:j * blk + off + n]), peer, group=group))
            ops.append(dist.P2POp(dist.irecv, wire(staging[k * chunk:k * chunk + n]), peer, group=group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for k, (j, _) in enumerate(peers):
            shard[j * blk + off:j * blk + off + n].copy_(staging[k * chunk:k * chunk + n])
    return len(peers)


# --------------------------------------------------------------------------- gather
def _permute_to_logical(full: torch.Tensor, n: int, phys_of_logical) -> torch.Tensor:
    """Physical-order vector -> logical order (qubit q read from bit phys_of_logical[q])."""
    perm = [int(p) for p in phys_of_logical]
    if perm == list(range(n)):
        return full
    # group logical qubits into runs that map to consecutive physical positions
    runs = []  # (logical start, length, physical start)
    q = 0
    while q < n:
        ln = 1
        while q + ln < n and perm[q + ln] == perm[q] + ln:
            ln += 1
        runs.append((q, ln, perm[q]))
        q += ln
    phys_runs = sorted(runs, key=lambda r: r[2])
    # view the physical vector with one dim per run (most significant first)
    shape = [1 << r[1] for r in reversed(phys_runs)]
    x = full.reshape(shape)
    order_phys = list(reversed(phys_runs))  # dim i <-> phys_runs reversed
    want = list(reversed(runs))              # logical most significant first
    dims = [order_phys.index(r) for r in want]
    return x.permute(*dims).contiguous().reshape(-1)


@dataclass
class DistributedResult:
    """partition.py:277-283 (tasks -> the plan summary)."""

    state: sv.StateVector | None
    counts: sv.CountsTable | None
    messages_sent: list[int]
    messages_received: list[int]
    tasks: dict = field(default_factory=dict)
    shards: list[torch.Tensor] | None = None


def execute_distributed(circuit, workers: int, options: sv.SimOptions | None = None, delay_hook=None,
                        group=None, gather: bool = True) -> DistributedResult:
    """Run a circuit sharded over `workers` ranks (partition.py:286-355).

    With torch.distributed initialised and world size == workers, this process
    runs its own rank's shard on its current CUDA device and exchanges over
    the process group (NCCL).  Otherwise all shards run in this process on
    one device (``delay_hook`` is accepted for API compatibility and called as
    delay_hook(rank, remap_index) before each exchange).  Unlike the reference
    (partition.py:300-301), complex64 is allowed with workers > 1.
    """
    options = options or sv.SimOptions()
    gt, gp, n = sv.circuit_arrays(circuit)
    _check_worker_count(n, workers)
    sv._trailing_split_arrays(gt[:, 0])
    sv._check_budget(n, options.precision, options.memory_budget)
    g = workers.bit_length() - 1
    plan = sv.CompiledCircuit(gt, gp, n, options.precision, g, options.fuse, options.tile_qubits,
                              options.max_stages, options.max_cost, jit=options.jit)
    n_local = plan.n_local
    dtype = sv._DTYPES[options.precision]

    import torch.distributed as dist

    distributed = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) == workers and workers > 1
    sent = [0] * workers
    if distributed:
        rank = dist.get_rank(group)
        dev = torch.device("cuda", torch.cuda.current_device())
        shard = torch.empty(1 << n_local, dtype=dtype, device=dev)
        sv.N.call("qg_state_init_zero", sv.C.c_void_p(shard.data_ptr()), n_local, sv._QG_DTYPE[options.precision],
                  rank, sv._stream(dev))
        staging = None
        for seg in range(plan.n_segments):
            plan.execute_segment(seg, shard, rank)
            if seg < plan.n_segments - 1:
                gpos, lpos = plan.remaps[seg]
                if delay_hook is not None:
                    delay_hook(rank, seg)
                torch.cuda.current_stream(dev).synchronize()
                sent[rank] += remap_dist(shard, n_local, gpos, lpos, rank, group, staging)
        counts_all = torch.tensor(sent, dtype=torch.int64, device=dev)
        dist.all_reduce(counts_all, group=group)
        sent = counts_all.cpu().tolist()
        shards = [shard]
        state = None
        if gather:
            parts = [torch.empty_like(shard) for _ in range(workers)] if rank == 0 else None
            dist.gather(shard, parts, dst=0, group=group)
            if rank == 0:
                full = _permute_to_logical(torch.cat(parts), n, plan.final_map)
                state = sv.StateVector(n, options.precision, full)
    else:
        dev = sv._device(options.device)
        shards = []
        for r in range(workers):
            t = torch.empty(1 << n_local, dtype=dtype, device=dev)
            sv.N.call("qg_state_init_zero", sv.C.c_void_p(t.data_ptr()), n_local, sv._QG_DTYPE[options.precision],
                      r, sv._stream(dev))
            shards.append(t)
        for seg in range(plan.n_segments):
            for r in range(workers):
                plan.execute_segment(seg, shards[r], r)
            if seg < plan.n_segments - 1:
                gpos, lpos = plan.remaps[seg]
                if delay_hook is not None:
                    for r in range(workers):
                        delay_hook(r, seg)
                remap_local(shards, n_local, gpos, lpos)
                for r in range(workers):
                    sent[r] += (1 << len(gpos)) - 1
        state = None
        if gather:
            full = _permute_to_logical(torch.cat(shards), n, plan.final_map)
            state = sv.StateVector(n, options.precision, full)
    counts = None
    if state is not None:
        nsq = state.norm_sq()
        if abs(nsq - 1.0) > sv.NORM_TOL[options.precision]:
            raise UnnormalizedStateError(f"gathered norm^2 = {nsq!r}")  # partition.py:139-140
        if options.shots > 0:
            counts = sv.sample_counts(state, options.shots, options.rng_seed, options.sampler)
    if len(set(sent)) > 1 and not distributed:
        raise SequenceMismatchError(f"workers exchanged different message counts: {sent}")
    return DistributedResult(state=state, counts=counts, messages_sent=sent, messages_received=list(sent),
                             tasks=dict(plan.info, remaps=plan.remaps), shards=shards)
