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
from .errors import BadWorkerCountError, ProtocolViolationError, SequenceMismatchError, UnnormalizedStateError


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

    Local position local_pos[i] swaps with global position global_pos[i] (rank bit
    global_pos[i] - n_local).  Block j of a shard = the amplitudes whose local bits
    local_pos[i] equal bit i of j.  Rank r keeps block g_r (its own G-bits) and
    trades block j with the rank whose G-bits are j."""
    s = len(global_pos)
    assert len(local_pos) == s and all(0 <= p < n_local for p in local_pos)
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


def _contiguous(n_local: int, local_pos) -> bool:
    """Blocks are contiguous ranges iff the swapped local positions are the top ones."""
    s = len(local_pos)
    return list(local_pos) == list(range(n_local - s, n_local))


def block_view(t: torch.Tensor, n_local: int, local_pos, j: int) -> torch.Tensor:
    """Strided view of block j of a shard (local bit local_pos[i] = bit i of j): one
    dimension per run of untouched index bits, runs of 2^min(local_pos) amplitudes."""
    order = sorted(range(len(local_pos)), key=lambda i: -local_pos[i])  # most significant first
    shape, idx, hi = [], [], n_local
    for i in order:
        p = local_pos[i]
        shape += [1 << (hi - 1 - p), 2]
        idx += [slice(None), (j >> i) & 1]
        hi = p
    shape.append(1 << hi)
    idx.append(slice(None))
    return t.view(shape)[tuple(idx)]


def _chunks(v: torch.Tensor, max_elems: int):
    """Split a (strided) view into sub-views of at most max_elems elements."""
    if v.numel() <= max_elems:
        yield v
        return
    d = next(i for i, sz in enumerate(v.shape) if sz > 1)
    h = v.shape[d] // 2
    yield from _chunks(v.narrow(d, 0, h), max_elems)
    yield from _chunks(v.narrow(d, h, v.shape[d] - h), max_elems)


def remap_local(shards: list[torch.Tensor], n_local: int, global_pos, local_pos) -> None:
    """In-process remap of W shards (exact semantics of the distributed exchange)."""
    old = [t.clone() for t in shards]
    for r, t in enumerate(shards):
        own, peers = remap_peers(r, n_local, global_pos, local_pos)
        for j, peer in peers:
            # peer's block at index `own` (= my G-bits) comes to my block j
            block_view(t, n_local, local_pos, j).copy_(block_view(old[peer], n_local, local_pos, own))


REMAP_CHUNK_BYTES = 1 << 30  # per peer and round: bounds the staging memory (37 q / 8 ranks = 128 GiB shards)
_STAGING: dict = {}


def _host_wire(group) -> bool:
    """gloo moves host tensors only: device blocks are staged through host memory."""
    import torch.distributed as dist

    return dist.get_backend(group) == "gloo"


def _staging(numel: int, dtype, device) -> torch.Tensor:
    key = (str(device), dtype)
    t = _STAGING.get(key)
    if t is None or t.numel() < numel:
        _STAGING.pop(key, None)
        t = torch.empty(numel, dtype=dtype, device=device)
        _STAGING[key] = t
    return t


def remap_dist(shard: torch.Tensor, n_local: int, global_pos, local_pos, rank: int, group=None,
               staging: torch.Tensor | None = None, chunk_bytes: int | None = None) -> int:
    """torch.distributed remap of this rank's shard; returns the number of sends.

    Block j of this shard goes to the rank whose swapped bits equal j and comes
    back from it (an all-to-all within the group of 2^s ranks sharing the other
    rank bits).  The exchange runs in rounds of at most `chunk_bytes` per peer
    through two staging halves of (2^s - 1) chunks each (a 37-qubit / 8-rank
    shard is 128 GiB: a whole-block staging buffer would not fit next to it):
    round r+1's transfers run while round r's received blocks are copied into
    the shard on a side stream.  Nothing here blocks the host on NCCL: the
    collectives are ordered after the fused passes on the current stream and the
    current stream waits for the last copy-back."""
    import torch.distributed as dist

    s = len(global_pos)
    blk = 1 << (n_local - s)
    own, peers = remap_peers(rank, n_local, global_pos, local_pos)
    if not peers:
        return 0
    host = shard.is_cuda and _host_wire(group)
    chunk_bytes = REMAP_CHUNK_BYTES if chunk_bytes is None else chunk_bytes
    if not _contiguous(n_local, local_pos):
        return _remap_dist_strided(shard, n_local, local_pos, peers, group, host, chunk_bytes)
    chunk = max(1, min(blk, chunk_bytes // shard.element_size()))
    rounds = list(range(0, blk, chunk))
    nbuf = 2 if len(rounds) > 1 and not host else 1
    per = len(peers) * chunk
    sdev = torch.device("cpu") if host or not shard.is_cuda else shard.device
    if staging is None or staging.numel() < nbuf * per or staging.dtype != shard.dtype or staging.device != sdev:
        staging = _staging(nbuf * per, shard.dtype, sdev)

    def wire(t: torch.Tensor) -> torch.Tensor:  # complex blocks travel as (re, im) pairs
        return torch.view_as_real(t) if t.is_complex() else t

    side = cur = None
    done = [None] * nbuf
    if shard.is_cuda and not host:
        cur = torch.cuda.current_stream(shard.device)
        side = torch.cuda.Stream(shard.device)
    for r, off in enumerate(rounds):
        n = min(chunk, blk - off)
        buf = staging[(r % nbuf) * per:(r % nbuf + 1) * per]
        if done[r % nbuf] is not None:  # this half's previous copy-back must have read it
            cur.wait_event(done[r % nbuf])
        ops = []
        for k, (j, peer) in enumerate(peers):
            src = shard[j * blk + off:j * blk + off + n]
            ops.append(dist.P2POp(dist.isend, wire(src.cpu() if host else src), peer, group=group))
            ops.append(dist.P2POp(dist.irecv, wire(buf[k * chunk:k * chunk + n]), peer, group=group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        if side is None:
            for k, (j, _) in enumerate(peers):
                shard[j * blk + off:j * blk + off + n].copy_(buf[k * chunk:k * chunk + n])
            continue
        side.wait_stream(cur)  # the received round
        with torch.cuda.stream(side):
            for k, (j, _) in enumerate(peers):
                shard[j * blk + off:j * blk + off + n].copy_(buf[k * chunk:k * chunk + n])
            ev = torch.cuda.Event()
            ev.record(side)
            done[r % nbuf] = ev
    if side is not None:
        cur.wait_stream(side)
    return len(peers)


def _remap_dist_strided(shard, n_local, local_pos, peers, group, host, chunk_bytes) -> int:
    """remap_dist for swapped local positions below the top ones (the planner's
    Belady victims): block j is a strided set of runs of 2^min(local_pos)
    amplitudes; each round packs one chunk of every outgoing block into a send
    buffer, exchanges, and unpacks the received chunks into the same positions."""
    import torch.distributed as dist

    chunk = max(1, chunk_bytes // shard.element_size())
    per = len(peers) * chunk
    sdev = torch.device("cpu") if host or not shard.is_cuda else shard.device
    sendbuf = torch.empty(per, dtype=shard.dtype, device=sdev)
    recvbuf = torch.empty(per, dtype=shard.dtype, device=sdev)
    views = [list(_chunks(block_view(shard, n_local, local_pos, j), chunk)) for j, _ in peers]

    def wire(t: torch.Tensor) -> torch.Tensor:
        return torch.view_as_real(t) if t.is_complex() else t

    for c in range(len(views[0])):
        ops = []
        for k, (_, peer) in enumerate(peers):
            v = views[k][c]
            m = v.numel()
            sendbuf[k * chunk:k * chunk + m].view(v.shape).copy_(v)  # pack
            ops.append(dist.P2POp(dist.isend, wire(sendbuf[k * chunk:k * chunk + m]), peer, group=group))
            ops.append(dist.P2POp(dist.irecv, wire(recvbuf[k * chunk:k * chunk + m]), peer, group=group))
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for k in range(len(peers)):
            v = views[k][c]
            v.copy_(recvbuf[k * chunk:k * chunk + v.numel()].view(v.shape))  # unpack
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


# --------------------------------------------------------------------------- rank agreement
def plan_fingerprint(gate_type: np.ndarray, gate_param: np.ndarray, n_qubits: int, workers: int) -> int:
    """63-bit digest of what every rank must agree on before exchanging blocks."""
    import hashlib

    h = hashlib.blake2b(digest_size=8)
    h.update(np.ascontiguousarray(gate_type, dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(gate_param, dtype=np.float64).tobytes())
    h.update(np.array([n_qubits, workers], dtype=np.int64).tobytes())
    return int.from_bytes(h.digest(), "little") & ((1 << 63) - 1)


def check_step(seq: int, fingerprint: int, group=None, final: bool = False, device=None) -> None:
    """Every rank at the same exchange step of the same plan, or an error on every rank.

    The reference checks each message's (sequence number, sender) and the workers'
    final sequence numbers at the gather (partition.py:168-173, 112-141): here one
    all-gather of (seq, plan fingerprint) per remap stands in for the per-message
    check; a mismatch raises ProtocolViolationError (SequenceMismatchError for the
    final step), and a failed or timed-out collective (the process group's timeout,
    the reference's _JOIN_TIMEOUT, partition.py:50) is re-raised as
    ProtocolViolationError."""
    import torch.distributed as dist

    try:
        t = torch.tensor([seq, fingerprint], dtype=torch.int64,
                         device=device if device is not None and not _host_wire(group) else "cpu")
        allv = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
        dist.all_gather(allv, t, group=group)
    except Exception as e:  # NCCL / gloo failure or timeout
        raise ProtocolViolationError(f"exchange step {seq}: collective failed: {e}") from e
    vals = [tuple(int(x) for x in v.tolist()) for v in allv]
    if len(set(v[1] for v in vals)) > 1:
        raise ProtocolViolationError(f"ranks run different plans at step {seq}: {[v[1] for v in vals]}")
    if len(set(v[0] for v in vals)) > 1:
        err = SequenceMismatchError if final else ProtocolViolationError
        raise err(f"ranks at different exchange steps: {[v[0] for v in vals]}")


# --------------------------------------------------------------------------- sampling
def logical_indices(phys: torch.Tensor, phys_of_logical) -> torch.Tensor:
    """Physical basis indices (rank bits on top) -> logical indices: logical qubit q
    is physical bit phys_of_logical[q] (the plan's final map)."""
    perm = [int(p) for p in phys_of_logical]
    if perm == list(range(len(perm))):
        return phys
    out = torch.zeros_like(phys)
    for q, p in enumerate(perm):
        out |= ((phys >> p) & 1) << q
    return out


def _comm(t: torch.Tensor, group) -> torch.Tensor:
    return t.cpu() if _host_wire(group) else t


def sample_shards(shards: list[torch.Tensor], n_local: int, phys_of_logical, shots: int, rng_seed: int,
                  norm_tol: float, ranks=None, group=None) -> tuple[torch.Tensor, torch.Tensor] | None:
    """Counts of `shots` draws from a sharded state without gathering it.

    Every rank: tree masses of its shard (one HBM read); the P masses are
    all-gathered (P doubles); the shots are split over the ranks by the top of the
    binomial tree (same seed everywhere, so every rank computes the same split);
    each rank draws its own count from its shard (tag 2 + rank); outcome indices
    get the rank bits and the logical qubit order; rank 0 gathers the (index,
    count) lists.  The reference gathers the state and samples it centrally
    (partition.py:345-348, statevec.py:221-234).  In-process shards (``ranks``
    None, all shards here): the same steps without communication.
    Returns (logical index ascending, count) on rank 0 (None on other ranks)."""
    import torch.distributed as dist

    distributed = ranks is not None
    samplers = [sv.TreeSampler(t, (r if not distributed else ranks) << n_local)
                for r, t in enumerate(shards)]
    mine = [s.prepare() for s in samplers]
    if distributed:
        rank, workers = ranks, dist.get_world_size(group)
        mt = _comm(torch.tensor(mine, dtype=torch.float64, device=shards[0].device), group)
        allm = [torch.empty_like(mt) for _ in range(workers)]
        dist.all_gather(allm, mt, group=group)
        masses = [float(x.item()) for x in allm]
    else:
        rank, workers, masses = 0, len(shards), mine
    total = float(sum(masses))
    if not abs(total - 1.0) <= norm_tol:  # statevec.py:226-228, on every rank
        raise UnnormalizedStateError(f"sharded norm^2 = {total!r}")
    per_rank = sv.split_shots(masses, shots, rng_seed, shards[0].device)
    idx_parts, cnt_parts = [], []
    for i, s in enumerate(samplers):
        r = rank if distributed else i
        idx, cnt = s.draw(per_rank[r], rng_seed, tag=2 + r)
        idx_parts.append(logical_indices(idx, phys_of_logical))
        cnt_parts.append(cnt)
    idx, cnt = torch.cat(idx_parts), torch.cat(cnt_parts)
    if distributed:
        k = _comm(torch.tensor([idx.numel()], dtype=torch.int64, device=idx.device), group)
        sizes = [torch.empty_like(k) for _ in range(workers)]
        dist.all_gather(sizes, k, group=group)
        mx = max(int(x.item()) for x in sizes)
        pair = torch.full((2, mx), -1, dtype=torch.int64, device=idx.device)
        pair[0, :idx.numel()] = idx
        pair[1, :idx.numel()] = cnt
        pair = _comm(pair, group)
        parts = [torch.empty_like(pair) for _ in range(workers)] if rank == 0 else None
        dist.gather(pair, parts, dst=0, group=group)
        if rank != 0:
            return None
        allp = torch.cat([p[:, :int(sz.item())] for p, sz in zip(parts, sizes)], dim=1)
        idx, cnt = allp[0], allp[1]
    order = torch.argsort(idx)
    return idx[order], cnt[order]


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
    sampled = None
    if distributed:
        rank = dist.get_rank(group)
        dev = torch.device("cuda", torch.cuda.current_device())
        shard = torch.empty(1 << n_local, dtype=dtype, device=dev)
        sv.N.call("qg_state_init_zero", sv.C.c_void_p(shard.data_ptr()), n_local, sv._QG_DTYPE[options.precision],
                  rank, sv._stream(dev))
        staging = None
        fp = plan_fingerprint(gt, gp, n, workers)
        for seg in range(plan.n_segments):
            plan.execute_segment(seg, shard, rank)
            if seg < plan.n_segments - 1:
                gpos, lpos = plan.remaps[seg]
                if delay_hook is not None:
                    delay_hook(rank, seg)
                check_step(seg, fp, group, device=dev)
                try:
                    sent[rank] += remap_dist(shard, n_local, gpos, lpos, rank, group, staging)
                except Exception as e:
                    raise ProtocolViolationError(f"remap {seg} failed: {e}") from e
        check_step(plan.n_segments, fp, group, final=True, device=dev)
        counts_all = _comm(torch.tensor(sent, dtype=torch.int64, device=dev), group)
        dist.all_reduce(counts_all, group=group)
        sent = counts_all.cpu().tolist()
        shards = [shard]
        state = None
        if options.shots > 0:  # sampled where the shards live; no state gather
            res = sample_shards(shards, n_local, plan.final_map, options.shots, options.rng_seed,
                                sv.NORM_TOL[options.precision], ranks=rank, group=group)
            if res is not None:
                sampled = sv.counts_from_arrays(res[0].cpu().numpy(), res[1].cpu().numpy(), options.shots, n)
        if gather:
            host = _host_wire(group)
            mine = torch.view_as_real(shard)  # complex blocks travel as (re, im) pairs
            mine = mine.cpu() if host else mine
            parts = [torch.empty_like(mine) for _ in range(workers)] if rank == 0 else None
            dist.gather(mine, parts, dst=0, group=group)
            if rank == 0:
                full = torch.view_as_complex(torch.cat(parts).to(dev))
                full = _permute_to_logical(full, n, plan.final_map)
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
        if options.shots > 0 and (not gather or options.sampler == "tree"):
            res = sample_shards(shards, n_local, plan.final_map, options.shots, options.rng_seed,
                                sv.NORM_TOL[options.precision])
            sampled = sv.counts_from_arrays(res[0].cpu().numpy(), res[1].cpu().numpy(), options.shots, n)
    counts = sampled
    if state is not None:
        nsq = state.norm_sq()
        if abs(nsq - 1.0) > sv.NORM_TOL[options.precision]:
            raise UnnormalizedStateError(f"gathered norm^2 = {nsq!r}")  # partition.py:139-140
        if options.shots > 0 and counts is None:
            counts = sv.sample_counts(state, options.shots, options.rng_seed, options.sampler)
    if len(set(sent)) > 1 and not distributed:
        raise SequenceMismatchError(f"workers exchanged different message counts: {sent}")
    return DistributedResult(state=state, counts=counts, messages_sent=sent, messages_received=list(sent),
                             tasks=dict(plan.info, remaps=plan.remaps), shards=shards)
