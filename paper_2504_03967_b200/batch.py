"""Batched circuit execution (the paper's multi-QPU "mqpu" mode, PAPER.md:231,
SPEC.md:353/504/576): a CircuitSet (ir.py:165-180, the container's unit) is run
circuit by circuit on the B200s.

* Plan reuse.  Circuits whose live gate_type rows are identical (the batched
  parameter sets of one ansatz, e.g. QCrank images or a parameter sweep) share
  one plan: the first is scheduled, the others only rebind their gate_param
  (`CompiledCircuit.rebind` -> qg_plan_rebind: same schedule, new program).
* Concurrency.  Circuits run round-robin on `streams` CUDA streams, each with
  its own state buffer, so small circuits overlap on one GPU.
* Multi-GPU.  Under torch.distributed, rank r runs circuits r, r + W, ...
  (no data-path collective: the circuits are independent) and the per-circuit
  results are gathered to every rank (`all_gather_object`, counts only).

Each result carries the counts (shots > 0) and, with keep_states=True, the
final state (device tensor; memory permitting).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import statevec as sv
from .ir import CircuitSet, set_to_arrays


@dataclass
class BatchResult:
    index: int
    n_qubits: int
    counts: sv.CountsTable | None
    state: sv.StateVector | None
    norm_sq: float
    rank: int = 0
    planned: bool = True       # False: reused another circuit's schedule (rebind)


def assign_circuits(n_circuits: int, world: int, rank: int) -> list[int]:
    """Circuits owned by `rank` when `world` ranks share a batch (round-robin)."""
    return list(range(rank, n_circuits, world))


def _live(gt_row: np.ndarray, gp_row: np.ndarray, n_gates: int):
    gt = np.ascontiguousarray(gt_row[:n_gates], dtype=np.int32)
    gp = np.ascontiguousarray(gp_row[:n_gates], dtype=np.float64)
    return gt, gp


def run_circuit_set(circuit_set: CircuitSet, options: sv.SimOptions | None = None, keep_states: bool = False,
                    streams: int = 4, indices: list[int] | None = None) -> list[BatchResult]:
    """Run `indices` (default: all) of a CircuitSet on this process's GPU."""
    options = options or sv.SimOptions()
    headers, gate_type, gate_param = set_to_arrays(circuit_set)
    todo = list(range(headers.shape[0])) if indices is None else list(indices)
    dev = sv._device(options.device)
    pool = [torch.cuda.Stream(dev) for _ in range(max(1, streams))]
    plans: dict[bytes, sv.CompiledCircuit] = {}
    buffers: dict[tuple[int, int], sv.StateVector] = {}
    results = []
    for k, i in enumerate(todo):
        _, n, ng = (int(v) for v in headers[i])
        gt, gp = _live(gate_type[i], gate_param[i], ng)
        nb = sv._trailing_split_arrays(gt[:, 0])
        s = pool[k % len(pool)]
        with torch.cuda.stream(s):
            if options.fuse and nb >= 32:
                from . import qcrank

                if any(it[0] == "ucry" for it in qcrank.collapse_ucry(gt[:nb], gp[:nb])):
                    st, counts = qcrank.run_gates(gt, gp, n, options)
                    results.append(BatchResult(i, n, counts, st if keep_states else None, st.norm_sq()))
                    continue
            sv._check_budget(n, options.precision, options.memory_budget)
            key = bytes(np.int64(n).tobytes()) + gt[:nb].tobytes()
            planned = key not in plans
            if planned:
                plans[key] = sv.CompiledCircuit(gt, gp, n, options.precision, 0, options.fuse,
                                                options.tile_qubits, options.max_stages, options.max_cost, jit=options.jit)
            else:
                plans[key].rebind(gp[:nb])
            plan = plans[key]
            if keep_states:
                st = sv.init_zero_state(n, options.precision, options.memory_budget, options.device)
            else:  # reuse one buffer per (stream, size)
                bkey = (k % len(pool), n)
                st = buffers.get(bkey)
                if st is None:
                    st = sv.init_zero_state(n, options.precision, options.memory_budget, options.device)
                    buffers[bkey] = st
                else:
                    sv.N.call("qg_state_init_zero", sv.C.c_void_p(st.amplitudes.data_ptr()), n,
                              sv._QG_DTYPE[options.precision], 0, sv._stream(dev))
            plan.execute(st)
            counts = None
            if options.shots > 0:
                counts = sv.sample_counts(st, options.shots, options.rng_seed + i, options.sampler)
            results.append(BatchResult(i, n, counts, st if keep_states else None, st.norm_sq(), planned=planned))
    torch.cuda.synchronize(dev)
    return results


def run_circuit_set_distributed(circuit_set: CircuitSet, options: sv.SimOptions | None = None,
                                streams: int = 4) -> list[BatchResult]:
    """All ranks of the default torch.distributed group share the batch (weak
    scaling); every rank returns the full, index-ordered result list (counts)."""
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    mine = assign_circuits(len(circuit_set.circuits), world, rank)
    local = run_circuit_set(circuit_set, options, keep_states=False, streams=streams, indices=mine)
    for r in local:
        r.rank = rank
    if world == 1:
        return local
    gathered: list = [None] * world
    dist.all_gather_object(gathered, local)
    out = [r for part in gathered for r in part]
    out.sort(key=lambda r: r.index)
    return out
