"""numpy interpreter of an exported fused program (test helper, CPU only).

Applies the op records of CompiledCircuit.export() to a full state vector with
the SAME semantics the CUDA kernel implements (include/qgear_b200.h,
paper_2504_03967_b200/csrc/desc.h): register-level ops act on physical qubit
positions, thread-phase ops (OP_TPHASE) are accumulated and applied at the end
of their register stage, remaps between segments swap physical positions.
This checks the planner (scheduling, commutation, fusion, remaps) on a CPU box.
"""

from __future__ import annotations

import numpy as np

OP_DENSE, OP_DIAG, OP_X, OP_CX, OP_CPHASE, OP_TPHASE = range(6)


def _bit(idx, q):
    return (idx >> q) & 1


def _cond(idx, cmask):
    return (idx & cmask) == cmask


def _apply_2x2(psi, idx, t, m, sel):
    lo = np.flatnonzero((_bit(idx, t) == 0) & sel)
    hi = lo | (1 << t)
    a, b = psi[lo].copy(), psi[hi].copy()
    psi[lo] = m[0, 0] * a + m[0, 1] * b
    psi[hi] = m[1, 0] * a + m[1, 1] * b


def _swap_positions(psi, n, p1, p2):
    """Exchange physical index bits p1 and p2 (a remap on the full vector)."""
    idx = np.arange(psi.size, dtype=np.int64)
    b1, b2 = _bit(idx, p1), _bit(idx, p2)
    src = idx ^ ((b1 ^ b2) << p1) ^ ((b1 ^ b2) << p2)
    return psi[src]


def run_program(plan, dtype=np.complex128) -> np.ndarray:
    """Full 2^n state (logical order) after executing `plan` (a CompiledCircuit)."""
    n = plan.n_qubits
    rec, mats = plan.export()
    psi = np.zeros(1 << n, dtype=dtype)
    psi[0] = 1
    idx = np.arange(1 << n, dtype=np.int64)
    remaps = list(plan.remaps)
    last_pass = -1
    pending_phase = np.ones(1 << n, dtype=np.complex128)
    cur_stage = None

    def flush():
        nonlocal pending_phase
        psi[:] = psi * pending_phase.astype(dtype)
        pending_phase = np.ones(1 << n, dtype=np.complex128)

    for r in rec:
        p, s, kind, tq, cq, cmask, qmask, mi = (int(v) for v in r)
        if cur_stage is not None and (p, s) != cur_stage:
            flush()
        cur_stage = (p, s)
        if p > last_pass + 1:
            # a skipped pass id marks a segment boundary -> apply the remap(s) in between
            for _ in range(p - last_pass - 1):
                g, loc = remaps.pop(0)
                for a, b in zip(g, loc):
                    psi = _swap_positions(psi, n, a, b)
        last_pass = p
        m = mats[mi]
        c = lambda k: complex(m[2 * k], m[2 * k + 1])  # noqa: E731
        sel = _cond(idx, cmask)
        if kind in (OP_DENSE, 100):
            u = np.array([[c(0), c(1)], [c(2), c(3)]], dtype=np.complex128).astype(dtype)
            _apply_2x2(psi, idx, tq, u, sel)
        elif kind == OP_DIAG:
            d = np.where(_bit(idx, tq) == 1, c(1), c(0))
            psi[sel] = psi[sel] * d[sel].astype(dtype)
        elif kind in (OP_X, OP_CX):
            if kind == OP_CX:
                sel = sel & (_bit(idx, cq) == 1)
            _apply_2x2(psi, idx, tq, np.array([[0, 1], [1, 0]], dtype=dtype), sel)
        elif kind == OP_CPHASE:
            both = (_bit(idx, tq) == 1) & (_bit(idx, cq) == 1) & sel
            psi[both] = psi[both] * dtype(c(0))
        elif kind == OP_TPHASE:
            v = np.where((idx & qmask) != 0, c(1), c(0))
            pending_phase = np.where(sel, pending_phase * v, pending_phase)
        elif kind == 101:
            v = np.where((idx & qmask) != 0, c(1), c(0))
            psi[sel] = psi[sel] * v[sel].astype(dtype)
        else:
            raise AssertionError(f"unknown op kind {kind}")
    flush()
    while remaps:  # trailing remaps (no passes after them)
        g, loc = remaps.pop(0)
        for a, b in zip(g, loc):
            psi = _swap_positions(psi, n, a, b)
    # physical -> logical order: logical qubit q sits at physical position final_map[q]
    fm = np.asarray(plan.final_map)
    if np.any(fm != np.arange(n)):
        src = np.zeros(1 << n, dtype=np.int64)
        for q in range(n):
            src |= _bit(idx, q) << int(fm[q])
        psi = psi[src]
    return psi
