"""numpy restatement of the reference single-worker simulator (TEST ORACLE).

Follows /root/reference/pkg/src/qgear/statevec.py line by line in arithmetic
(same dtype casts, same operation order) so that fp64 AND fp32 results are
bit-identical to the reference; the structure is array-first (the circuit is
the (d,3) int32 gate_type + (d,) f64 gate_param pair of ir.py:281-303) instead
of GateRecord objects.  See oracle/__init__.py for the usage rule.
"""

from __future__ import annotations

import math

import numpy as np

# statevec.py:34-38
DTYPE = {"fp32": np.complex64, "fp64": np.complex128}
NORM_TOL = {"fp32": 1e-3, "fp64": 1e-9}

H, RX, RY, RZ, CX, CR1, MEASURE = range(7)  # ir.py:31-40


def gate_matrix(kind: int, param: float) -> np.ndarray:
    """Half-angle 2x2 in complex128 — statevec.py:97-110."""
    if kind == H:
        r = 1.0 / math.sqrt(2.0)
        return np.array([[r, r], [r, -r]], dtype=np.complex128)
    h = param / 2.0
    c, s = math.cos(h), math.sin(h)
    if kind == RX:
        return np.array([[c, -1j * s], [-1j * s, c]], dtype=np.complex128)
    if kind == RY:
        return np.array([[c, -s], [s, c]], dtype=np.complex128)
    if kind == RZ:
        return np.array([[np.exp(-1j * h), 0.0], [0.0, np.exp(1j * h)]], dtype=np.complex128)
    raise ValueError(f"kind {kind} has no 2x2 matrix")


def apply_pair_matrix(psi: np.ndarray, t: int, u: np.ndarray) -> None:
    """Dense 2x2 on every (bit t = 0, bit t = 1) pair, in place — statevec.py:115-122.

    The matrix is cast to the state dtype first (statevec.py:117), then each
    output is u_r0*lo + u_r1*hi evaluated in that dtype.
    """
    m = u.astype(psi.dtype, copy=False)
    blocks = psi.reshape(-1, 2, 1 << t)
    lo = blocks[:, 0, :].copy()
    hi = blocks[:, 1, :]
    blocks[:, 0, :] = m[0, 0] * lo + m[0, 1] * hi
    blocks[:, 1, :] = m[1, 0] * lo + m[1, 1] * hi


def _pair_view(psi: np.ndarray, q1: int, q2: int) -> np.ndarray:
    """5-D view (hi-bit, middle, lo-bit, low) over two distinct qubits."""
    a, b = max(q1, q2), min(q1, q2)
    return psi.reshape(-1, 2, 1 << (a - b - 1), 2, 1 << b)


def apply_cx_swap(psi: np.ndarray, c: int, t: int) -> None:
    """CX: exchange target-bit halves where the control bit is 1 — statevec.py:125-137."""
    v = _pair_view(psi, c, t)
    if c > t:
        lo, hi = v[:, 1, :, 0, :], v[:, 1, :, 1, :]
    else:
        lo, hi = v[:, 0, :, 1, :], v[:, 1, :, 1, :]
    keep = lo.copy()
    lo[...] = hi
    hi[...] = keep


def apply_cr1_phase(psi: np.ndarray, c: int, t: int, lam: float) -> None:
    """CR1: amplitudes with both bits set times exp(i lam) — statevec.py:140-144.

    The factor is a numpy complex128 scalar; for complex64 states numpy
    evaluates the product in complex128 and casts back (same as reference).
    """
    _pair_view(psi, c, t)[:, 1, :, 1, :] *= np.exp(1j * lam)


def trailing_body(kinds: np.ndarray) -> int:
    """Length of the gate body before the trailing MEASURE block — statevec.py:187-197.

    Raises ValueError (the reference raises MeasureMidCircuitError) when a
    MEASURE is followed by a non-MEASURE record.
    """
    meas = np.flatnonzero(kinds == MEASURE)
    if meas.size == 0:
        return int(kinds.size)
    first = int(meas[0])
    if np.any(kinds[first:] != MEASURE):
        raise ValueError("MEASURE records must form a trailing block")
    return first


def apply_gate(psi: np.ndarray, kind: int, ctrl: int, tgt: int, param: float) -> None:
    """Dispatch one live record — statevec.py:177-184."""
    if kind == CX:
        apply_cx_swap(psi, ctrl, tgt)
    elif kind == CR1:
        apply_cr1_phase(psi, ctrl, tgt, param)
    elif kind == MEASURE:
        return
    else:
        apply_pair_matrix(psi, tgt, gate_matrix(kind, param))


def zero_state(n: int, precision: str) -> np.ndarray:
    """|0...0> — statevec.py:81-94 (budget check left to callers)."""
    psi = np.zeros(1 << n, dtype=DTYPE[precision])
    psi[0] = 1.0
    return psi


def run_arrays(gate_type: np.ndarray, gate_param: np.ndarray, n_qubits: int, n_gates: int,
               precision: str = "fp64") -> np.ndarray:
    """run_circuit (statevec.py:200-212) on the array form; returns the amplitudes."""
    gt = np.asarray(gate_type, dtype=np.int64)[:n_gates]
    gp = np.asarray(gate_param, dtype=np.float64)[:n_gates]
    body = trailing_body(gt[:, 0])
    psi = zero_state(n_qubits, precision)
    for i in range(body):
        apply_gate(psi, int(gt[i, 0]), int(gt[i, 1]), int(gt[i, 2]), float(gp[i]))
    return psi


def exact_probabilities(psi: np.ndarray) -> np.ndarray:
    """|a|^2 accumulated in float64 — statevec.py:215-218."""
    return psi.real.astype(np.float64) ** 2 + psi.imag.astype(np.float64) ** 2


def sample_counts_arrays(psi: np.ndarray, shots: int, seed: int, precision: str):
    """Multinomial draw, returned as sorted (index, count) arrays — statevec.py:221-234.

    numpy's Generator.choice(p=...) is cumsum -> divide by last -> random(shots)
    -> searchsorted(side='right'); calling choice itself keeps the stream identical.
    """
    if shots < 1:
        raise ValueError(f"shots must be >= 1, got {shots}")
    p = exact_probabilities(psi)
    tot = p.sum()
    if abs(tot - 1.0) > NORM_TOL[precision]:
        raise ArithmeticError(f"norm^2 = {tot!r} outside tolerance")
    p = p / tot
    draws = np.random.default_rng(seed).choice(p.size, size=shots, p=p)
    idx, cnt = np.unique(draws, return_counts=True)
    return idx.astype(np.int64), cnt.astype(np.int64)


def bitstring(index: int, n: int) -> str:
    """qubit 0 leftmost — statevec.py:71-73."""
    return "".join("1" if (index >> k) & 1 else "0" for k in range(n))
