"""Workload generators producing the reference's gate streams directly as arrays.

Bit-identical to /root/reference/pkg/src/qgear/generators.py (checked against
tests/golden/golden.npz): the PCG64 draws are made in the same order and with
the same calls (generators.py:67-73), but the output is the (d,3) int32 /
(d,) f64 array pair the executor consumes, so 10^3..10^8-gate circuits never
build GateRecord objects.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import TooFewQubitsError
from .ir import NO_CONTROL, CircType, CircuitTensor, GateKind

TWO_PI = 2.0 * math.pi


@dataclass(frozen=True)
class RandomSpec:
    """generators.py:21-33."""

    n_qubits: int
    n_blocks: int
    seed: int = 0
    include_measure: bool = False


@dataclass(frozen=True)
class QftSpec:
    """generators.py:36-39."""

    n_qubits: int
    reversed: bool = False


def _pair_from_flat(u, n: int):
    control, r = np.divmod(np.asarray(u, dtype=np.int64), n - 1)
    target = np.where(r < control, r, r + 1)
    return control, target


def random_qubit_pairs(n_qubits: int, k: int, seed: int = 0) -> list[tuple[int, int]]:
    """generators.py:42-58 (one vector draw of k flat pair ids)."""
    if n_qubits < 2:
        raise TooFewQubitsError(f"need >= 2 qubits for pairs, got {n_qubits}")
    if k < 0:
        raise ValueError(f"k must be >= 0, got {k}")
    flat = np.random.default_rng(seed).integers(0, n_qubits * (n_qubits - 1), size=k)
    c, t = _pair_from_flat(flat, n_qubits)
    return list(zip(c.tolist(), t.tolist()))


def random_arrays(spec: RandomSpec) -> tuple[np.ndarray, np.ndarray]:
    """Gate arrays of generate_random_gate_list (generators.py:61-79).

    Per block the reference draws one bounded integer then a size-2 uniform;
    PCG64 buffers half-words between those calls, so the draws are made
    block by block exactly as there, and only the array fill is vectorised.
    """
    n, b = spec.n_qubits, spec.n_blocks
    if n < 2:
        raise TooFewQubitsError(f"need >= 2 qubits, got {n}")
    if b < 0:
        raise ValueError(f"n_blocks must be >= 0, got {b}")
    rng = np.random.default_rng(spec.seed)
    n_pairs = n * (n - 1)
    flat = np.empty(b, dtype=np.int64)
    ang = np.empty((b, 2), dtype=np.float64)
    for i in range(b):
        flat[i] = rng.integers(0, n_pairs)
        ang[i] = rng.uniform(0.0, TWO_PI, size=2)
    c, t = _pair_from_flat(flat, n)
    m = n if spec.include_measure else 0
    gt = np.empty((3 * b + m, 3), dtype=np.int32)
    gp = np.zeros(3 * b + m, dtype=np.float64)
    gt[0:3 * b:3] = np.stack([np.full(b, GateKind.RY), np.full(b, NO_CONTROL), c], axis=1)
    gt[1:3 * b:3] = np.stack([np.full(b, GateKind.RZ), np.full(b, NO_CONTROL), t], axis=1)
    gt[2:3 * b:3] = np.stack([np.full(b, GateKind.CX), c, t], axis=1)
    gp[0:3 * b:3] = ang[:, 0]
    gp[1:3 * b:3] = ang[:, 1]
    if m:
        gt[3 * b:] = np.stack([np.full(m, GateKind.MEASURE), np.full(m, NO_CONTROL), np.arange(m)], axis=1)
    return gt, gp


def generate_random_gate_list(spec: RandomSpec) -> CircuitTensor:
    gt, gp = random_arrays(spec)
    return CircuitTensor.from_arrays(CircType.RANDOM, spec.n_qubits, gt, gp)


def qft_arrays(n: int, reversed: bool = False) -> tuple[np.ndarray, np.ndarray]:
    """Gate arrays of build_qft (generators.py:82-101): H(q(i)) then CR1(q(j)->q(i), 2pi/2^(j-i+1))."""
    if n < 1:
        raise ValueError(f"n_qubits must be >= 1, got {n}")
    rows, params = [], []
    for i in range(n):
        qi = n - 1 - i if reversed else i
        rows.append((GateKind.H, NO_CONTROL, qi))
        params.append(0.0)
        for j in range(i + 1, n):
            qj = n - 1 - j if reversed else j
            rows.append((GateKind.CR1, qj, qi))
            params.append(TWO_PI / (1 << (j - i + 1)))
    return np.array(rows, dtype=np.int32).reshape(-1, 3), np.array(params, dtype=np.float64)


def build_qft(spec: QftSpec) -> CircuitTensor:
    gt, gp = qft_arrays(spec.n_qubits, spec.reversed)
    return CircuitTensor.from_arrays(CircType.QFT, spec.n_qubits, gt, gp)
