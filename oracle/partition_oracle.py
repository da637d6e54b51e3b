"""numpy + threads restatement of the reference partitioned executor (TEST ORACLE).

Follows /root/reference/pkg/src/qgear/partition.py:
  chunking / partner masks      partition.py:82-109
  local gates, id-bit controls  partition.py:144-155, 196-198, 218-232
  exchange arithmetic           partition.py:234-263
  lockstep + barrier            partition.py:265-274
  gather + central sampling     partition.py:121-141, 345-348

Instead of per-worker inboxes (partition.py:200-216) the workers publish
their payload for sequence s into a shared slot and read the partner's slot
between two barrier waits; the arithmetic on every amplitude is the
reference's, so the gathered state is bit-identical to it (and to the
single-worker run).  Also used as the multi-core CPU baseline (fp64 only, as
the reference enforces at partition.py:300-301).
"""

from __future__ import annotations

import threading

import numpy as np

from .statevec_oracle import (
    CR1,
    CX,
    NORM_TOL,
    apply_cr1_phase,
    apply_cx_swap,
    apply_pair_matrix,
    gate_matrix,
    sample_counts_arrays,
    trailing_body,
    zero_state,
)


def partner_masks(n: int, workers: int, targets: np.ndarray) -> np.ndarray:
    """0 for a local target, else 1 << (t - n_local) — partition.py:94-97."""
    if workers < 1 or workers & (workers - 1) or workers > (1 << n):
        raise ValueError(f"bad worker count {workers}")
    n_local = n - (workers.bit_length() - 1)
    t = np.asarray(targets, dtype=np.int64)
    return np.where(t < n_local, 0, np.left_shift(1, np.maximum(t - n_local, 0)))


def _flip(chunk: np.ndarray, t: int) -> None:
    v = chunk.reshape(-1, 2, 1 << t)
    keep = v[:, 0, :].copy()
    v[:, 0, :] = v[:, 1, :]
    v[:, 1, :] = keep


def _phase_bit(chunk: np.ndarray, q: int, lam: float) -> None:
    chunk.reshape(-1, 2, 1 << q)[:, 1, :] *= np.exp(1j * lam)


def execute_partitioned(gate_type, gate_param, n_qubits: int, n_gates: int, workers: int,
                        precision: str = "fp64", shots: int = 0, seed: int = 0):
    """Returns (state, counts (idx,cnt) or None, messages_sent per worker, partner masks)."""
    if workers > 1 and precision != "fp64":
        raise ValueError("distributed mode supports fp64 only")  # partition.py:300-301
    gt = np.asarray(gate_type, dtype=np.int64)[:n_gates]
    gp = np.asarray(gate_param, dtype=np.float64)[:n_gates]
    body = trailing_body(gt[:, 0])
    gt, gp = gt[:body], gp[:body]
    masks = partner_masks(n_qubits, workers, gt[:, 2])
    full = zero_state(n_qubits, precision)
    L = full.size // workers
    n_local = L.bit_length() - 1
    chunks = [full[w * L:(w + 1) * L].copy() for w in range(workers)]
    del full
    slots: list = [None] * workers
    sent = [0] * workers
    bar = threading.Barrier(workers)
    errors: list[BaseException] = []

    def idbit(w: int, q: int) -> int:
        return (w >> (q - n_local)) & 1

    def worker(w: int) -> None:
        ch = chunks[w]
        empty = ch[:0]
        for i in range(body):
            k, c, t, lam = int(gt[i, 0]), int(gt[i, 1]), int(gt[i, 2]), float(gp[i])
            m = int(masks[i])
            if m == 0:  # partition.py:218-232
                if k == CX:
                    if c < n_local:
                        apply_cx_swap(ch, c, t)
                    elif idbit(w, c):
                        _flip(ch, t)
                elif k == CR1:
                    if c < n_local:
                        apply_cr1_phase(ch, c, t, lam)
                    elif idbit(w, c):
                        _phase_bit(ch, t, lam)
                else:
                    apply_pair_matrix(ch, t, gate_matrix(k, lam))
                continue
            p = w ^ m  # partition.py:234-263
            if k == CX:
                if c < n_local:
                    sel = ch.reshape(-1, 2, 1 << c)[:, 1, :]
                    payload = sel.copy()
                elif idbit(w, c):
                    payload = ch.copy()
                else:
                    payload = empty
            elif k == CR1:
                payload = empty
            else:
                payload = ch.copy()
            slots[w] = payload
            sent[w] += 1
            bar.wait(timeout=60)
            theirs = slots[p]
            bar.wait(timeout=60)
            if k == CX:
                if c < n_local:
                    ch.reshape(-1, 2, 1 << c)[:, 1, :] = theirs.reshape(-1, 1 << c)
                elif idbit(w, c):
                    ch[:] = theirs
            elif k == CR1:
                if idbit(w, t):
                    if c < n_local:
                        _phase_bit(ch, c, lam)
                    elif idbit(w, c):
                        ch *= np.exp(1j * lam)
            else:
                u = gate_matrix(k, lam).astype(ch.dtype, copy=False)
                if idbit(w, t) == 0:
                    ch[:] = u[0, 0] * ch + u[0, 1] * theirs
                else:
                    ch[:] = u[1, 0] * theirs + u[1, 1] * ch

    def guarded(w: int) -> None:
        try:
            worker(w)
        except BaseException as exc:  # surfaced below
            errors.append(exc)
            bar.abort()

    if workers == 1:
        worker(0)
    else:
        ths = [threading.Thread(target=guarded, args=(w,), daemon=True) for w in range(workers)]
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        if errors:
            raise errors[0]
    state = np.concatenate(chunks)
    p = state.real.astype(np.float64) ** 2 + state.imag.astype(np.float64) ** 2
    if abs(p.sum() - 1.0) > NORM_TOL[precision]:
        raise ArithmeticError("gathered norm outside tolerance")
    counts = sample_counts_arrays(state, shots, seed, precision) if shots > 0 else None
    return state, counts, sent, masks
