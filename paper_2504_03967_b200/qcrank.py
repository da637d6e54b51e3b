"""QCrank grayscale-image encoding on the B200 simulator.

The reference specifies QCrank (§Results, App. D.3,
App. F; errors PlanTooSmallError / LengthMismatchError at errors.py:93-101;
ir.CircType.QCRANK at ir.py:52) but ships no implementation, so this module
follows the spec's operations and examples:

  prepare_angles       v = 2p/255 - 1, theta = arccos v, pixel group g -> address
                       bitrev_m(g), padding theta = pi/2
  build_qcrank_circuit H on the m address qubits, then per data qubit one
                       uniformly controlled RY as the Gray-code block of 2^m RY
                       (Walsh-Hadamard-in-Gray-order angles, 2^-m scaled) and
                       2^m CX, trailing MEASURE
  decode_counts /      v = (n0 - n1) / (n0 + n1) per address and data lane,
  decode_exact         p = round(255 (v + 1) / 2)

Qubit layout (the spec leaves it open): address qubits 0..m-1 (address index
bit k = qubit k), data qubit d = qubit m + d.

Execution.  The gate form is 2 * n_data * 2^m gates (2.7e8 for the 24 + 8
configuration); `collapse_ucry` recognises every Gray-code UCRY block in a gate
array and recovers its per-address angles (the inverse transform), and
`run_gates` executes the circuit as fused-pass segments (libqgear_b200 planner)
interleaved with one-pass uniformly-controlled-RY kernels (`qg_apply_ucry`,
up to 5 data qubits per HBM pass).  Arrays throughout: no GateRecord objects.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import statevec as sv
from .errors import IndexOutOfRangeError, LengthMismatchError, PlanTooSmallError
from .ir import CircType, GateKind

SHOTS_PER_ADDRESS = 3000


@dataclass(frozen=True)
class ImageGray:
    """Row-major 8-bit grayscale image."""

    width: int
    height: int
    pixels: np.ndarray

    def __post_init__(self):
        px = np.ascontiguousarray(self.pixels, dtype=np.uint8).reshape(-1)
        if self.width < 1 or self.height < 1 or px.size != self.width * self.height:
            raise ValueError(f"{px.size} pixels for a {self.width}x{self.height} image")
        object.__setattr__(self, "pixels", px)


@dataclass(frozen=True)
class QCrankPlan:
    """m address qubits x n_data data qubits."""

    n_addr: int
    n_data: int
    width: int = 0
    height: int = 0
    shots_per_address: int = SHOTS_PER_ADDRESS

    @property
    def padded_len(self) -> int:
        return (1 << self.n_addr) * self.n_data

    @property
    def n_qubits(self) -> int:
        return self.n_addr + self.n_data

    @property
    def shots(self) -> int:
        return self.shots_per_address << self.n_addr


@dataclass
class ReconstructionReport:
    """per-pixel estimates and fidelity metrics vs the source."""

    estimates: np.ndarray              # v-hat per pixel (row-major), clamped to [-1, 1]
    correlation: float | None = None
    mse: float | None = None
    max_abs_error: float | None = None
    empty_addresses: list = field(default_factory=list)


def make_plan(image: ImageGray, n_addr: int, n_data: int, shots_per_address: int = SHOTS_PER_ADDRESS) -> QCrankPlan:
    plan = QCrankPlan(n_addr, n_data, image.width, image.height, shots_per_address)
    if n_addr < 0 or n_data < 1 or plan.padded_len < image.pixels.size:
        raise PlanTooSmallError(f"2^{n_addr} x {n_data} = {plan.padded_len} slots < {image.pixels.size} pixels")
    return plan


def bitrev(x: np.ndarray | int, m: int):
    """Reverse the m low bits (SPEC.md:457 'reversed addressing qubits')."""
    x = np.asarray(x, dtype=np.int64)
    r = np.zeros_like(x)
    for k in range(m):
        r |= ((x >> k) & 1) << (m - 1 - k)
    return r


def prepare_angles(image: ImageGray, n_addr: int, n_data: int) -> np.ndarray:
    """AngleTensor (2^m, n_data): pixel k -> group g = k // n_data, lane k % n_data,
    address bitrev_m(g); theta = arccos(2p/255 - 1); padding pi/2."""
    make_plan(image, n_addr, n_data)
    n_slots = (1 << n_addr) * n_data
    theta = np.full(n_slots, math.pi / 2)
    v = 2.0 * image.pixels.astype(np.float64) / 255.0 - 1.0
    k = np.arange(image.pixels.size, dtype=np.int64)
    addr = bitrev(k // n_data, n_addr)
    theta[addr * n_data + k % n_data] = np.arccos(np.clip(v, -1.0, 1.0))
    return theta.reshape(1 << n_addr, n_data)


def _gray(i: np.ndarray) -> np.ndarray:
    return i ^ (i >> 1)


def _fwht(x: np.ndarray) -> np.ndarray:
    """Unnormalised Walsh-Hadamard transform along axis 0 (natural order)."""
    y = np.array(x, dtype=np.float64, copy=True)
    h = 1
    n = y.shape[0]
    while h < n:
        y = y.reshape(n // (2 * h), 2, h, *y.shape[1:])
        a, b = y[:, 0].copy(), y[:, 1].copy()
        y[:, 0], y[:, 1] = a + b, a - b
        y = y.reshape(n, *y.shape[3:])
        h *= 2
    return y


def gray_walsh(alpha: np.ndarray) -> np.ndarray:
    """Per-address angles alpha[a] -> Gray-block rotation angles theta_hat[i] =
    2^-m sum_a (-1)^popcount(a & gray(i)) alpha[a]."""
    alpha = np.asarray(alpha, dtype=np.float64)
    n = alpha.shape[0]
    w = _fwht(alpha)
    return w[_gray(np.arange(n))] / n


def inverse_gray_walsh(theta_hat: np.ndarray) -> np.ndarray:
    """alpha[a] = sum_i (-1)^popcount(a & gray(i)) theta_hat[i] (the block's net angle)."""
    theta_hat = np.asarray(theta_hat, dtype=np.float64)
    n = theta_hat.shape[0]
    v = np.zeros_like(theta_hat)
    v[_gray(np.arange(n))] = theta_hat
    return _fwht(v)


def gray_controls(m: int) -> np.ndarray:
    """Address bit whose CX follows rotation i: the bit changing from gray(i) to gray(i+1 mod 2^m)."""
    i = np.arange(1 << m, dtype=np.int64)
    nxt = _gray((i + 1) & ((1 << m) - 1))
    change = _gray(i) ^ nxt
    return np.log2(change).astype(np.int64)


def ucry_gate_arrays(alpha: np.ndarray, addr_qubits, target: int) -> tuple[np.ndarray, np.ndarray]:
    """Gray-code uniformly controlled RY: 2^m x (RY(theta_hat_i) on target, CX(addr[c_i] -> target))."""
    addr = np.asarray(addr_qubits, dtype=np.int32)
    m = addr.size
    th = gray_walsh(alpha)
    if m == 0:
        return np.array([[int(GateKind.RY), -1, target]], dtype=np.int32), th[:1].copy()
    ctrl = addr[gray_controls(m)]
    n = 1 << m
    gt = np.zeros((2 * n, 3), dtype=np.int32)
    gp = np.zeros(2 * n, dtype=np.float64)
    gt[0::2] = (int(GateKind.RY), -1, target)
    gt[1::2, 0] = int(GateKind.CX)
    gt[1::2, 1] = ctrl
    gt[1::2, 2] = target
    gp[0::2] = th
    return gt, gp


def build_qcrank_circuit(angles: np.ndarray, measure: bool = True) -> tuple[np.ndarray, np.ndarray, int]:
    """(gate_type, gate_param, n_qubits) of the QCrank circuit."""
    angles = np.asarray(angles, dtype=np.float64)
    n_addr_states, n_data = angles.shape
    m = n_addr_states.bit_length() - 1
    if 1 << m != n_addr_states:
        raise ValueError("angle tensor rows must be a power of two")
    n = m + n_data
    parts_t = [np.array([[int(GateKind.H), -1, q] for q in range(m)], dtype=np.int32).reshape(-1, 3)]
    parts_p = [np.zeros(m)]
    addr = list(range(m))
    for d in range(n_data):
        t, p = ucry_gate_arrays(angles[:, d], addr, m + d)
        parts_t.append(t)
        parts_p.append(p)
    if measure:
        parts_t.append(np.array([[int(GateKind.MEASURE), -1, q] for q in range(n)], dtype=np.int32))
        parts_p.append(np.zeros(n))
    return np.concatenate(parts_t), np.concatenate(parts_p), n


def cx_count(gate_type: np.ndarray) -> int:
    return int(np.count_nonzero(np.asarray(gate_type)[:, 0] == int(GateKind.CX)))


# ------------------------------------------------------------------ collapse + run
@dataclass
class UcrySegment:
    target: int
    addr_qubits: list
    alpha: np.ndarray   # (2^m,) net RY angle per address


def _block_at(gt: np.ndarray, gp: np.ndarray, start: int, pairs: int, min_addr: int):
    """Largest Gray-code UCRY block (m >= min_addr) at `start` within a run of
    `pairs` (RY(t), CX(*, t)) row pairs: (n_pairs_used, UcrySegment) or None."""
    target = int(gt[start, 2])
    m = pairs.bit_length() - 1
    while m >= min_addr:
        n = 1 << m
        ctrls = gt[start + 1:start + 2 * n:2, 1]
        bits = gray_controls(m)
        first = np.array([int(np.argmax(bits == b)) for b in range(m)])
        addr = ctrls[first]
        if len(set(addr.tolist())) == m and target not in addr and np.array_equal(ctrls, addr[bits]):
            return n, UcrySegment(target, addr.tolist(), inverse_gray_walsh(gp[start:start + 2 * n:2]))
        m -= 1
    return None


def _pair_runs(gt: np.ndarray, min_pairs: int):
    """(start row, pairs) of maximal runs of (RY(t), CX(*, t)) row pairs on one t."""
    k, t = gt[:, 0], gt[:, 2]
    if k.size < 2:
        return []
    pair = (k[:-1] == GateKind.RY) & (k[1:] == GateKind.CX) & (t[:-1] == t[1:])
    runs = []
    for par in (0, 1):
        ok = pair[par::2]
        tt = t[par::2][:ok.size]
        cont = np.zeros(ok.size, dtype=bool)  # cont[j]: pair j continues the run of pair j - 1
        cont[1:] = ok[1:] & ok[:-1] & (tt[1:] == tt[:-1])
        starts = np.flatnonzero(ok & ~cont)
        ends = np.flatnonzero(ok & ~np.append(cont[1:], False))
        for j0, j1 in zip(starts.tolist(), ends.tolist()):
            if j1 - j0 + 1 >= min_pairs:
                runs.append((par + 2 * j0, j1 - j0 + 1))
    return sorted(runs)


def collapse_ucry(gate_type: np.ndarray, gate_param: np.ndarray, min_addr: int = 4):
    """Split a gate array into [("gates", gt, gp) | ("ucry", UcrySegment)] items,
    replacing every Gray-code uniformly controlled RY block over >= min_addr
    address qubits by one UCRY item (its angles recovered exactly up to fp64).
    Candidate runs are found with vectorised scans (2.7e8-row QCrank tensors)."""
    gt = np.asarray(gate_type, dtype=np.int32).reshape(-1, 3)
    gp = np.asarray(gate_param, dtype=np.float64).reshape(-1)
    items, last = [], 0
    for start, pairs in _pair_runs(gt, 1 << min_addr):
        if start < last:
            continue
        pos, left = start, pairs
        while left >= (1 << min_addr):
            hit = _block_at(gt, gp, pos, left, min_addr)
            if hit is None:
                pos, left = pos + 2, left - 1
                continue
            used, seg = hit
            if pos > last:
                items.append(("gates", gt[last:pos], gp[last:pos]))
            items.append(("ucry", seg))
            pos, left = pos + 2 * used, left - used
            last = pos
    if last < gt.shape[0] or not items:
        items.append(("gates", gt[last:], gp[last:]))
    return items


def apply_ucry(state: sv.StateVector, addr_qubits, targets, alpha) -> None:
    """RY(alpha[a, j]) on targets[j] for every address a (one HBM pass per 5 targets).
    alpha: (2^m, len(targets)) float64, numpy or a CUDA tensor (no host copy)."""
    amps = state.amplitudes
    n = sv._check_amps(amps)
    addr = np.ascontiguousarray(addr_qubits, dtype=np.int32)
    tg = np.ascontiguousarray(targets, dtype=np.int32)
    if not isinstance(alpha, torch.Tensor):
        alpha = torch.from_numpy(np.ascontiguousarray(alpha, dtype=np.float64))
    alpha = alpha.to(device=amps.device, dtype=torch.float64).reshape(1 << addr.size, tg.size)
    dt = sv._QG_DTYPE[state.precision]
    for j0 in range(0, tg.size, 5):
        tj = np.ascontiguousarray(tg[j0:j0 + 5])
        al = alpha[:, j0:j0 + 5].contiguous()
        ws_bytes = N.lib().qg_ucry_workspace_bytes(addr.size, tj.size, dt)
        if ws_bytes < 0:
            raise ValueError("bad UCRY register sizes")
        ws = torch.empty(max(ws_bytes, 16), dtype=torch.uint8, device=amps.device)
        N.call("qg_apply_ucry", C.c_void_p(amps.data_ptr()), n, dt, addr.ctypes.data_as(C.c_void_p), addr.size,
               tj.ctypes.data_as(C.c_void_p), tj.size, C.c_void_p(al.data_ptr()), C.c_void_p(ws.data_ptr()),
               ws.numel(), sv._stream(amps.device))


def run_gates(gate_type: np.ndarray, gate_param: np.ndarray, n_qubits: int, options: sv.SimOptions | None = None,
              min_addr: int = 4):
    """run_circuit for gate arrays with UCRY collapse: fused-pass segments + UCRY passes.
    Consecutive UCRY blocks over the same address register share one pass."""
    options = options or sv.SimOptions()
    gt = np.asarray(gate_type, dtype=np.int32).reshape(-1, 3)
    gp = np.asarray(gate_param, dtype=np.float64).reshape(-1)
    nb = sv._trailing_split_arrays(gt[:, 0])
    sv._check_budget(n_qubits, options.precision, options.memory_budget)
    lead, lead_mask = 0, 0
    while lead < nb and gt[lead, 0] == GateKind.H:
        q = int(gt[lead, 2])
        if not 0 <= q < n_qubits:  # the reference's _check_record order: range before anything else
            raise IndexOutOfRangeError(f"gate {lead}: target {q} outside [0, {n_qubits})")
        if (lead_mask >> q) & 1:
            break
        lead_mask |= 1 << q
        lead += 1
    if lead < 4:  # not worth a special case
        lead, lead_mask = 0, 0
    items = collapse_ucry(gt[lead:nb], gp[lead:nb], min_addr)
    plans = []
    for it in items:  # plan everything first: gate errors raise before any device work
        if it[0] == "gates":
            plans.append(sv.CompiledCircuit(it[1], it[2], n_qubits, options.precision, 0, options.fuse,
                                            options.tile_qubits, options.max_stages, options.max_cost, jit=options.jit))
    state = sv.init_zero_state(n_qubits, options.precision, options.memory_budget, options.device)
    if lead_mask:  # leading H layer on distinct qubits, applied to |0...0>: uniform superposition
        N.call("qg_state_init_uniform", C.c_void_p(state.amplitudes.data_ptr()), n_qubits,
               sv._QG_DTYPE[options.precision], C.c_uint64(lead_mask), 0, sv._stream(state.amplitudes.device))
    pi, k = 0, 0
    while k < len(items):
        if items[k][0] == "gates":
            plans[pi].execute(state)
            pi += 1
            k += 1
            continue
        group = [items[k][1]]
        while k + len(group) < len(items) and items[k + len(group)][0] == "ucry" and \
                items[k + len(group)][1].addr_qubits == group[0].addr_qubits:
            group.append(items[k + len(group)][1])
        apply_ucry(state, group[0].addr_qubits, [g.target for g in group],
                   np.stack([g.alpha for g in group], axis=1))
        k += len(group)
    counts = None
    if options.shots > 0:
        counts = sv.sample_counts(state, options.shots, options.rng_seed, options.sampler)
    return state, counts


def simulate(angles: np.ndarray, options: sv.SimOptions | None = None, state: sv.StateVector | None = None):
    """Run the QCrank circuit of an AngleTensor without materialising its gate
    arrays: the H layer on |0...0> is the uniform superposition of the address
    register (qg_state_init_uniform, one write pass), then the data register's
    uniformly controlled RYs (qg_apply_ucry, 5 data qubits per pass) — the
    kernels run_gates uses after collapse_ucry.  `state` (optional) is a reusable
    buffer of the right size (batched images)."""
    options = options or sv.SimOptions()
    if not isinstance(angles, torch.Tensor):
        angles = np.asarray(angles, dtype=np.float64)
    m = int(angles.shape[0]).bit_length() - 1
    nd = angles.shape[1]
    n = m + nd
    sv._check_budget(n, options.precision, options.memory_budget)
    if state is None:
        state = sv.init_zero_state(n, options.precision, options.memory_budget, options.device)
    # H on the address register applied to |0...0>: the uniform superposition, one write pass
    N.call("qg_state_init_uniform", C.c_void_p(state.amplitudes.data_ptr()), n, sv._QG_DTYPE[options.precision],
           C.c_uint64((1 << m) - 1), 0, sv._stream(state.amplitudes.device))
    apply_ucry(state, list(range(m)), list(range(m, n)), angles)
    counts = None
    if options.shots > 0:
        counts = sv.sample_counts(state, options.shots, options.rng_seed, options.sampler)
    return state, counts


# ------------------------------------------------------------------ decode
def _lane_marginals(idx: np.ndarray, weight: np.ndarray, plan: QCrankPlan):
    """n0[a, d], n1[a, d]: weight of outcomes with address a and data bit d = 0 / 1."""
    m, nd = plan.n_addr, plan.n_data
    idx = np.asarray(idx, dtype=np.int64)
    w = np.asarray(weight, dtype=np.float64)
    a = idx & ((1 << m) - 1)
    tot = np.bincount(a, weights=w, minlength=1 << m)
    n1 = np.zeros((1 << m, nd))
    for d in range(nd):
        bit = (idx >> (m + d)) & 1
        n1[:, d] = np.bincount(a, weights=w * bit, minlength=1 << m)
    n0 = tot[:, None] - n1
    return n0, n1, tot


def _reconstruct(n0, n1, tot, plan: QCrankPlan, source: ImageGray | None):
    with np.errstate(invalid="ignore", divide="ignore"):
        v = np.where(tot[:, None] > 0, (n0 - n1) / tot[:, None], 0.0)
    v = np.clip(v, -1.0, 1.0)
    empty = np.flatnonzero(tot == 0).tolist()
    n_px = plan.width * plan.height if plan.width else plan.padded_len
    k = np.arange(n_px, dtype=np.int64)
    est = v[bitrev(k // plan.n_data, plan.n_addr), k % plan.n_data]
    px = np.clip(np.rint(255.0 * (est + 1.0) / 2.0), 0, 255).astype(np.uint8)
    rep = ReconstructionReport(estimates=est, empty_addresses=empty)
    if source is not None:
        truth = 2.0 * source.pixels.astype(np.float64) / 255.0 - 1.0
        err = est - truth
        rep.mse = float(np.mean(err * err))
        rep.max_abs_error = float(np.max(np.abs(err)))
        rep.correlation = float(np.corrcoef(est, truth)[0, 1]) if np.std(truth) > 0 and np.std(est) > 0 else None
    img = ImageGray(plan.width, plan.height, px) if plan.width else None
    return rep, img


def decode_counts(counts, plan: QCrankPlan, source: ImageGray | None = None):
    """SPEC.md:473-480.  `counts`: a CountsTable (statevec.sample_counts) or an
    (indices, counts) pair of arrays (statevec.sample_indices)."""
    if isinstance(counts, sv.CountsTable):
        if counts.indices is not None:
            idx, cnt = np.asarray(counts.indices), np.asarray(counts.values)
        else:
            keys = list(counts.counts)
            idx = np.array([sv.index_of_bitstring(k) for k in keys], dtype=np.int64)
            cnt = np.array([counts.counts[k] for k in keys], dtype=np.int64)
    else:
        idx, cnt = (np.asarray(x.cpu() if isinstance(x, torch.Tensor) else x) for x in counts)
    n0, n1, tot = _lane_marginals(idx, cnt, plan)
    return _reconstruct(n0, n1, tot, plan, source)


def sample_decode(state: sv.StateVector, plan: QCrankPlan, rng_seed: int = 0, source: ImageGray | None = None,
                  shots: int | None = None):
    """SPEC.md:473-480 at the paper's shot budget s * 2^m (~5e10 for
    m = 24): the tree sampler draws the multinomial counts straight into a dense
    per-outcome array in HBM (no per-shot records), the (address, data bit)
    marginals are reduced on the device, and only the 2^m x n_data tallies reach
    the host for the reconstruction."""
    shots = plan.shots if shots is None else int(shots)
    m, nd = plan.n_addr, plan.n_data
    ts = sv.TreeSampler(state.amplitudes)
    mass = ts.prepare()
    if not abs(mass - 1.0) <= sv.NORM_TOL[state.precision]:
        raise sv.UnnormalizedStateError(f"norm^2 = {mass!r} outside tolerance")
    dense = ts.draw(shots, rng_seed, dense=True)  # index = address + 2^m * data bits
    dev = dense.device
    tot = torch.empty(1 << m, dtype=torch.int64, device=dev)
    n1 = torch.empty((1 << m, nd), dtype=torch.int64, device=dev)
    N.call("qg_qcrank_tally", C.c_void_p(dense.data_ptr()), m, nd, C.c_void_p(tot.data_ptr()),
           C.c_void_p(n1.data_ptr()), sv._stream(dev))
    del dense
    return _reconstruct_device(tot, n1, plan, source)


def _reconstruct_device(tot: torch.Tensor, n1: torch.Tensor, plan: QCrankPlan, source: ImageGray | None):
    """_reconstruct on the device (2^27 pixels at m = 24: the numpy version takes
    ~20 s on the host); same estimator, same outputs."""
    m, nd = plan.n_addr, plan.n_data
    dev = tot.device
    t = tot.to(torch.float64)[:, None]
    v = torch.where(t > 0, (t - 2.0 * n1.to(torch.float64)) / torch.clamp(t, min=1.0), torch.zeros_like(t))
    v = v.clamp(-1.0, 1.0)
    empty = torch.nonzero(tot == 0).flatten().cpu().tolist()
    n_px = plan.width * plan.height if plan.width else plan.padded_len
    k = torch.arange(n_px, dtype=torch.int64, device=dev)
    g = k // nd
    a = torch.zeros_like(g)
    for b in range(m):
        a |= ((g >> b) & 1) << (m - 1 - b)
    est = v[a, k % nd]
    px = torch.clamp(torch.round(255.0 * (est + 1.0) / 2.0), 0, 255).to(torch.uint8)
    rep = ReconstructionReport(estimates=est.cpu().numpy(), empty_addresses=empty)
    if source is not None:
        truth = 2.0 * torch.from_numpy(np.asarray(source.pixels)).to(dev, torch.float64) / 255.0 - 1.0
        err = est - truth
        rep.mse = float((err * err).mean())
        rep.max_abs_error = float(err.abs().max())
        if float(truth.std()) > 0 and float(est.std()) > 0:
            rep.correlation = float(torch.corrcoef(torch.stack([est, truth]))[0, 1])
    img = ImageGray(plan.width, plan.height, px.cpu().numpy()) if plan.width else None
    return rep, img


def decode_exact(probabilities, plan: QCrankPlan, source: ImageGray | None = None):
    """the same estimator with exact marginals."""
    p = probabilities.cpu().numpy() if isinstance(probabilities, torch.Tensor) else np.asarray(probabilities)
    p = np.asarray(p, dtype=np.float64).reshape(-1)
    if p.size != 1 << plan.n_qubits:
        raise LengthMismatchError(f"{p.size} probabilities for a {plan.n_qubits}-qubit plan")
    n0, n1, tot = _lane_marginals(np.arange(p.size, dtype=np.int64), p, plan)
    return _reconstruct(n0, n1, tot, plan, source)


def circuit_type() -> CircType:
    return CircType.QCRANK
