"""B200 state-vector simulator with the reference's Python API
(/root/reference/pkg/src/qgear/statevec.py).

Same names, argument meaning and error types as the reference; the state now
lives in HBM as a torch CUDA tensor (complex64 for "fp32", complex128 for
"fp64") and every amplitude update runs in libqgear_b200.so:

  run_circuit          statevec.py:200-212  -> plan (C++) + fused passes (CUDA)
  apply_*_array        statevec.py:115-144  -> one single-gate kernel each
  exact_probabilities  statevec.py:215-218  -> fp64 |a|^2 kernel (device tensor)
  sample_counts        statevec.py:221-234  -> device two-level inverse-CDF sampler

Conventions are unchanged: qubit k is bit k of the basis index; display
bitstrings put qubit 0 leftmost (statevec.py:5-8, 71-78).
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import (
    IndexOutOfRangeError,
    MeasureMidCircuitError,
    SelfPairError,
    TooManyQubitsError,
    UnnormalizedStateError,
)
from .ir import CircuitTensor, GateKind, GateRecord, records_to_arrays

DEFAULT_MEMORY_BUDGET = 16 * 2**30  # statevec.py:32

_DTYPES = {"fp32": torch.complex64, "fp64": torch.complex128}
_COMPLEX_WIDTH = {"fp32": 8, "fp64": 16}
_QG_DTYPE = {"fp32": N.DTYPE_C64, "fp64": N.DTYPE_C128}
NORM_TOL = {"fp32": 1e-3, "fp64": 1e-9}  # statevec.py:38


def _stream(dev: torch.device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _precision_of(t: torch.Tensor) -> str:
    if t.dtype == torch.complex64:
        return "fp32"
    if t.dtype == torch.complex128:
        return "fp64"
    raise ValueError(f"amplitudes must be complex64/complex128, got {t.dtype}")


def _check_amps(t: torch.Tensor) -> int:
    if not t.is_cuda:
        raise ValueError("amplitudes must be a CUDA tensor (libqgear_b200 has no CPU path)")
    if not t.is_contiguous() or t.dim() != 1:
        raise ValueError("amplitudes must be a contiguous 1-D tensor")
    n = t.numel()
    if n < 1 or n & (n - 1):
        raise ValueError(f"amplitude count {n} is not a power of two")
    return n.bit_length() - 1


@dataclass
class StateVector:
    """statevec.py:41-53 — amplitudes is a device tensor (one shard per rank when distributed)."""

    n_qubits: int
    precision: str
    amplitudes: torch.Tensor

    def norm_sq(self) -> float:
        """Squared norm accumulated in float64 (statevec.py:47-50)."""
        return _norm_sq(self.amplitudes)

    def copy(self) -> "StateVector":
        return StateVector(self.n_qubits, self.precision, self.amplitudes.clone())

    def to_numpy(self) -> np.ndarray:
        return self.amplitudes.cpu().numpy()


@dataclass
class SimOptions:
    """statevec.py:56-61, plus B200 knobs.

    The reference fields keep their meaning and defaults.  One default differs in
    effect: ``sampler="philox"`` draws the shots from a device Philox stream, so
    counts are deterministic per ``rng_seed`` but NOT the reference's PCG64
    counts; ``sampler="numpy"`` reproduces the reference's
    ``default_rng(seed).choice`` stream (statevec.py:229-232) exactly, up to
    cumulative-sum rounding ties."""

    precision: str = "fp64"
    shots: int = 0
    rng_seed: int = 0
    memory_budget: int = DEFAULT_MEMORY_BUDGET
    sampler: str = "philox"      # "philox" (device RNG) | "numpy" (reference's PCG64 uniforms) |
                                 # "tree" (binomial splits: int64 shots, O(n/256) workspace, sharded states)
    device: str | int | None = None
    fuse: bool = True
    tile_qubits: int = 0
    max_stages: int = 0
    max_cost: int = 0
    jit: int = 0                 # circuit-specialised pass kernels: 0 auto (large complex64 shards), 1 on, -1 off


@dataclass
class CountsTable:
    """statevec.py:64-68; ``indices``/``values`` hold the same data as sorted arrays."""

    counts: dict[str, int]
    total: int
    n_qubits: int
    indices: np.ndarray | None = field(default=None, repr=False)
    values: np.ndarray | None = field(default=None, repr=False)


def bitstring(index: int, n_qubits: int) -> str:
    """qubit 0 leftmost (statevec.py:71-73)."""
    return "".join("1" if (index >> k) & 1 else "0" for k in range(n_qubits))


def index_of_bitstring(bits: str) -> int:
    return int(bits[::-1], 2) if bits else 0


def _device(d) -> torch.device:
    if d is None:
        return torch.device("cuda", torch.cuda.current_device())
    if isinstance(d, int):
        return torch.device("cuda", d)
    return torch.device(d)


def _check_budget(n_qubits: int, precision: str, memory_budget: int) -> None:
    if n_qubits < 1:
        raise ValueError(f"n_qubits must be >= 1, got {n_qubits}")
    if precision not in _DTYPES:
        raise ValueError(f"precision must be fp32 or fp64, got {precision!r}")
    required = _COMPLEX_WIDTH[precision] * (1 << n_qubits)
    if required > memory_budget:
        raise TooManyQubitsError(n_qubits, required, memory_budget)


def init_zero_state(n_qubits: int, precision: str = "fp64", memory_budget: int = DEFAULT_MEMORY_BUDGET,
                    device=None) -> StateVector:
    """|0...0> in HBM (statevec.py:81-94)."""
    _check_budget(n_qubits, precision, memory_budget)
    dev = _device(device)
    amps = torch.empty(1 << n_qubits, dtype=_DTYPES[precision], device=dev)
    N.call("qg_state_init_zero", C.c_void_p(amps.data_ptr()), n_qubits, _QG_DTYPE[precision], 0, _stream(dev))
    return StateVector(n_qubits, precision, amps)


def gate_matrix_2x2(kind: GateKind, param: float = 0.0) -> np.ndarray:
    """Host fp64 half-angle matrices (statevec.py:97-110)."""
    if kind == GateKind.H:
        r = 1.0 / math.sqrt(2.0)
        return np.array([[r, r], [r, -r]], dtype=np.complex128)
    h = param / 2.0
    c, s = math.cos(h), math.sin(h)
    if kind == GateKind.RX:
        return np.array([[c, -1j * s], [-1j * s, c]], dtype=np.complex128)
    if kind == GateKind.RY:
        return np.array([[c, -s], [s, c]], dtype=np.complex128)
    if kind == GateKind.RZ:
        return np.array([[complex(math.cos(h), -math.sin(h)), 0], [0, complex(math.cos(h), math.sin(h))]],
                        dtype=np.complex128)
    raise ValueError(f"{GateKind(kind).name} has no 2x2 matrix")


# --- array-level kernels (statevec.py:113-144) --------------------------------------

def apply_matrix_array(amps: torch.Tensor, target: int, u: np.ndarray) -> None:
    """Dense 2x2 on every (target=0, target=1) pair, in place (statevec.py:115-122)."""
    n = _check_amps(amps)
    m = np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(2, 2)).view(np.float64)
    N.call("qg_apply_matrix", C.c_void_p(amps.data_ptr()), n, _QG_DTYPE[_precision_of(amps)], int(target),
           m.ctypes.data_as(C.c_void_p), _stream(amps.device))


def swap_target_pairs_array(amps: torch.Tensor, control: int, target: int) -> None:
    """CX kernel (statevec.py:125-137): touches only the control = 1 half."""
    n = _check_amps(amps)
    N.call("qg_apply_cx", C.c_void_p(amps.data_ptr()), n, _QG_DTYPE[_precision_of(amps)], int(control),
           int(target), _stream(amps.device))


def phase_pairs_array(amps: torch.Tensor, control: int, target: int, lam: float) -> None:
    """CR1 kernel (statevec.py:140-144)."""
    n = _check_amps(amps)
    N.call("qg_apply_cr1", C.c_void_p(amps.data_ptr()), n, _QG_DTYPE[_precision_of(amps)], int(control),
           int(target), float(lam), _stream(amps.device))


def apply_1q(state: StateVector, kind: GateKind, target: int, param: float = 0.0) -> StateVector:
    if not 0 <= target < state.n_qubits:
        raise IndexOutOfRangeError(f"target {target} out of range for {state.n_qubits} qubits")
    apply_matrix_array(state.amplitudes, target, gate_matrix_2x2(kind, param))
    return state


def _check_pair(state: StateVector, control: int, target: int) -> None:
    for q in (control, target):
        if q is None or not 0 <= q < state.n_qubits:
            raise IndexOutOfRangeError(f"qubit {q} out of range for {state.n_qubits} qubits")
    if control == target:
        raise SelfPairError(f"control == target == {control}")


def apply_cx(state: StateVector, control: int, target: int) -> StateVector:
    _check_pair(state, control, target)
    swap_target_pairs_array(state.amplitudes, control, target)
    return state


def apply_cr1(state: StateVector, control: int, target: int, lam: float) -> StateVector:
    _check_pair(state, control, target)
    phase_pairs_array(state.amplitudes, control, target, lam)
    return state


def apply_record(state: StateVector, g: GateRecord) -> StateVector:
    """statevec.py:177-184."""
    if g.kind == GateKind.CX:
        return apply_cx(state, g.control, g.target)
    if g.kind == GateKind.CR1:
        return apply_cr1(state, g.control, g.target, g.param)
    if g.kind == GateKind.MEASURE:
        return state
    return apply_1q(state, g.kind, g.target, g.param)


def split_trailing_measures(gates):
    """statevec.py:187-197 on GateRecords."""
    first = len(gates)
    for i, g in enumerate(gates):
        if g.kind == GateKind.MEASURE:
            first = i
            break
    for g in gates[first:]:
        if g.kind != GateKind.MEASURE:
            raise MeasureMidCircuitError("MEASURE records must form a trailing block")
    return tuple(gates[:first]), tuple(gates[first:])


def _trailing_split_arrays(kinds: np.ndarray) -> int:
    meas = np.flatnonzero(kinds == GateKind.MEASURE)
    if meas.size == 0:
        return int(kinds.size)
    if np.any(kinds[meas[0]:] != GateKind.MEASURE):
        raise MeasureMidCircuitError("MEASURE records must form a trailing block")
    return int(meas[0])


def circuit_arrays(circuit) -> tuple[np.ndarray, np.ndarray, int]:
    """(gate_type live rows int32 (g,3), gate_param (g,) f64, n_qubits) of a circuit.

    Accepts this package's CircuitTensor, or any object with the reference's
    CircuitTensor interface (``active_gates`` of GateRecord-like objects).
    """
    if isinstance(circuit, CircuitTensor):
        gt, gp = circuit.active_arrays
        return np.ascontiguousarray(gt, dtype=np.int32), np.ascontiguousarray(gp, dtype=np.float64), circuit.n_qubits
    gates = list(circuit.active_gates)
    gt, gp = records_to_arrays(gates)
    return gt, gp, int(circuit.n_qubits)


class CompiledCircuit:
    """A planned circuit (libqgear_b200 qg_plan): fused passes + remaps, reusable across runs."""

    def __init__(self, gate_type: np.ndarray, gate_param: np.ndarray, n_qubits: int, precision: str = "fp64",
                 log2_ranks: int = 0, fuse: bool = True, tile_qubits: int = 0, max_stages: int = 0,
                 max_cost: int = 0, kernel_cfg: int = 0, jit: int = 0, low_qubits: int = 0):
        gt = np.ascontiguousarray(gate_type, dtype=np.int32).reshape(-1, 3)
        gp = np.ascontiguousarray(gate_param, dtype=np.float64).reshape(-1)
        if gt.shape[0] != gp.shape[0]:
            raise ValueError("gate_type and gate_param lengths differ")
        if precision not in _DTYPES:
            raise ValueError(f"precision must be fp32 or fp64, got {precision!r}")
        self.n_qubits = int(n_qubits)
        self.precision = precision
        self.log2_ranks = int(log2_ranks)
        opts = N.PlanOpts(dtype=_QG_DTYPE[precision], log2_ranks=log2_ranks, fuse=1 if fuse else 0,
                          tile_qubits=tile_qubits, max_stages=max_stages, max_cost=max_cost,
                          kernel_cfg=kernel_cfg, jit=int(jit), low_qubits=int(low_qubits))
        h = C.c_void_p()
        self._lib = N.lib()
        N.check(self._lib.qg_plan_create(gt.ctypes.data_as(C.c_void_p), gp.ctypes.data_as(C.c_void_p),
                                         gt.shape[0], self.n_qubits, C.byref(opts), C.byref(h)))
        self._h = h
        info = N.PlanInfo()
        N.check(self._lib.qg_plan_get_info(self._h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in N.PlanInfo._fields_}
        self.n_local = info.n_local
        self.remaps = []
        for i in range(info.n_remaps):
            r = N.Remap()
            N.check(self._lib.qg_plan_get_remap(self._h, i, C.byref(r)))
            self.remaps.append((list(r.global_pos[: r.s]), list(r.local_pos[: r.s])))
        fm = np.zeros(self.n_qubits, dtype=np.int32)
        N.check(self._lib.qg_plan_get_final_map(self._h, fm.ctypes.data_as(C.c_void_p)))
        self.final_map = fm  # logical qubit -> physical position

    def jit_status(self, wait: bool = False) -> dict:
        """Circuit-specialised pass kernels (include/qgear_b200.h qg_plan_jit_status)."""
        st = N.JitStatus()
        N.check(self._lib.qg_plan_jit_status(self._h, 1 if wait else 0, C.byref(st)))
        return {f: getattr(st, f) for f, _ in N.JitStatus._fields_}

    def pass_ptx(self, index: int) -> str:
        """PTX the emitter produces for fused pass `index` (complex64 plans)."""
        n = C.c_int64()
        N.check(self._lib.qg_plan_pass_ptx(self._h, int(index), None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        N.check(self._lib.qg_plan_pass_ptx(self._h, int(index), buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def rebind(self, gate_param: np.ndarray) -> "CompiledCircuit":
        """New parameters for the same gate structure (a CircuitSet's batched
        parameter sets): reuses the schedule, rebuilds only the program."""
        gp = np.ascontiguousarray(gate_param, dtype=np.float64).reshape(-1)
        N.check(self._lib.qg_plan_rebind(self._h, gp.ctypes.data_as(C.c_void_p), gp.shape[0]))
        info = N.PlanInfo()
        N.check(self._lib.qg_plan_get_info(self._h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in N.PlanInfo._fields_}
        return self

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.qg_plan_destroy(h)
            self._h = None

    @property
    def n_segments(self) -> int:
        return int(self.info["n_segments"])

    def execute(self, state: StateVector, timed: bool = False) -> N.ExecStats:
        if self.log2_ranks:
            raise ValueError("multi-rank plan: use paper_2504_03967_b200.partition")
        return self.execute_segment(0, state.amplitudes, 0, timed)

    def execute_segment(self, seg: int, shard: torch.Tensor, rank: int = 0, timed: bool = False) -> N.ExecStats:
        n = _check_amps(shard)
        if n != self.n_local or _precision_of(shard) != self.precision:
            raise ValueError(f"shard has {n} qubits / {_precision_of(shard)}, plan expects "
                             f"{self.n_local} / {self.precision}")
        st = N.ExecStats()
        N.check(self._lib.qg_plan_execute_segment(self._h, seg, C.c_void_p(shard.data_ptr()), rank,
                                                  _stream(shard.device), 1 if timed else 0, C.byref(st)))
        return st

    def export(self) -> tuple[np.ndarray, np.ndarray]:
        """(records (r,8) int64, coefficients (m,8) f64) — see include/qgear_b200.h."""
        nr, nm = C.c_int64(), C.c_int64()
        N.check(self._lib.qg_plan_export(self._h, None, C.byref(nr), None, C.byref(nm)))
        rec = np.zeros((nr.value, 8), dtype=np.int64)
        mats = np.zeros((nm.value, 8), dtype=np.float64)
        N.check(self._lib.qg_plan_export(self._h, rec.ctypes.data_as(C.c_void_p), C.byref(nr),
                                         mats.ctypes.data_as(C.c_void_p), C.byref(nm)))
        return rec, mats


def compile_circuit(circuit, options: SimOptions | None = None, log2_ranks: int = 0) -> CompiledCircuit:
    options = options or SimOptions()
    gt, gp, n = circuit_arrays(circuit)
    _trailing_split_arrays(gt[:, 0])
    return CompiledCircuit(gt, gp, n, options.precision, log2_ranks, options.fuse, options.tile_qubits,
                           options.max_stages, options.max_cost, jit=options.jit)


def run_circuit(circuit, options: SimOptions | None = None):
    """Apply the live gates in order; sample once iff shots > 0 (statevec.py:200-212)."""
    options = options or SimOptions()
    gt, gp, n = circuit_arrays(circuit)
    nb = _trailing_split_arrays(gt[:, 0])                          # MeasureMidCircuitError first
    if options.fuse and nb >= 32:
        # QCrank-style uniformly controlled RY blocks (2^m RY + 2^m CX each) run as
        # one-pass UCRY kernels instead of 2^(m+1) gates (qcrank.collapse_ucry)
        from . import qcrank

        if any(it[0] == "ucry" for it in qcrank.collapse_ucry(gt[:nb], gp[:nb])):
            return qcrank.run_gates(gt, gp, n, options)
    _check_budget(n, options.precision, options.memory_budget)     # then TooManyQubitsError
    # the state first, as the reference does (statevec.py:205-208): its |0..0> init runs on
    # the device while the host plans
    state = init_zero_state(n, options.precision, options.memory_budget, options.device)
    plan = CompiledCircuit(gt, gp, n, options.precision, 0, options.fuse, options.tile_qubits,
                           options.max_stages, options.max_cost, jit=options.jit)   # then gate errors
    plan.execute(state)
    counts = None
    if options.shots > 0:
        counts = sample_counts(state, options.shots, options.rng_seed, options.sampler)
    return state, counts


def _norm_sq(amps: torch.Tensor) -> float:
    n = _check_amps(amps)
    ws = torch.empty(8 * 1024, dtype=torch.uint8, device=amps.device)
    out = C.c_double()
    N.call("qg_norm_sq", C.c_void_p(amps.data_ptr()), 1 << n, _QG_DTYPE[_precision_of(amps)],
           C.c_void_p(ws.data_ptr()), ws.numel(), C.byref(out), _stream(amps.device))
    return out.value


def exact_probabilities(state: StateVector) -> torch.Tensor:
    """|amplitude|^2 in float64, as a device tensor (statevec.py:215-218)."""
    amps = state.amplitudes
    n = _check_amps(amps)
    out = torch.empty(1 << n, dtype=torch.float64, device=amps.device)
    N.call("qg_probabilities", C.c_void_p(amps.data_ptr()), 1 << n, _QG_DTYPE[_precision_of(amps)],
           C.c_void_p(out.data_ptr()), _stream(amps.device))
    return out


class TreeSampler:
    """Device tree sampler over one state or shard (include/qgear_b200.h
    qg_sample_tree_*): ``prepare()`` reads the state once and returns its mass
    sum |a|^2; ``draw(shots)`` returns the multinomial counts of `shots` draws,
    as (index, count) int64 device tensors of the outcomes with a count (index
    ascending, offset by ``index_base``) or, with ``dense=True``, one int64
    count per amplitude."""

    def __init__(self, amps: torch.Tensor, index_base: int = 0):
        self.n = _check_amps(amps)
        self.amps = amps
        self.dtype = _QG_DTYPE[_precision_of(amps)]
        self.index_base = int(index_base)
        self.ws = torch.empty(max(N.lib().qg_sample_tree_workspace_bytes(1 << self.n), 1024), dtype=torch.uint8,
                              device=amps.device)
        self.mass = None

    def prepare(self) -> float:
        m = C.c_double()
        N.call("qg_sample_tree_prepare", C.c_void_p(self.amps.data_ptr()), 1 << self.n, self.dtype,
               C.c_void_p(self.ws.data_ptr()), self.ws.numel(), C.byref(m), _stream(self.amps.device))
        self.mass = m.value
        return self.mass

    def prepare_async(self) -> None:
        """prepare() without reading the mass back (stream-ordered; CUDA-graph safe)."""
        N.call("qg_sample_tree_prepare", C.c_void_p(self.amps.data_ptr()), 1 << self.n, self.dtype,
               C.c_void_p(self.ws.data_ptr()), self.ws.numel(), None, _stream(self.amps.device))

    def mass_device(self) -> torch.Tensor:
        """The mass computed by the last prepare, as a 1-element device view (heap root)."""
        return self.ws[:8].view(torch.float64)

    def draw_into(self, shots: int, rng_seed: int, tag: int, idx: torch.Tensor, cnt: torch.Tensor,
                  n_out: torch.Tensor) -> None:
        """(index, count) pairs into preallocated buffers and their number into the
        1-element int64 device tensor n_out, with no host synchronisation."""
        N.call("qg_sample_tree_draw", C.c_void_p(self.amps.data_ptr()), 1 << self.n, self.dtype,
               C.c_void_p(self.ws.data_ptr()), self.ws.numel(), int(shots), C.c_uint64(rng_seed & (2**64 - 1)),
               int(tag), 0, self.index_base, C.c_void_p(idx.data_ptr()), C.c_void_p(cnt.data_ptr()), idx.numel(),
               None, C.c_void_p(n_out.data_ptr()), _stream(self.amps.device))

    def draw(self, shots: int, rng_seed: int = 0, tag: int = 2, dense: bool = False):
        if self.mass is None:
            self.prepare()
        na = 1 << self.n
        dev = self.amps.device
        if not dense and na >= 1 << 16 and shots >= na // 8:
            # many shots per outcome: the level-synchronous dense draw (the same counts
            # bit for bit) and a device compaction beat the warp-per-leaf splits
            d = self.draw(shots, rng_seed, tag, dense=True)
            nz = torch.nonzero(d).flatten()
            return nz + self.index_base, d[nz]
        cap = na if dense else max(1, min(int(shots), na))
        cnt = torch.empty(cap, dtype=torch.int64, device=dev)
        idx = None if dense else torch.empty(cap, dtype=torch.int64, device=dev)
        nout = C.c_int64()
        N.call("qg_sample_tree_draw", C.c_void_p(self.amps.data_ptr()), na, self.dtype, C.c_void_p(self.ws.data_ptr()),
               self.ws.numel(), int(shots), C.c_uint64(rng_seed & (2**64 - 1)), int(tag), 1 if dense else 0,
               self.index_base, C.c_void_p(0 if idx is None else idx.data_ptr()), C.c_void_p(cnt.data_ptr()), cap,
               C.byref(nout), None, _stream(dev))
        if dense:
            return cnt
        k = nout.value
        return idx[:k], cnt[:k]


class CircuitGraph:
    """One planned circuit captured as a CUDA graph: |0..0> init, every fused pass
    and (shots > 0) the sampler (per-shot Philox up to 2^24 shots, else the tree).
    replay() is one graph launch with no host synchronisation; result() reads the
    norm and the outcome count back (one
    sync) and checks the norm like sample_counts (statevec.py:226-228).  For
    small, launch-bound circuits run many times (BASELINE configs[0]: 16 q,
    300 gates, complex128, 3000 shots)."""

    def __init__(self, plan: "CompiledCircuit", shots: int = 0, rng_seed: int = 0, device=None):
        if plan.log2_ranks:
            raise ValueError("multi-rank plan: use paper_2504_03967_b200.partition")
        n, prec = plan.n_qubits, plan.precision
        self.plan, self.shots, self.seed = plan, int(shots), int(rng_seed)
        self.state = init_zero_state(n, prec, 1 << 62, device)
        amps = self.state.amplitudes
        dev = amps.device
        # per-shot Philox sampler (fewest graph nodes) up to 2^24 shots, the tree sampler above
        self.per_shot = 0 < self.shots <= (1 << 24)
        self.ts = TreeSampler(amps) if shots > 0 and not self.per_shot else None
        cap = max(1, self.shots if self.per_shot else min(self.shots, 1 << n))
        self.idx = torch.empty(cap, dtype=torch.int64, device=dev)
        self.cnt = torch.empty(cap, dtype=torch.int64, device=dev)
        self.nout = torch.zeros(1, dtype=torch.int64, device=dev)
        self.norm = torch.zeros(1, dtype=torch.float64, device=dev)
        if self.per_shot:
            self.ws = torch.empty(max(N.lib().qg_sample_workspace_bytes(1 << n, self.shots), 256), dtype=torch.uint8,
                                  device=dev)
        side = torch.cuda.Stream(dev)  # warm-up off the capture: JIT libraries load, CUB settles
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            self._body()
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, capture_error_mode="relaxed"):
            self._body()

    def _body(self):
        amps = self.state.amplitudes
        N.call("qg_state_init_zero", C.c_void_p(amps.data_ptr()), self.plan.n_qubits,
               _QG_DTYPE[self.plan.precision], 0, _stream(amps.device))
        self.plan.execute(self.state)
        if self.per_shot:
            N.call("qg_sample_async", C.c_void_p(amps.data_ptr()), 1 << self.plan.n_qubits,
                   _QG_DTYPE[self.plan.precision], self.shots, C.c_uint64(self.seed & (2**64 - 1)),
                   C.c_void_p(self.ws.data_ptr()), self.ws.numel(), C.c_void_p(self.idx.data_ptr()),
                   C.c_void_p(self.cnt.data_ptr()), C.c_void_p(self.nout.data_ptr()), C.c_void_p(self.norm.data_ptr()),
                   _stream(amps.device))
        elif self.ts is not None:
            self.ts.prepare_async()
            self.ts.draw_into(self.shots, self.seed, 2, self.idx, self.cnt, self.nout)

    def replay(self) -> None:
        self.graph.replay()

    def result(self):
        """(StateVector, CountsTable | None) of the last replay."""
        counts = None
        if self.shots > 0:
            m = float((self.norm if self.per_shot else self.ts.mass_device()).item())
            if not abs(m - 1.0) <= NORM_TOL[self.plan.precision]:
                raise UnnormalizedStateError(f"norm^2 = {m!r} outside tolerance")
            k = int(self.nout.item())
            counts = counts_from_arrays(self.idx[:k].cpu().numpy(), self.cnt[:k].cpu().numpy(), self.shots,
                                        self.plan.n_qubits)
        return self.state, counts


def split_shots(masses, shots: int, rng_seed: int, device=None) -> list[int]:
    """Shots per part (a sharded state's ranks) from the parts' masses: the top of
    the tree sampler's binomial tree (qg_split_shots); identical on every rank."""
    m = np.ascontiguousarray(np.asarray(masses, dtype=np.float64))
    out = np.zeros(m.shape[0], dtype=np.int64)
    dev = _device(device)
    ws = torch.empty(1024, dtype=torch.uint8, device=dev)
    N.call("qg_split_shots", m.ctypes.data_as(C.c_void_p), m.shape[0], int(shots), C.c_uint64(rng_seed & (2**64 - 1)),
           C.c_void_p(ws.data_ptr()), ws.numel(), out.ctypes.data_as(C.c_void_p), _stream(dev))
    return out.tolist()


def sample_indices(amps: torch.Tensor, shots: int, rng_seed: int = 0, sampler: str = "philox",
                   norm_tol: float | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """Device sampler: (unique outcome indices ascending, counts) as int64 device tensors.

    ``sampler="philox"`` switches to the tree sampler above 2^31 - 1 shots (the
    per-shot sampler keeps one record per shot)."""
    if shots < 1:
        raise ValueError(f"shots must be >= 1, got {shots}")
    n = _check_amps(amps)
    prec = _precision_of(amps)
    tol = NORM_TOL[prec] if norm_tol is None else norm_tol
    dev = amps.device
    if sampler == "tree" or (sampler == "philox" and shots > 2**31 - 1):
        ts = TreeSampler(amps)
        m = ts.prepare()
        if not abs(m - 1.0) <= tol:  # statevec.py:226-228
            raise UnnormalizedStateError(f"norm^2 = {m!r} outside tolerance")
        return ts.draw(shots, rng_seed)
    ws_bytes = N.lib().qg_sample_workspace_bytes(1 << n, shots)
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
    idx = torch.empty(shots, dtype=torch.int64, device=dev)
    cnt = torch.empty(shots, dtype=torch.int64, device=dev)
    uni = None
    if sampler == "numpy":  # the reference's exact uniform stream: Generator.choice -> random(shots)
        uni = torch.from_numpy(np.random.default_rng(rng_seed).random(shots)).to(dev)
    elif sampler != "philox":
        raise ValueError(f"sampler must be 'philox', 'numpy' or 'tree', got {sampler!r}")
    nu = C.c_int64()
    nsq = C.c_double()
    N.call("qg_sample", C.c_void_p(amps.data_ptr()), 1 << n, _QG_DTYPE[prec], shots, C.c_uint64(rng_seed & (2**64 - 1)),
           C.c_void_p(uni.data_ptr() if uni is not None else 0), tol, C.c_void_p(ws.data_ptr()), ws.numel(),
           C.c_void_p(idx.data_ptr()), C.c_void_p(cnt.data_ptr()), C.byref(nu), C.byref(nsq), _stream(dev))
    k = nu.value
    return idx[:k], cnt[:k]


def bitstrings(idx: np.ndarray, n_qubits: int) -> list[str]:
    """bitstring() of many indices at once (qubit 0 leftmost), vectorised."""
    idx = np.asarray(idx, dtype=np.int64)
    if idx.size == 0 or n_qubits == 0:
        return [""] * idx.size
    chars = (((idx[:, None] >> np.arange(n_qubits, dtype=np.int64)) & 1).astype(np.uint8) + ord("0"))
    return np.ascontiguousarray(chars).view(f"S{n_qubits}").ravel().astype(f"U{n_qubits}").tolist()


def counts_from_arrays(idx: np.ndarray, cnt: np.ndarray, shots: int, n_qubits: int) -> CountsTable:
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    cnt = np.ascontiguousarray(cnt, dtype=np.int64)
    try:  # host-side formatting helper built with the library (csrc/counts_dict.c)
        from ._counts import counts_dict
    except ImportError:
        counts_dict = None
    if counts_dict is not None and n_qubits <= 64:
        counts = counts_dict(idx, cnt, n_qubits)
    else:
        counts = dict(zip(bitstrings(idx, n_qubits), cnt.tolist()))
    return CountsTable(counts=counts, total=shots, n_qubits=n_qubits, indices=idx, values=cnt)


def sample_counts(state: StateVector, shots: int, rng_seed: int = 0, sampler: str = "philox") -> CountsTable:
    """Multinomial draw from |amplitude|^2 (statevec.py:221-234), deterministic per seed."""
    idx, cnt = sample_indices(state.amplitudes, shots, rng_seed, sampler, NORM_TOL[state.precision])
    return counts_from_arrays(idx.cpu().numpy(), cnt.cpu().numpy(), shots, state.n_qubits)


@dataclass
class TimedRun:
    """statevec.py:237-243."""

    state: StateVector
    counts: CountsTable | None
    wall_ms: float


def run_circuit_timed(circuit, options: SimOptions | None = None) -> TimedRun:
    """statevec.py:246-250: wall time of run_circuit (device work included)."""
    dev = _device((options or SimOptions()).device)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    state, counts = run_circuit(circuit, options)
    torch.cuda.synchronize(dev)
    return TimedRun(state=state, counts=counts, wall_ms=(time.perf_counter() - t0) * 1000.0)
