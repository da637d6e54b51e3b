"""Planner + C-ABI checks that need no GPU.

The fused program exported by libqgear_b200's planner is executed by a numpy
interpreter (tests/plan_interp.py) and compared with the CPU oracle: this
proves the scheduling (gate reordering under commutation), the fp64 gate
fusion, register/thread control placement and the multi-rank remap
bookkeeping on any box.  The CUDA kernels are checked against the same oracle
in tests/test_gpu_parity.py.
"""

import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2504_03967_b200 import _native as N
from paper_2504_03967_b200 import errors as E
from paper_2504_03967_b200.generators import QftSpec, RandomSpec, qft_arrays, random_arrays
from paper_2504_03967_b200.statevec import CompiledCircuit
from tests.plan_interp import run_program


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def mixed(n, g, seed):
    rng = np.random.default_rng(seed)
    gt = np.zeros((g, 3), dtype=np.int32)
    gp = np.zeros(g)
    for i in range(g):
        k = int(rng.integers(0, 6)) if n > 1 else int(rng.integers(0, 4))
        t = int(rng.integers(0, n))
        c = -1
        if k in (4, 5):
            c = int(rng.integers(0, n - 1))
            c = c if c < t else c + 1
        gt[i] = (k, c, t)
        if k in (1, 2, 3, 5):
            gp[i] = rng.uniform(-7, 7)
    return gt, gp


def test_library_exports_every_header_symbol():
    lib = N.lib()
    names = N.header_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert lib.qg_abi_version() == 1


CASES = [
    ("random", 10, lambda: random_arrays(RandomSpec(10, 120, 3))),
    ("random", 12, lambda: random_arrays(RandomSpec(12, 200, 4))),
    ("qft", 11, lambda: qft_arrays(11)),
    ("qftr", 12, lambda: qft_arrays(12, True)),
    ("mixed", 9, lambda: mixed(9, 300, 1)),
    ("mixed", 12, lambda: mixed(12, 400, 2)),
]


@pytest.mark.parametrize("name,n,make", CASES, ids=[f"{c[0]}{c[1]}" for c in CASES])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_fused_program_matches_oracle(name, n, make, precision):
    gt, gp = make()
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    plan = CompiledCircuit(gt, gp, n, precision)
    assert plan.info["n_passes"] >= 1
    got = run_program(plan)
    assert rel_l2(got, ref) < 1e-12


@pytest.mark.parametrize("opts", [dict(max_stages=1), dict(max_stages=2, max_cost=20), dict(max_cost=10),
                                  dict(tile_qubits=8), dict(fuse=False)])
def test_planner_knobs_preserve_semantics(opts):
    n = 11
    gt, gp = mixed(n, 250, 7)
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    plan = CompiledCircuit(gt, gp, n, "fp32", **opts)
    assert rel_l2(run_program(plan), ref) < 1e-12


@pytest.mark.parametrize("log2_ranks", [1, 2, 3])
@pytest.mark.parametrize("fuse", [True, False])
def test_multirank_program_with_remaps(log2_ranks, fuse):
    n = 12
    gt, gp = random_arrays(RandomSpec(n, 150, 11))
    gt2, gp2 = mixed(n, 150, 3)
    gt, gp = np.concatenate([gt, gt2]), np.concatenate([gp, gp2])
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    plan = CompiledCircuit(gt, gp, n, "fp64", log2_ranks=log2_ranks, fuse=fuse)
    assert plan.n_local == n - log2_ranks
    assert len(plan.remaps) == plan.info["n_remaps"] == plan.n_segments - 1
    assert len(plan.remaps) >= 1
    assert rel_l2(run_program(plan), ref) < 1e-12


def test_fusion_reduces_passes_for_qft_and_random():
    gt, gp = qft_arrays(28)
    plan = CompiledCircuit(gt, gp, 28, "fp32")
    assert plan.info["n_passes"] <= 12, plan.info
    gt, gp = random_arrays(RandomSpec(32, 1000, 0))
    plan = CompiledCircuit(gt, gp, 32, "fp32")
    # one HBM pass per ~> 10 gates (SURVEY.md §7.3 simulated ~164 passes at k=13 without reordering)
    assert plan.info["n_passes"] < 300, plan.info


def _plan_error(gt, gp, n, **kw):
    with pytest.raises(E.QgearError) as ei:
        CompiledCircuit(np.asarray(gt, dtype=np.int32), np.asarray(gp, dtype=np.float64), n, **kw)
    return ei.value


def test_planner_error_mapping():
    assert isinstance(_plan_error([[0, -1, 3]], [0.0], 3), E.IndexOutOfRangeError)
    assert isinstance(_plan_error([[4, 1, 1]], [0.0], 3), E.SelfPairError)
    assert isinstance(_plan_error([[4, 5, 1]], [0.0], 3), E.IndexOutOfRangeError)
    assert isinstance(_plan_error([[6, -1, 0], [0, -1, 0]], [0.0, 0.0], 2), E.MeasureMidCircuitError)
    assert isinstance(_plan_error([[9, -1, 0]], [0.0], 2), E.CorruptTensorError)
    assert isinstance(_plan_error([[2, -1, 0]], [float("nan")], 2), E.NonFiniteParamError)
    assert isinstance(_plan_error([[0, -1, 0]], [0.0], 2, log2_ranks=3), E.BadWorkerCountError)
    # trailing MEASURE block is fine and not executed
    plan = CompiledCircuit(np.array([[0, -1, 0], [6, -1, 0], [6, -1, 1]], dtype=np.int32), np.zeros(3), 2)
    assert plan.info["n_body_gates"] == 1


def test_empty_circuit_plan():
    plan = CompiledCircuit(np.zeros((0, 3), dtype=np.int32), np.zeros(0), 3)
    assert plan.info["n_passes"] == 0
    got = run_program(plan)
    assert got[0] == 1 and np.count_nonzero(got) == 1


@pytest.mark.parametrize("n,log2_ranks", [(3, 2), (5, 4), (6, 4), (4, 3), (2, 1)])
def test_small_states_with_many_ranks(n, log2_ranks):
    """remaps must never reach below local position 0 when 2^g > 2^(n/2)."""
    gt, gp = random_arrays(RandomSpec(n, 40, 5))
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    for fuse in (True, False):
        plan = CompiledCircuit(gt, gp, n, "fp64", log2_ranks=log2_ranks, fuse=fuse)
        for rm in plan.remaps:
            assert all(0 <= p < plan.n_local for p in rm[1])
        assert rel_l2(run_program(plan), ref) < 1e-12


def test_all_qubits_global_needs_a_local_qubit():
    gt, gp = random_arrays(RandomSpec(3, 5, 5))
    assert isinstance(_plan_error(gt, gp, 3, log2_ranks=3), E.BadWorkerCountError)
    # diagonal-only circuits need no remap and run with every qubit global
    gt = np.array([[3, -1, 0], [5, 0, 1]], dtype=np.int32)
    plan = CompiledCircuit(gt, np.array([0.3, 0.7]), 2, "fp64", log2_ranks=2)
    assert plan.info["n_remaps"] == 0


@pytest.mark.parametrize("precision,n,k", [("fp32", 16, 11), ("fp32", 19, 11), ("fp64", 16, 10), ("fp64", 17, 10),
                                           ("fp64", 20, 13)])
def test_small_state_tile_choice(precision, n, k):
    gt, gp = random_arrays(RandomSpec(n, 20, 0))
    assert CompiledCircuit(gt, gp, n, precision).info["tile_qubits"] == k


def test_belady_remap_counts():
    """Remap planner: a remap brings in the global targets
    needed next and evicts the local qubits whose next non-diagonal-target use is
    furthest away (Belady), at positions >= 10 so each exchanged block is a set of
    >= 8 KiB runs.  Bounds: SURVEY's Belady estimates (28 at 32 q / 8 ranks, 23 at
    37 q / 8 ranks); the pre-eviction planner needed 37 and 32."""
    from paper_2504_03967_b200.generators import RandomSpec, random_arrays

    got = {}
    for n, g in [(32, 1), (32, 2), (32, 3), (37, 3)]:
        gt, gp = random_arrays(RandomSpec(n, 1000, 0))
        p = CompiledCircuit(gt, gp, n, "fp32", g, jit=-1)
        got[(n, 1 << g)] = p.info["n_remaps"]
        n_local = n - g
        for gpos, lpos in p.remaps:
            assert all(10 <= q < n_local for q in lpos) and all(q >= n_local for q in gpos)
    assert got[(32, 8)] <= 28 and got[(37, 8)] <= 23
    assert got[(32, 2)] <= 16 and got[(32, 4)] <= 22
