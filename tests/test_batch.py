"""Batched circuit sets (mqpu mode): plan reuse through qg_plan_rebind, stream
concurrency, rank assignment.  Each circuit is checked against the oracle."""

import numpy as np
import pytest

import oracle
from paper_2504_03967_b200 import batch
from paper_2504_03967_b200.generators import RandomSpec, qft_arrays, random_arrays
from paper_2504_03967_b200.ir import CircType, CircuitHeader, CircuitSet, CircuitTensor
from paper_2504_03967_b200.statevec import CompiledCircuit
from tests.plan_interp import run_program


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def make_set(capacity=None):
    """Three parameter sets of one random ansatz, a QFT and a smaller random circuit."""
    rng = np.random.default_rng(4)
    gt, gp = random_arrays(RandomSpec(10, 60, 7))
    circs = []
    for _ in range(3):
        p = gp.copy()
        live = np.isin(gt[:, 0], [1, 2, 3])
        p[live] = rng.uniform(0, 2 * np.pi, int(live.sum()))
        circs.append((CircType.RANDOM, 10, gt, p))
    q_t, q_p = qft_arrays(9)
    circs.append((CircType.QFT, 9, q_t, q_p))
    s_t, s_p = random_arrays(RandomSpec(7, 20, 1))
    circs.append((CircType.RANDOM, 7, s_t, s_p))
    d = capacity or max(c[2].shape[0] for c in circs)
    tensors = []
    for ct, n, t, p in circs:
        gt_pad = np.zeros((d, 3), dtype=np.int32)
        gp_pad = np.zeros(d)
        gt_pad[: t.shape[0]] = t
        gp_pad[: t.shape[0]] = p
        tensors.append(CircuitTensor(CircuitHeader(ct, n, t.shape[0]), gt_pad, gp_pad))
    return CircuitSet(capacity=d, circuits=tuple(tensors)), circs


def test_assign_circuits_round_robin():
    assert batch.assign_circuits(7, 3, 0) == [0, 3, 6]
    assert batch.assign_circuits(7, 3, 2) == [2, 5]
    owned = sorted(i for r in range(4) for i in batch.assign_circuits(10, 4, r))
    assert owned == list(range(10))


def test_rebind_reproduces_fresh_plan_semantics():
    _, circs = make_set()
    base = CompiledCircuit(circs[0][2], circs[0][3], 10, "fp64")
    for _, n, gt, gp in circs[1:3]:
        base.rebind(gp)
        ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
        assert rel_l2(run_program(base), ref) < 1e-12


def test_rebind_rejects_nonfinite():
    from paper_2504_03967_b200.errors import NonFiniteParamError

    _, circs = make_set()
    plan = CompiledCircuit(circs[0][2], circs[0][3], 10, "fp64")
    bad = circs[0][3].copy()
    bad[np.flatnonzero(circs[0][2][:, 0] == 2)[0]] = np.nan
    with pytest.raises(NonFiniteParamError):
        plan.rebind(bad)


@pytest.mark.gpu
@pytest.mark.parametrize("precision,tol", [("fp64", 1e-12), ("fp32", 1e-5)])
def test_circuit_set_matches_oracle(precision, tol):
    from paper_2504_03967_b200 import statevec as sv

    cset, circs = make_set()
    res = batch.run_circuit_set(cset, sv.SimOptions(precision, shots=500), keep_states=True, streams=3)
    assert [r.index for r in res] == list(range(len(circs)))
    assert [r.planned for r in res] == [True, False, False, True, True]
    for r, (_, n, gt, gp) in zip(res, circs):
        ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
        assert rel_l2(r.state.to_numpy(), ref) < tol
        assert r.counts.total == 500 and sum(r.counts.counts.values()) == 500
        assert abs(r.norm_sq - 1) < 1e-4
