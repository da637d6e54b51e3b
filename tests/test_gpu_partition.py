"""GPU: sharded execution (in-process shards, the multi-rank plans with qubit
remaps) against the reference's partitioned executor golden vectors and the oracle."""

import numpy as np
import pytest

import oracle
from paper_2504_03967_b200 import partition as pt
from paper_2504_03967_b200 import statevec as sv
from paper_2504_03967_b200.generators import RandomSpec, random_arrays, qft_arrays
from paper_2504_03967_b200.ir import CircType, CircuitTensor

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a, dtype=np.complex128) - b) / np.linalg.norm(b))


@pytest.mark.parametrize("j", range(3))
@pytest.mark.parametrize("fuse", [True, False])
def test_partitioned_golden(golden, j, fuse):
    nq, ng, w = (int(v) for v in golden[f"part{j}_meta"])
    c = CircuitTensor.from_arrays(CircType.IMPORTED, nq, golden[f"part{j}_type"][:ng], golden[f"part{j}_param"][:ng])
    res = pt.execute_distributed(c, w, sv.SimOptions("fp64", 2000, 5, fuse=fuse))
    assert rel_l2(res.state.to_numpy(), golden[f"part{j}_state"]) <= 1e-12
    assert res.counts.total == 2000
    assert len(res.messages_sent) == w and len(set(res.messages_sent)) == 1


@pytest.mark.parametrize("workers", [2, 4, 8])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_sharded_random_vs_oracle(workers, precision):
    n = 20
    gt, gp = random_arrays(RandomSpec(n, 250, workers))
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    c = CircuitTensor.from_arrays(CircType.RANDOM, n, gt, gp)
    res = pt.execute_distributed(c, workers, sv.SimOptions(precision))
    assert res.tasks["n_remaps"] >= 1
    assert rel_l2(res.state.to_numpy(), ref) <= (1e-12 if precision == "fp64" else 1e-5)


def test_sharded_qft_single_remap():
    n = 18
    gt, gp = qft_arrays(n)
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    res = pt.execute_distributed(CircuitTensor.from_arrays(CircType.QFT, n, gt, gp), 8, sv.SimOptions("fp32"))
    assert rel_l2(res.state.to_numpy(), ref) <= 1e-5
