"""Circuit-specialised pass kernels (csrc/jit.cpp) on the CPU: every fused pass of
a complex64 plan is emitted as PTX and compiled by the in-process PTX compiler
(no GPU needed); passes the emitter does not cover are counted as fallbacks and
run the interpreter.  GPU parity (bit-exact vs the interpreter and vs the
oracle) is in tests/test_gpu_jit.py."""

import numpy as np
import pytest

from paper_2504_03967_b200.generators import QftSpec, RandomSpec, qft_arrays, random_arrays
from paper_2504_03967_b200.statevec import CompiledCircuit


@pytest.mark.parametrize("make,n", [(lambda: random_arrays(RandomSpec(22, 40, 3)), 22),
                                    (lambda: qft_arrays(22), 22)])
def test_every_pass_compiles_or_falls_back(make, n):
    gt, gp = make()
    plan = CompiledCircuit(gt, gp, n, "fp32", jit=1)
    st = plan.jit_status(wait=True)
    assert st["enabled"] == 1 and st["n_pending"] == 0
    assert st["n_jit"] + st["n_fallback"] == st["n_passes"] == plan.info["n_passes"]
    assert st["n_jit"] >= 1
    ptx = [plan.pass_ptx(i) for i in range(st["n_passes"])]
    assert sum(1 for x in ptx if x) == st["n_jit"]  # "" = not covered (tile-uniform phase slots)
    assert all(".target sm_100a" in x and "qg_jit_pass" in x for x in ptx if x)


def test_jit_policy():
    g26, p26 = random_arrays(RandomSpec(26, 4, 0))
    assert CompiledCircuit(g26, p26, 26, "fp32").jit_status(wait=True)["enabled"] == 2  # auto: tiered
    gt, gp = random_arrays(RandomSpec(22, 10, 0))
    assert CompiledCircuit(gt, gp, 22, "fp32").jit_status()["enabled"] == 0          # auto: small shard
    assert CompiledCircuit(gt, gp, 22, "fp64", jit=1).jit_status(wait=True)["enabled"] == 1  # complex128 too
    assert CompiledCircuit(gt, gp, 22, "fp64").jit_status()["enabled"] == 0          # auto: small shard
    assert CompiledCircuit(gt, gp, 22, "fp32", jit=-1).jit_status()["enabled"] == 0


def test_rebind_recompiles():
    gt, gp = random_arrays(RandomSpec(21, 20, 1))
    plan = CompiledCircuit(gt, gp, 21, "fp32", jit=1)
    plan.rebind(np.asarray(gp) * 0.5)
    st = plan.jit_status(wait=True)
    assert st["enabled"] == 1 and st["n_jit"] + st["n_fallback"] == st["n_passes"]
