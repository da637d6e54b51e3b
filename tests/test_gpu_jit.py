"""GPU: circuit-specialised pass kernels (csrc/jit.cpp) against the op-stream
interpreter (csrc/fused.cu) — the same program, op semantics and FP operation
order, so the states must agree BIT FOR BIT — and against the CPU oracle."""

import numpy as np
import pytest
import torch

import oracle
from paper_2504_03967_b200 import partition as pt
from paper_2504_03967_b200 import statevec as sv
from paper_2504_03967_b200.generators import RandomSpec, qft_arrays, random_arrays
from paper_2504_03967_b200.ir import CircType, CircuitTensor, GateKind

pytestmark = pytest.mark.gpu


def mixed(n, g, seed):
    rng = np.random.default_rng(seed)
    gt = np.zeros((g, 3), dtype=np.int32)
    gp = np.zeros(g)
    for i in range(g):
        k = int(rng.integers(0, 6))
        t = int(rng.integers(0, n))
        c = -1
        if k in (4, 5):
            c = int(rng.integers(0, n - 1))
            c = c if c < t else c + 1
        gt[i] = (k, c, t)
        if k in (1, 2, 3, 5):
            gp[i] = rng.uniform(-7, 7)
    return gt, gp


def run(gt, gp, n, jit):
    plan = sv.CompiledCircuit(gt, gp, n, "fp32", jit=jit)
    st = sv.init_zero_state(n, "fp32", 1 << 40)
    plan.execute(st)
    return st.amplitudes, plan.jit_status(wait=True)


def same_bits(a, b):
    ra, rb = torch.view_as_real(a), torch.view_as_real(b)
    step = 1 << 26
    return all(torch.equal(ra[i:i + step], rb[i:i + step]) for i in range(0, ra.shape[0], step))


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a, dtype=np.complex128) - b) / np.linalg.norm(b))


CASES = [
    ("random22", 22, lambda: random_arrays(RandomSpec(22, 300, 1))),
    ("random24", 24, lambda: random_arrays(RandomSpec(24, 600, 2))),
    ("mixed22", 22, lambda: mixed(22, 1500, 3)),
    ("qft23r", 23, lambda: qft_arrays(23, True)),
]


@pytest.mark.parametrize("name,n,make", CASES, ids=[c[0] for c in CASES])
def test_jit_bitexact_vs_interpreter(name, n, make):
    gt, gp = make()
    a, st0 = run(gt, gp, n, -1)
    b, st1 = run(gt, gp, n, 1)
    assert st0["enabled"] == 0 and st1["enabled"] == 1 and st1["n_jit"] >= 1
    assert same_bits(a, b)
    if n <= 22:
        ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
        assert rel_l2(b.cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("workers", [2, 4])
def test_jit_sharded_with_remaps(workers):
    """rank-bit predicates and remapped qubit positions through the JIT kernels"""
    n = 22
    gt, gp = random_arrays(RandomSpec(n, 300, 10 + workers))
    gt2, gp2 = mixed(n, 300, workers)
    gt, gp = np.concatenate([gt, gt2]), np.concatenate([gp, gp2])
    c = CircuitTensor.from_arrays(CircType.IMPORTED, n, gt, gp)
    r0 = pt.execute_distributed(c, workers, sv.SimOptions("fp32", jit=-1))
    r1 = pt.execute_distributed(c, workers, sv.SimOptions("fp32", jit=1))
    assert r1.tasks["n_remaps"] >= 1
    assert same_bits(r0.state.amplitudes, r1.state.amplitudes)
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    assert rel_l2(r1.state.to_numpy(), ref) <= 1e-5


def test_jit_bitexact_at_32_qubits():
    """the auto policy's regime (2^31+ amplitudes per shard): 32 GiB states"""
    free, _ = torch.cuda.mem_get_info()
    if free < 2 * (1 << 32) * 8 + (4 << 30):
        pytest.skip("not enough device memory")
    gt, gp = random_arrays(RandomSpec(32, 60, 4))
    a, st0 = run(gt, gp, 32, -1)
    b, st1 = run(gt, gp, 32, 0)  # auto -> on at 32 qubits
    assert st1["enabled"] == 1 and st1["n_jit"] == st1["n_passes"]
    assert same_bits(a, b)
    del a, b
    torch.cuda.empty_cache()


def test_tiered_jit_is_bit_identical_across_tiers():
    """jit=auto on a 2^26 shard compiles in the background: the first execution mixes
    interpreter and compiled passes, a later plan of the same circuit starts fully
    compiled from the process-wide cache; every tier gives the same bits."""
    import torch

    n = 26
    gt, gp = random_arrays(RandomSpec(n, 300, 11))
    first = sv.CompiledCircuit(gt, gp, n, "fp32")
    assert first.jit_status()["enabled"] == 2
    s1 = sv.init_zero_state(n, "fp32")
    first.execute(s1)
    st = first.jit_status(wait=True)
    assert st["n_jit"] + st["n_fallback"] == st["n_passes"]
    second = sv.CompiledCircuit(gt, gp, n, "fp32")
    st2 = second.jit_status(wait=True)
    s2 = sv.init_zero_state(n, "fp32")
    second.execute(s2)
    ref = sv.init_zero_state(n, "fp32")
    sv.CompiledCircuit(gt, gp, n, "fp32", jit=-1).execute(ref)
    a, b, c = (torch.view_as_real(x.amplitudes) for x in (s1, s2, ref))
    assert torch.equal(a, c) and torch.equal(b, c)
    assert st2["n_jit"] == st["n_jit"]


@pytest.mark.parametrize("kind", ["random", "qft", "mixed"])
def test_jit_complex128_vs_oracle(kind):
    """complex128 circuit-specialised kernels (f64 DFMA code, .b128 amplitudes): the
    north_star fp64 tolerance 1e-12 against the oracle's fp64 run, and within a few
    ulps of the interpreter kernel (a different FMA association)."""
    n = 20
    if kind == "random":
        gt, gp = random_arrays(RandomSpec(n, 300, 4))
    elif kind == "qft":
        gt, gp = qft_arrays(n)
    else:
        g1, p1 = random_arrays(RandomSpec(n, 80, 5))
        g2, p2 = qft_arrays(n)
        gt, gp = np.concatenate([g1, g2]), np.concatenate([p1, p2])
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    plan = sv.CompiledCircuit(gt, gp, n, "fp64", jit=1)
    st = plan.jit_status(wait=True)
    assert st["enabled"] == 1 and st["n_jit"] == st["n_passes"]
    s1 = sv.init_zero_state(n, "fp64")
    plan.execute(s1)
    got = s1.to_numpy()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
    s0 = sv.init_zero_state(n, "fp64")
    sv.CompiledCircuit(gt, gp, n, "fp64", jit=-1).execute(s0)
    assert np.linalg.norm(got - s0.to_numpy()) / np.linalg.norm(ref) <= 1e-14


_STICKY_CHILD = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2504_03967_b200 import statevec as sv
from paper_2504_03967_b200.generators import RandomSpec, random_arrays
gt, gp = random_arrays(RandomSpec(24, 600, 5))
out = []
for jit in (-1, 1):
    plan = sv.CompiledCircuit(gt, gp, 24, "fp32", jit=jit)
    plan.jit_status(wait=True)
    st = sv.init_zero_state(24, "fp32", 1 << 40)
    plan.execute(st)
    out.append(torch.view_as_real(st.amplitudes).clone())
assert plan.jit_status(wait=True)["n_jit"] == plan.info["n_passes"]
print("bitexact", torch.equal(out[0], out[1]))
"""


def test_scoped_barriers_bitexact_with_sticky_warps():
    """The scoped SMEM hand-over barriers (jit.cpp hand_sync) are rarely scoped below the
    CTA on the default plans; QG_DEV_STICKY=1 makes the planner share warp bits between
    consecutive mappings, so most hand-overs sync a warp or a warp pair: the JIT state
    must still equal the interpreter's bit for bit (a missing barrier shows up as a race)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, QG_DEV_STICKY="1")
    r = subprocess.run([sys.executable, "-c", _STICKY_CHILD, root], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "bitexact True" in r.stdout, r.stdout + r.stderr[-2000:]
