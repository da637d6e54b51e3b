"""GPU parity: libqgear_b200 CUDA kernels vs the CPU oracle and the reference's golden vectors.

Tolerances (BASELINE.json:north_star): relative L2 <= 1e-12 for complex128
("fp64") and <= 1e-5 for complex64 ("fp32"), against the oracle's fp64 run.
Counts: total-variation bound on marginals (SPEC.md:239 style binomial bound).
"""

import math

import numpy as np
import pytest
import torch

import oracle
from paper_2504_03967_b200 import errors as E
from paper_2504_03967_b200 import statevec as sv
from paper_2504_03967_b200.generators import QftSpec, RandomSpec, build_qft, generate_random_gate_list
from paper_2504_03967_b200.generators import qft_arrays, random_arrays
from paper_2504_03967_b200.ir import CircType, CircuitTensor, GateKind, GateRecord

pytestmark = pytest.mark.gpu

TOL = {"fp64": 1e-12, "fp32": 1e-5}


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a, dtype=np.complex128) - b) / np.linalg.norm(b))


def circuit(gt, gp, n):
    return CircuitTensor.from_arrays(CircType.IMPORTED, n, gt, gp)


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


# ----------------------------------------------------------------- golden states
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("fuse", [True, False])
def test_golden_states(golden, precision, fuse):
    for name in golden["state_cases"]:
        nq, ng = (int(v) for v in golden[f"state_{name}_hdr"])
        c = circuit(golden[f"state_{name}_type"][:ng], golden[f"state_{name}_param"][:ng], nq)
        st, _ = sv.run_circuit(c, sv.SimOptions(precision=precision, fuse=fuse))
        got = st.to_numpy()
        assert got.dtype == (np.complex128 if precision == "fp64" else np.complex64)
        err = rel_l2(got, golden[f"state_{name}_fp64"])
        assert err <= TOL[precision], (name, precision, fuse, err)


def test_cfg1_state_and_counts(golden):
    """BASELINE config 1: RandomSpec(16,100,0), complex128, 3000 shots."""
    c = generate_random_gate_list(RandomSpec(16, 100, 0))
    st, counts = sv.run_circuit(c, sv.SimOptions("fp64", 3000, 0, sampler="numpy"))
    assert rel_l2(st.to_numpy(), golden["cfg1_state_fp64"]) <= 1e-12
    assert counts.total == 3000 and sum(counts.counts.values()) == 3000
    # numpy-uniform mode reproduces the reference's Generator.choice draws
    ref = dict(zip(golden["cfg1_count_keys"].tolist(), golden["cfg1_count_value"].tolist()))
    diff = sum(abs(counts.counts.get(k, 0) - v) for k, v in ref.items()) + sum(
        v for k, v in counts.counts.items() if k not in ref)
    assert diff <= 4, diff  # only cdf-rounding ties may move a shot


@pytest.mark.parametrize("j", range(4))
def test_sampler_numpy_mode_matches_reference_counts(golden, j):
    n, shots, seed = (int(v) for v in golden[f"sample{j}_meta"])
    amps = torch.from_numpy(golden[f"sample{j}_amps"]).cuda()
    idx, cnt = sv.sample_indices(amps, shots, seed, "numpy")
    got = dict(zip(idx.cpu().tolist(), cnt.cpu().tolist()))
    ref = dict(zip(golden[f"sample{j}_index"].tolist(), golden[f"sample{j}_value"].tolist()))
    diff = sum(abs(got.get(k, 0) - v) for k, v in ref.items()) + sum(v for k, v in got.items() if k not in ref)
    assert diff <= 2, diff


# ----------------------------------------------------------------- random / qft / mixed at larger n
@pytest.mark.parametrize("n,blocks", [(18, 400), (20, 200), (22, 60)])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_random_cx_vs_oracle(n, blocks, precision):
    gt, gp = random_arrays(RandomSpec(n, blocks, n))
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    st, _ = sv.run_circuit(circuit(gt, gp, n), sv.SimOptions(precision=precision))
    assert rel_l2(st.to_numpy(), ref) <= TOL[precision]


@pytest.mark.parametrize("n", [14, 20])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_mixed_vs_oracle(n, precision):
    gt, gp = mixed(n, 400, n + 100)
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    for fuse in (True, False):
        st, _ = sv.run_circuit(circuit(gt, gp, n), sv.SimOptions(precision=precision, fuse=fuse))
        assert rel_l2(st.to_numpy(), ref) <= TOL[precision], fuse


@pytest.mark.parametrize("opts", [dict(max_stages=1), dict(max_stages=2, max_cost=30), dict(max_cost=12),
                                  dict(tile_qubits=8), dict(tile_qubits=11), dict(max_stages=8, max_cost=400)])
def test_planner_knobs_on_gpu(opts):
    n = 20
    gt, gp = mixed(n, 300, 5)
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    prec = "fp64" if opts.get("tile_qubits") not in (11,) else "fp32"
    if opts.get("tile_qubits") == 8:
        prec = "fp32"
    st, _ = sv.run_circuit(circuit(gt, gp, n), sv.SimOptions(precision=prec, **opts))
    assert rel_l2(st.to_numpy(), ref) <= TOL[prec]


@pytest.mark.parametrize("n,precision", [(24, "fp32"), (26, "fp32"), (25, "fp64")])
def test_qft_closed_form(n, precision):
    """build_qft on |0..0> is the uniform state (controls never fire)."""
    st, _ = sv.run_circuit(build_qft(QftSpec(n)), sv.SimOptions(precision=precision, memory_budget=1 << 40))
    a = st.amplitudes
    expect = 2.0 ** (-n / 2)
    err = torch.linalg.vector_norm(a - expect).item() / 1.0
    assert err <= TOL[precision] * 10, err


def test_qft_on_basis_state_is_dft():
    """Verified identity: input bitrev(k) -> exp(+2*pi*i*j*k/2^n)/sqrt(2^n) at index j."""
    n, k = 18, 77777
    rk = int(format(k, f"0{n}b")[::-1], 2)
    gt, gp = qft_arrays(n)
    # prepare |rk> with X = RX(pi) up to a global phase (-i)^popcount
    pre = [(GateKind.RX, -1, q) for q in range(n) if (rk >> q) & 1]
    gt2 = np.concatenate([np.array(pre, dtype=np.int32).reshape(-1, 3), gt])
    gp2 = np.concatenate([np.full(len(pre), math.pi), gp])
    st, _ = sv.run_circuit(circuit(gt2, gp2, n), sv.SimOptions(precision="fp64"))
    got = st.to_numpy() * (1j ** len(pre))
    j = np.arange(1 << n, dtype=np.int64)
    ph = ((j * k) % (1 << n)).astype(np.float64) / (1 << n)  # exact phase index, then one rounding
    expect = np.exp(2j * np.pi * ph) / math.sqrt(1 << n)
    assert rel_l2(got, expect) <= 1e-11


def _basis_then_qft(n, k, reversed_=False):
    """|bitrev(k)> prepared with X = RX(pi) (global phase (-i)^popcount), then QFT(n)."""
    rk = int(format(k, f"0{n}b")[::-1], 2)
    gt, gp = qft_arrays(n, reversed_)
    pre = [(GateKind.RX, -1, q) for q in range(n) if (rk >> q) & 1]
    gt2 = np.concatenate([np.array(pre, dtype=np.int32).reshape(-1, 3), gt])
    gp2 = np.concatenate([np.full(len(pre), math.pi), gp])
    return gt2, gp2, len(pre)


@pytest.mark.parametrize("jit", [-1, 1])
def test_qft28_complex64_on_basis_state_is_dft(jit):
    """C2 scale (QFT 28 q, complex64) with FIRING controlled phases: on |0...0> every
    CR1 acts as the identity, on |bitrev(k)> every row's phase list is non-trivial
    (long predicated PH lists, tile-uniform slots, register/thread-controlled factors).
    Checked on the device against the closed form e^{2 pi i j k / 2^n} / sqrt(2^n),
    rel-L2 <= 1e-5 (north_star complex64 tolerance)."""
    n, k = 28, 0x5A5A5A7
    gt, gp, npre = _basis_then_qft(n, k)
    st, _ = sv.run_circuit(circuit(gt, gp, n), sv.SimOptions(precision="fp32", memory_budget=1 << 40, jit=jit))
    a = st.amplitudes
    phase = complex(1j ** npre)
    num = den = 0.0
    step = 1 << 24
    for j0 in range(0, 1 << n, step):
        j = torch.arange(j0, j0 + step, dtype=torch.int64, device=a.device)
        ph = ((j * k) % (1 << n)).to(torch.float64) * (2 * math.pi / (1 << n))
        expect = torch.polar(torch.full_like(ph, 2.0 ** (-n / 2)), ph)
        got = a[j0:j0 + step].to(torch.complex128) * phase
        num += float(torch.linalg.vector_norm(got - expect) ** 2)
        den += float(torch.linalg.vector_norm(expect) ** 2)
    assert math.sqrt(num / den) <= 1e-5


@pytest.mark.parametrize("n,reversed_", [(24, False), (22, True)])
def test_qft_after_random_ry_layer_vs_oracle(n, reversed_):
    """QFT on a generic (non-basis) input: every phase list fires with amplitude-dependent
    weight; complex64 against the oracle's fp64 run."""
    rng = np.random.default_rng(n)
    pre_t = np.array([(GateKind.RY, -1, q) for q in range(n)], dtype=np.int32)
    pre_p = rng.uniform(0, 2 * math.pi, n)
    gt, gp = qft_arrays(n, reversed_)
    gt2, gp2 = np.concatenate([pre_t, gt]), np.concatenate([pre_p, gp])
    ref = oracle.run_arrays(gt2, gp2, n, gt2.shape[0], "fp64")
    st, _ = sv.run_circuit(circuit(gt2, gp2, n), sv.SimOptions(precision="fp32", memory_budget=1 << 40))
    assert rel_l2(st.to_numpy(), ref) <= 1e-5


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_circuit_then_inverse_is_identity(precision):
    n = 27 if precision == "fp32" else 26
    gt, gp = random_arrays(RandomSpec(n, 400, 9))
    inv_t = gt[::-1].copy()
    inv_p = -gp[::-1]
    c = circuit(np.concatenate([gt, inv_t]), np.concatenate([gp, inv_p]), n)
    st, _ = sv.run_circuit(c, sv.SimOptions(precision=precision, memory_budget=1 << 40))
    a0 = st.amplitudes[0].item()
    rest = torch.linalg.vector_norm(st.amplitudes[1:]).item()
    tol = 1e-10 if precision == "fp64" else 1e-4
    assert abs(a0 - 1) < tol and rest < tol


# ----------------------------------------------------------------- array kernels & per-gate API
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_array_kernels_vs_oracle(precision):
    rng = np.random.default_rng(3)
    n = 12
    a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    a /= np.linalg.norm(a)
    a = a.astype(np.complex64 if precision == "fp32" else np.complex128)
    dev = torch.from_numpy(a.copy()).cuda()
    ref = a.copy()
    for step in range(60):
        kind = int(rng.integers(0, 6))
        t = int(rng.integers(0, n))
        c = int(rng.integers(0, n - 1))
        c = c if c < t else c + 1
        th = float(rng.uniform(-6, 6))
        if kind == 4:
            sv.swap_target_pairs_array(dev, c, t)
            oracle.apply_cx_swap(ref, c, t)
        elif kind == 5:
            sv.phase_pairs_array(dev, c, t, th)
            oracle.apply_cr1_phase(ref, c, t, th)
        else:
            u = sv.gate_matrix_2x2(GateKind(kind), th)
            sv.apply_matrix_array(dev, t, u)
            oracle.apply_pair_matrix(ref, t, oracle.gate_matrix(kind, th))
    tol = 1e-13 if precision == "fp64" else 1e-6
    assert rel_l2(dev.cpu().numpy(), ref.astype(np.complex128)) <= tol
    if precision == "fp64":  # CX is a pure permutation: bit-exact
        b = torch.from_numpy(a.copy()).cuda()
        sv.swap_target_pairs_array(b, 3, 7)
        r = a.copy()
        oracle.apply_cx_swap(r, 3, 7)
        assert np.array_equal(b.cpu().numpy(), r)


def test_gate_api_errors():
    st = sv.init_zero_state(3, "fp64")
    with pytest.raises(E.IndexOutOfRangeError):
        sv.apply_1q(st, GateKind.H, 3)
    with pytest.raises(E.SelfPairError):
        sv.apply_cx(st, 1, 1)
    with pytest.raises(E.IndexOutOfRangeError):
        sv.apply_cr1(st, 0, 5, 0.3)
    with pytest.raises(E.TooManyQubitsError) as ei:
        sv.init_zero_state(60, "fp64")
    assert ei.value.required_bytes == 16 * 2**60
    with pytest.raises(ValueError):
        sv.init_zero_state(0)
    # App. A: 3q, |100> (index 1), CX(q0 -> q2) -> |101> (index 5)
    st = sv.init_zero_state(3, "fp64")
    sv.apply_1q(st, GateKind.RX, 0, math.pi)
    sv.apply_cx(st, 0, 2)
    p = sv.exact_probabilities(st).cpu().numpy()
    assert abs(p[5] - 1) < 1e-15


def test_run_circuit_errors():
    bad = CircuitTensor.from_arrays(CircType.IMPORTED, 2, [[6, -1, 0], [0, -1, 0]], [0.0, 0.0])
    with pytest.raises(E.MeasureMidCircuitError):
        sv.run_circuit(bad)
    with pytest.raises(E.TooManyQubitsError):
        sv.run_circuit(build_qft(QftSpec(31)), sv.SimOptions(precision="fp64"))
    big = sv.init_zero_state(4, "fp32")
    big.amplitudes.mul_(2.0)
    with pytest.raises(E.UnnormalizedStateError):
        sv.sample_counts(big, 10)
    with pytest.raises(ValueError):
        sv.sample_counts(sv.init_zero_state(2), 0)


# ----------------------------------------------------------------- sampling statistics
def _tv_bound(k, shots):
    return 4 * 0.5 * math.sqrt(k / shots)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_sampler_tv_and_determinism(precision):
    n = 20
    gt, gp = random_arrays(RandomSpec(n, 200, 1))
    st, _ = sv.run_circuit(circuit(gt, gp, n), sv.SimOptions(precision=precision))
    p = oracle.exact_probabilities(oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64"))
    shots = 200_000
    t1 = sv.sample_counts(st, shots, 5)
    t2 = sv.sample_counts(st, shots, 5)
    assert t1.counts == t2.counts and t1.total == shots and sum(t1.values.tolist()) == shots
    # marginal over the b lowest qubits
    b = min(n, int(math.log2(shots / 64)))
    emp = np.bincount(t1.indices & ((1 << b) - 1), weights=t1.values, minlength=1 << b) / shots
    exact = np.bincount(np.arange(1 << n) & ((1 << b) - 1), weights=p, minlength=1 << b)
    tv = 0.5 * np.abs(emp - exact).sum()
    assert tv <= _tv_bound(1 << b, shots), tv
    # per-qubit z-test at 5 sigma
    for q in range(n):
        pq = float(p[(np.arange(1 << n) >> q) & 1 == 1].sum())
        eq = float(t1.values[((t1.indices >> q) & 1) == 1].sum()) / shots
        sd = math.sqrt(max(pq * (1 - pq), 1e-12) / shots)
        assert abs(eq - pq) <= 5 * sd + 1e-9, q


def test_sampler_edge_cases():
    st = sv.init_zero_state(1, "fp64")
    sv.apply_1q(st, GateKind.H, 0)
    t = sv.sample_counts(st, 100000, 0)
    assert 0.49 <= t.counts["0"] / 100000 <= 0.51
    st = sv.init_zero_state(2, "fp64")  # |01> display: qubit 0 = 0, qubit 1 = 1 -> index 2
    sv.apply_1q(st, GateKind.RY, 1, math.pi)
    t = sv.sample_counts(st, 777, 3)
    assert t.counts == {"01": 777}
    # deterministic zero-probability outcomes never appear
    st = sv.init_zero_state(17, "fp32")
    sv.apply_1q(st, GateKind.H, 16)
    t = sv.sample_counts(st, 50000, 1)
    assert set(t.indices.tolist()) <= {0, 1 << 16}
    # one shot; and the Philox path's ascending-order-statistics draws on a skewed
    # distribution (p = sin^2(0.05) ~ 2.5e-3 on |1>): unique ascending outcomes, exact total
    t = sv.sample_counts(st, 1, 9)
    assert t.total == 1 and sum(t.values.tolist()) == 1
    st = sv.init_zero_state(1, "fp32")
    sv.apply_1q(st, GateKind.RY, 0, 0.1)
    shots = 400_000
    t = sv.sample_counts(st, shots, 11)
    assert t.indices.tolist() == [0, 1] and sum(t.values.tolist()) == shots
    p1 = math.sin(0.05) ** 2
    assert abs(t.values[1] / shots - p1) <= 5 * math.sqrt(p1 * (1 - p1) / shots)

# every fused-kernel instantiation (kernel_cfg = 1 + id; c64: 8 configs incl. the
# 32/64-amplitude-per-thread ones, c128: 4) against the oracle on a mixed circuit
@pytest.mark.parametrize("precision,cfg", [("fp32", c) for c in range(1, 9)] + [("fp64", c) for c in range(1, 5)])
def test_every_kernel_config_vs_oracle(precision, cfg):
    n = 17
    gt, gp = mixed(n, 500, 30 + cfg)
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    plan = sv.CompiledCircuit(gt, gp, n, precision, kernel_cfg=cfg)
    st = sv.init_zero_state(n, precision)
    plan.execute(st)
    assert rel_l2(st.to_numpy(), ref) < (1e-12 if precision == "fp64" else 1e-5)


# tiny states (below every fused tile: the single-gate kernel path) and edge inputs
@pytest.mark.parametrize("n", range(1, 10))
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_small_states_vs_oracle(n, precision):
    gt, gp = mixed(n, 60, 200 + n)
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    st, counts = sv.run_circuit(circuit(gt, gp, n), sv.SimOptions(precision=precision, shots=256, rng_seed=1))
    assert rel_l2(st.to_numpy(), ref) <= TOL[precision]
    assert counts.total == 256 and all(len(k) == n for k in counts.counts)


def test_empty_and_measure_only_circuits():
    for gates in ([], [GateRecord.measure(0), GateRecord.measure(2)]):
        c = CircuitTensor.from_gates(CircType.IMPORTED, 3, gates)
        st, counts = sv.run_circuit(c, sv.SimOptions("fp64", shots=10))
        ref = np.zeros(8, dtype=np.complex128)
        ref[0] = 1
        assert np.array_equal(st.to_numpy(), ref)
        assert counts.counts == {"000": 10}
