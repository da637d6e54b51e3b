"""QCrank: encoder / circuit builder / decoder on CPU, and the
collapsed execution (fused passes + one-pass uniformly controlled RY kernel)
on the GPU, all checked against the reference simulator's algorithm (oracle)
running the full gate-level circuit.

The reference ships no QCrank code, so the pins are the spec's examples,
derived identities (SPEC.md "examples" / "Invariants") and the oracle.
"""

import math

import numpy as np
import pytest

import oracle
from paper_2504_03967_b200 import qcrank as qc
from paper_2504_03967_b200.errors import LengthMismatchError, PlanTooSmallError
from paper_2504_03967_b200.ir import GateKind


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def product_state(alpha: np.ndarray) -> np.ndarray:
    """amp(a, x) = 2^-m/2 prod_d (x_d ? sin : cos)(alpha[a, d] / 2): H^m then UCRYs from |0>."""
    n_a, nd = alpha.shape
    m = n_a.bit_length() - 1
    idx = np.arange(1 << (m + nd))
    a = idx & (n_a - 1)
    amp = np.full(idx.size, 2.0 ** (-m / 2))
    for d in range(nd):
        bit = (idx >> (m + d)) & 1
        amp = amp * np.where(bit == 1, np.sin(alpha[a, d] / 2), np.cos(alpha[a, d] / 2))
    return amp.astype(np.complex128)


def test_spec_example_m1():
    a0, a1 = 0.7, 2.1
    gt, gp = qc.ucry_gate_arrays(np.array([a0, a1]), [0], 1)
    assert gt.tolist() == [[GateKind.RY, -1, 1], [GateKind.CX, 0, 1], [GateKind.RY, -1, 1], [GateKind.CX, 0, 1]]
    assert gp[0] == pytest.approx((a0 + a1) / 2) and gp[2] == pytest.approx((a0 - a1) / 2)
    # dense check: address 0 sees RY(a0), address 1 sees RY(a1)
    for addr, ang in ((0, a0), (1, a1)):
        psi = np.zeros(4, dtype=np.complex128)
        psi[addr] = 1
        for (k, c, t), p in zip(gt, gp):
            oracle.statevec_oracle.apply_gate(psi, int(k), int(c), int(t), float(p))
        assert abs(psi[addr] - math.cos(ang / 2)) < 1e-12 and abs(psi[addr | 2] - math.sin(ang / 2)) < 1e-12


def test_gray_walsh_involution_and_controls():
    rng = np.random.default_rng(3)
    for m in range(0, 8):
        alpha = rng.uniform(0, math.pi, 1 << m)
        assert np.max(np.abs(qc.inverse_gray_walsh(qc.gray_walsh(alpha)) - alpha)) < 1e-12
    assert qc.gray_controls(3).tolist() == [0, 1, 0, 2, 0, 1, 0, 2]


@pytest.mark.parametrize("m,nd", [(1, 1), (3, 2), (4, 3), (5, 1)])
def test_circuit_matches_product_state_on_oracle(m, nd):
    rng = np.random.default_rng(m * 10 + nd)
    alpha = rng.uniform(0, math.pi, (1 << m, nd))
    gt, gp, n = qc.build_qcrank_circuit(alpha)
    assert n == m + nd
    assert qc.cx_count(gt) == nd << m                      # SPEC: CX count = padded pixel count
    got = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    assert rel_l2(got, product_state(alpha)) < 1e-12


def test_collapse_recovers_angles():
    rng = np.random.default_rng(7)
    alpha = rng.uniform(0, math.pi, (1 << 6, 3))
    gt, gp, n = qc.build_qcrank_circuit(alpha, measure=False)
    items = qc.collapse_ucry(gt, gp, min_addr=4)
    kinds = [it[0] for it in items]
    assert kinds == ["gates", "ucry", "ucry", "ucry"]
    for d, it in enumerate(items[1:]):
        seg = it[1]
        assert seg.target == 6 + d and seg.addr_qubits == list(range(6))
        assert np.max(np.abs(seg.alpha - alpha[:, d])) < 1e-12
    # below the threshold nothing is collapsed
    assert [it[0] for it in qc.collapse_ucry(gt, gp, min_addr=7)] == ["gates"]
    # permuted address register (non-contiguous, shuffled bit order) is recognised too
    perm = [5, 0, 3, 1, 4, 2]
    bt, bp = qc.ucry_gate_arrays(alpha[:, 0], perm, 6)
    seg = qc.collapse_ucry(bt, bp)[0][1]
    assert seg.addr_qubits == perm and np.max(np.abs(seg.alpha - alpha[:, 0])) < 1e-12


def test_prepare_angles_examples():
    img = qc.ImageGray(2, 1, np.array([255, 0], dtype=np.uint8))
    th = qc.prepare_angles(img, 1, 1)
    assert th[0, 0] == 0.0 and th[1, 0] == pytest.approx(math.pi)
    # bit reversal: m = 3, pixel group 1 lands at address 4; padding = pi/2
    img = qc.ImageGray(3, 1, np.array([10, 20, 30], dtype=np.uint8))
    th = qc.prepare_angles(img, 3, 1)
    assert th[4, 0] == pytest.approx(math.acos(2 * 20 / 255 - 1))
    assert th[0, 0] == pytest.approx(math.acos(2 * 10 / 255 - 1)) and th[2, 0] == pytest.approx(math.acos(2 * 30 / 255 - 1))
    assert np.all(th[[1, 3, 5, 6, 7], 0] == math.pi / 2)
    # Table 2 "Finger 64x80 5k 10 5": (1024, 5) tensor
    finger = qc.ImageGray(64, 80, np.zeros(64 * 80, dtype=np.uint8))
    assert qc.prepare_angles(finger, 10, 5).shape == (1024, 5)
    with pytest.raises(PlanTooSmallError):
        qc.prepare_angles(finger, 9, 5)
    assert qc.make_plan(finger, 10, 5).shots == 3_072_000      # "3M" shots (s * 2^m)
    zebra = qc.QCrankPlan(13, 12)
    assert zebra.padded_len == 98_304                          # Zebra row, CX count


def test_decode_exact_round_trip_and_errors():
    rng = np.random.default_rng(11)
    m, nd = 5, 2
    img = qc.ImageGray(8, 8, rng.integers(0, 256, 64, dtype=np.uint8))
    plan = qc.make_plan(img, m, nd)
    alpha = qc.prepare_angles(img, m, nd)
    gt, gp, n = qc.build_qcrank_circuit(alpha)
    psi = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    rep, out = qc.decode_exact(np.abs(psi) ** 2, plan, img)
    truth = 2 * img.pixels.astype(np.float64) / 255 - 1
    assert np.max(np.abs(rep.estimates - truth)) < 1e-9
    assert np.max(np.abs(out.pixels.astype(int) - img.pixels.astype(int))) <= 1
    assert rep.correlation > 0.999999
    uni, _ = qc.decode_exact(np.full(1 << n, 1 / (1 << n)), plan)
    assert np.allclose(uni.estimates, 0.0)
    with pytest.raises(LengthMismatchError):
        qc.decode_exact(np.ones(8), plan)


def test_decode_counts_deterministic():
    plan = qc.QCrankPlan(2, 1, 4, 1)
    # every address: all shots on data bit 0 -> v = +1 ; address 3 empty
    idx = np.array([0, 1, 2], dtype=np.int64)
    cnt = np.array([5, 7, 9], dtype=np.int64)
    rep, img = qc.decode_counts((idx, cnt), plan)
    assert rep.empty_addresses == [3]
    assert np.all(rep.estimates[[0, 2, 1]] == 1.0)  # addresses 0, 1, 2 = pixel groups 0, 2, 1
    assert rep.estimates[3] == 0.0 and img.pixels[0] == 255


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("precision,tol", [("fp64", 1e-12), ("fp32", 1e-5)])
def test_collapsed_run_matches_oracle(precision, tol):
    from paper_2504_03967_b200 import statevec as sv

    rng = np.random.default_rng(5)
    m, nd = 7, 4
    alpha = rng.uniform(0, math.pi, (1 << m, nd))
    gt, gp, n = qc.build_qcrank_circuit(alpha)
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    st, _ = qc.run_gates(gt, gp, n, sv.SimOptions(precision))
    assert rel_l2(st.to_numpy(), ref) < tol
    # gate-level path (no collapse) agrees as well
    st2, _ = qc.run_gates(gt, gp, n, sv.SimOptions(precision), min_addr=99)
    assert rel_l2(st2.to_numpy(), ref) < tol


@pytest.mark.gpu
def test_apply_ucry_general_registers():
    from paper_2504_03967_b200 import statevec as sv

    rng = np.random.default_rng(9)
    n = 11
    addr = [9, 2, 6, 0]          # shuffled, non-contiguous address register
    targets = [4, 10, 1]
    alpha = rng.uniform(-3, 3, (1 << len(addr), len(targets)))
    # oracle: random start state from a random circuit, then the gate-level Gray blocks
    from paper_2504_03967_b200.generators import RandomSpec, random_arrays

    g0, p0 = random_arrays(RandomSpec(n, 40, 2))
    parts_t, parts_p = [g0], [p0]
    for j, t in enumerate(targets):
        bt, bp = qc.ucry_gate_arrays(alpha[:, j], addr, t)
        parts_t.append(bt)
        parts_p.append(bp)
    gt, gp = np.concatenate(parts_t), np.concatenate(parts_p)
    ref = oracle.run_arrays(gt, gp, n, gt.shape[0], "fp64")
    plan = sv.CompiledCircuit(g0, p0, n, "fp64")
    st = sv.init_zero_state(n, "fp64", 1 << 30)
    plan.execute(st)
    qc.apply_ucry(st, addr, targets, alpha)
    assert rel_l2(st.to_numpy(), ref) < 1e-12


@pytest.mark.gpu
def test_image_round_trip_with_shots():
    from paper_2504_03967_b200 import statevec as sv

    rng = np.random.default_rng(21)
    img = qc.ImageGray(8, 8, rng.integers(0, 256, 64, dtype=np.uint8))
    m, nd = 4, 4
    plan = qc.make_plan(img, m, nd)
    st, counts = qc.simulate(qc.prepare_angles(img, m, nd), sv.SimOptions("fp32", shots=plan.shots, rng_seed=3))
    rep, out = qc.decode_counts(counts, plan, img)
    # SPEC: s = 3000 per address -> per-pixel sigma <= 1/sqrt(3000) in v units; correlation >= 0.99
    assert rep.correlation >= 0.99
    assert rep.max_abs_error < 6 / math.sqrt(plan.shots_per_address)
    rep_x, _ = qc.decode_exact(sv.exact_probabilities(st), plan, img)
    assert rep_x.max_abs_error < 1e-5


@pytest.mark.gpu
def test_sample_decode_dense_tally_matches_counts():
    """sample_decode (tree sampler dense counts -> qg_qcrank_tally on the device) agrees
    with the host marginals of the same counts, and reconstructs the image within the
    shot-noise bound at the paper's budget s * 2^m."""
    import torch

    from paper_2504_03967_b200 import statevec as sv

    rng = np.random.default_rng(5)
    m, nd = 10, 3
    img = qc.ImageGray(32, 96, rng.integers(0, 256, (1 << m) * nd, dtype=np.uint8))
    plan = qc.make_plan(img, m, nd)
    st, _ = qc.simulate(qc.prepare_angles(img, m, nd), sv.SimOptions("fp32"))
    rep, _ = qc.sample_decode(st, plan, 7, img)
    assert rep.correlation >= 0.99 and rep.max_abs_error < 6 / math.sqrt(plan.shots_per_address)
    # the device tally equals the host marginals of the same dense counts
    ts = sv.TreeSampler(st.amplitudes)
    ts.prepare()
    dense = ts.draw(plan.shots, 7, dense=True)
    tot = torch.empty(1 << m, dtype=torch.int64, device=dense.device)
    n1 = torch.empty((1 << m, nd), dtype=torch.int64, device=dense.device)
    sv.N.call("qg_qcrank_tally", sv.C.c_void_p(dense.data_ptr()), m, nd, sv.C.c_void_p(tot.data_ptr()),
              sv.C.c_void_p(n1.data_ptr()), sv._stream(dense.device))
    d = dense.cpu().numpy()
    idx = np.flatnonzero(d)
    h0, h1, ht = qc._lane_marginals(idx, d[idx], plan)
    assert np.array_equal(ht, tot.cpu().numpy()) and np.array_equal(h1, n1.cpu().numpy())
    assert int(tot.sum()) == plan.shots
    rep_h, img_h = qc._reconstruct(h0, h1, ht, plan, img)
    rep_d, img_d = qc._reconstruct_device(tot, n1, plan, img)
    assert np.array_equal(img_h.pixels, img_d.pixels) and np.allclose(rep_h.estimates, rep_d.estimates, atol=1e-15)
    assert abs(rep_h.mse - rep_d.mse) <= 1e-12 and rep_h.empty_addresses == rep_d.empty_addresses
