"""IR and generator parity with the reference (golden arrays from the reference itself)."""

import math

import numpy as np
import pytest

from paper_2504_03967_b200 import errors as E
from paper_2504_03967_b200 import ir
from paper_2504_03967_b200.generators import (QftSpec, RandomSpec, build_qft, generate_random_gate_list,
                                              random_qubit_pairs)

RSPECS = [(2, 5, 0, False), (5, 7, 3, True), (16, 100, 0, False), (32, 1000, 0, False),
          (32, 1000, 1, False), (36, 1000, 0, False), (37, 1000, 0, False), (20, 50, 7, True)]


@pytest.mark.parametrize("n,b,s,m", RSPECS)
def test_random_stream_bit_identical(golden, n, b, s, m):
    c = generate_random_gate_list(RandomSpec(n, b, s, m))
    key = f"gen_random_{n}_{b}_{s}_{int(m)}"
    assert np.array_equal(c.gate_type, golden[key + "_type"])
    assert np.array_equal(c.gate_param, golden[key + "_param"])  # exact float64 equality
    assert c.n_gates == 3 * b + (n if m else 0)


@pytest.mark.parametrize("n,rev", [(1, False), (6, False), (6, True), (28, False), (37, True)])
def test_qft_bit_identical(golden, n, rev):
    c = build_qft(QftSpec(n, rev))
    key = f"gen_qft_{n}_{int(rev)}"
    assert np.array_equal(c.gate_type, golden[key + "_type"])
    assert np.array_equal(c.gate_param, golden[key + "_param"])
    assert c.n_gates == n * (n + 1) // 2


def test_random_qubit_pairs(golden):
    assert random_qubit_pairs(5, 64, 1) == [tuple(p) for p in golden["pairs_5_64_1"].tolist()]
    pairs = random_qubit_pairs(5, 10000, 0)  # SPEC.md:379 frequencies 0.05 +- 0.01
    freq = np.bincount([c * 5 + t for c, t in pairs], minlength=25) / 10000
    assert all(0.04 <= freq[c * 5 + t] <= 0.06 for c in range(5) for t in range(5) if c != t)
    with pytest.raises(E.TooFewQubitsError):
        random_qubit_pairs(1, 3)


def test_encode_and_arrays_match_reference(golden):
    GR = ir.GateRecord
    lists = [
        (ir.CircType.IMPORTED, 3, [GR.h(0), GR.cr1(0, 2, -1.0), GR.cr1(2, 1, 7.5), GR.rz(1, -9.0)]),
        (ir.CircType.QFT, 2, [GR.cr1(1, 0, 2 * math.pi), GR.measure(0), GR.measure(1)]),
        (ir.CircType.RANDOM, 4, []),
    ]
    cs = ir.encode_circuits(lists)
    h, gt, gp = ir.set_to_arrays(cs)
    assert np.array_equal(h, golden["enc_headers"])
    assert np.array_equal(gt, golden["enc_type"])
    assert np.array_equal(gp, golden["enc_param"])
    back = ir.set_from_arrays(h, gt, gp, cs.metadata)
    assert back == cs
    dec = ir.decode_circuits(back)
    assert [len(g) for _, _, g in dec] == [4, 3, 0]
    assert dec[0][2][1] == GR.cr1(0, 2, (-1.0) % (2 * math.pi))
    assert ir.validate(cs).ok


def test_ir_error_cases():
    GR = ir.GateRecord
    with pytest.raises(E.EmptyInputError):
        ir.encode_circuits([])
    with pytest.raises(E.InvalidQubitIndexError):
        ir.encode_circuits([(0, 2, [GR.h(2)])])
    with pytest.raises(E.SelfPairError):
        ir.encode_circuits([(0, 2, [GR.cx(1, 1)])])
    with pytest.raises(E.NonFiniteParamError):
        ir.encode_circuits([(0, 2, [GR.rx(1, float("inf"))])])
    with pytest.raises(E.InvalidGateError):
        ir.encode_circuits([(0, 2, [GR(ir.GateKind.H, 1, 0)])])
    h = np.array([[0, 2, 1]], dtype=np.int32)
    gt = np.array([[[0, -1, 0], [7, -1, 0]]], dtype=np.int32)
    with pytest.raises(E.CorruptTensorError):
        ir.set_from_arrays(h, gt, np.zeros((1, 2)))
    with pytest.raises(E.CorruptTensorError):
        ir.set_from_arrays(np.array([[9, 2, 1]]), gt[:, :1], np.zeros((1, 1)))
    with pytest.raises(E.CorruptTensorError):
        ir.set_from_arrays(h, gt[:, :1], np.zeros((2, 1)))
    cs = ir.set_from_arrays(h, np.array([[[0, -1, 0], [0, -1, 1]]], dtype=np.int32), np.zeros((1, 2)))
    with pytest.raises(E.CorruptTensorError):  # non-zero padding after n_gates
        ir.decode_circuits(cs)
    rep = ir.validate(cs)
    assert not rep.ok and rep.violations[0].code == "PaddingViolation"


def test_circuit_tensor_records_roundtrip():
    c = build_qft(QftSpec(4))
    assert c.count_kind(ir.GateKind.CR1) == 6
    r = c.repadded(20)
    assert r.capacity == 20 and r.active_gates == c.active_gates
    assert ir.CircuitTensor.from_gates(ir.CircType.QFT, 4, list(c.active_gates)) == c
