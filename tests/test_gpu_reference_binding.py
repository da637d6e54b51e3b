"""GPU: the reference-side binding of INTEGRATION.md (tests/refshim.py) and this
package's run_circuit, both driven by the reference's OWN objects: circuits built
by qgear.generators from baseline/_ref (the unmodified reference install) and
checked against the reference's own statevec.run_circuit."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "qgear")), reason="baseline/_ref not installed")]


@pytest.fixture(scope="module")
def qgear():
    sys.path.insert(0, REF)
    import qgear.generators as g
    import qgear.ir as ir
    import qgear.statevec as s

    return g, s, ir


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
@pytest.mark.parametrize("kind", ["random", "qft"])
def test_shim_with_reference_circuits(qgear, prec, kind):
    g, s, _ = qgear
    from tests import refshim

    circ = g.generate_random_gate_list(g.RandomSpec(14, 80, 5)) if kind == "random" else g.build_qft(g.QftSpec(12))
    ref, _ = s.run_circuit(circ, s.SimOptions(precision=prec))
    got = refshim.run_circuit(circ, s.SimOptions(precision=prec)).cpu().numpy()
    want = ref.amplitudes.astype(np.complex128)
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert err <= (1e-12 if prec == "fp64" else 1e-5), err


def test_package_run_circuit_accepts_reference_objects(qgear):
    g, s, _ = qgear
    from paper_2504_03967_b200 import statevec as sv

    circ = g.generate_random_gate_list(g.RandomSpec(16, 100, 0, include_measure=True))
    ref, ref_counts = s.run_circuit(circ, s.SimOptions(precision="fp64", shots=3000, rng_seed=0))
    st, counts = sv.run_circuit(circ, sv.SimOptions("fp64", shots=3000, rng_seed=0, sampler="numpy"))
    assert np.linalg.norm(st.to_numpy() - ref.amplitudes) / np.linalg.norm(ref.amplitudes) <= 1e-12
    # the reference's exact uniform stream: the same counts up to cdf-rounding ties
    moved = sum(abs(counts.counts.get(k, 0) - v) for k, v in ref_counts.counts.items())
    assert counts.total == 3000 and moved <= 8


def test_shim_error_codes(qgear):
    _, s, ir = qgear
    from tests import refshim

    bad = type("C", (), {})()
    bad.n_qubits = 3
    bad.active_gates = [ir.GateRecord(ir.GateKind.H, None, 7, 0.0)]
    with pytest.raises(refshim.B200Error) as e:
        refshim.run_circuit(bad, s.SimOptions())
    assert e.value.code == -2  # QG_E_INDEX_OUT_OF_RANGE -> IndexOutOfRangeError
