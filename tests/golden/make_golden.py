"""Generate the golden fixtures under tests/golden/ from the REFERENCE package.

Run once in the dev container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference's own Python modules from /root/reference/pkg/src
(qgear.ir / statevec / partition / generators; container.py is not imported
because h5py is absent) and freezes their outputs as .npz files.  Nothing in
the GPU tests, smoke() or bench.py reads /root/reference; they read these
fixtures instead.

Reference entry points exercised (file:line in /root/reference/pkg/src/qgear):
  generators.generate_random_gate_list  generators.py:61-79
  generators.build_qft                  generators.py:82-101
  generators.random_qubit_pairs         generators.py:42-58
  statevec.run_circuit                  statevec.py:200-212
  statevec.sample_counts                statevec.py:221-234
  statevec.exact_probabilities          statevec.py:215-218
  partition.plan / execute_distributed  partition.py:100-109, 286-355
  ir.encode_circuits / set_to_arrays    ir.py:219-253, 281-303
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF_SRC)
    from qgear import generators, ir, partition, statevec  # noqa: E402

    return generators, ir, partition, statevec


def tensor_arrays(circ):
    """(gate_type (d,3) int32, gate_param (d,) f64, n_qubits, n_gates) of one CircuitTensor."""
    d = len(circ.gates)
    gt = np.zeros((d, 3), dtype=np.int32)
    for i, g in enumerate(circ.gates):
        gt[i] = (int(g.kind), -1 if g.control is None else g.control, g.target)
    return gt, np.asarray(circ.params, dtype=np.float64), circ.n_qubits, circ.n_gates


def mixed_gates(ir, n, n_gates, seed, kinds=(0, 1, 2, 3, 4, 5)):
    """Seeded circuit over every executable kind, angles outside [0, 2pi) on purpose."""
    rng = np.random.default_rng(seed)
    GK, GR = ir.GateKind, ir.GateRecord
    out = []
    for _ in range(n_gates):
        k = int(rng.choice(kinds)) if n >= 2 else int(rng.choice([x for x in kinds if x < 4]))
        t = int(rng.integers(0, n))
        th = float(rng.uniform(-4 * math.pi, 4 * math.pi))
        if k in (4, 5):
            c = int(rng.integers(0, n - 1))
            c = c if c < t else c + 1
            out.append(GR.cx(c, t) if k == 4 else GR.cr1(c, t, th))
        elif k == 0:
            out.append(GR.h(t))
        else:
            out.append(GR(GK(k), None, t, th))
    return out


def main() -> None:
    generators, ir, partition, statevec = _ref()
    fx: dict[str, np.ndarray] = {}

    # ---- generators: bit-exact gate streams -------------------------------------------------
    rspecs = [(2, 5, 0, False), (5, 7, 3, True), (16, 100, 0, False), (32, 1000, 0, False),
              (32, 1000, 1, False), (36, 1000, 0, False), (37, 1000, 0, False), (20, 50, 7, True)]
    for n, b, s, m in rspecs:
        c = generators.generate_random_gate_list(generators.RandomSpec(n, b, s, m))
        gt, gp, _, ng = tensor_arrays(c)
        key = f"gen_random_{n}_{b}_{s}_{int(m)}"
        fx[key + "_type"], fx[key + "_param"] = gt, gp
    for n, rev in [(1, False), (6, False), (6, True), (28, False), (37, True)]:
        c = generators.build_qft(generators.QftSpec(n, rev))
        gt, gp, _, _ = tensor_arrays(c)
        key = f"gen_qft_{n}_{int(rev)}"
        fx[key + "_type"], fx[key + "_param"] = gt, gp
    fx["pairs_5_64_1"] = np.array(generators.random_qubit_pairs(5, 64, 1), dtype=np.int32)

    # ---- run_circuit states (exact mode) -----------------------------------------------------
    cases = []  # (name, n, gates-or-tensor)
    for i, (n, ng) in enumerate([(1, 12), (2, 40), (3, 60), (5, 120), (8, 200), (10, 300), (12, 400)]):
        cases.append((f"mixed{i}", n, ir.CircuitTensor.from_gates(ir.CircType.IMPORTED, n,
                                                                  mixed_gates(ir, n, ng, 100 + i))))
    cases.append(("random12", 12, generators.generate_random_gate_list(generators.RandomSpec(12, 200, 5))))
    cases.append(("random14m", 14, generators.generate_random_gate_list(generators.RandomSpec(14, 150, 9, True))))
    cases.append(("qft10", 10, generators.build_qft(generators.QftSpec(10))))
    cases.append(("qft11r", 11, generators.build_qft(generators.QftSpec(11, True))))
    names = []
    for name, n, circ in cases:
        names.append(name)
        gt, gp, nq, ng = tensor_arrays(circ)
        fx[f"state_{name}_type"], fx[f"state_{name}_param"] = gt, gp
        fx[f"state_{name}_hdr"] = np.array([nq, ng], dtype=np.int64)
        for prec in ("fp64", "fp32"):
            st, _ = statevec.run_circuit(circ, statevec.SimOptions(precision=prec))
            fx[f"state_{name}_{prec}"] = st.amplitudes
    fx["state_cases"] = np.array(names)

    # ---- config 1: RandomSpec(16,100,0), fp64, 3000 shots, seed 0 ----------------------------
    c1 = generators.generate_random_gate_list(generators.RandomSpec(16, 100, 0))
    st, counts = statevec.run_circuit(c1, statevec.SimOptions("fp64", 3000, 0))
    fx["cfg1_state_fp64"] = st.amplitudes
    keys = sorted(counts.counts, key=statevec.index_of_bitstring)
    fx["cfg1_count_index"] = np.array([statevec.index_of_bitstring(k) for k in keys], dtype=np.int64)
    fx["cfg1_count_value"] = np.array([counts.counts[k] for k in keys], dtype=np.int64)
    fx["cfg1_count_keys"] = np.array(keys)

    # ---- sample_counts on fixed states (pins the cumsum/searchsorted convention) -------------
    srng = np.random.default_rng(42)
    for j, (n, shots, seed) in enumerate([(3, 1000, 0), (6, 5000, 11), (10, 20000, 3), (1, 100000, 0)]):
        a = srng.normal(size=1 << n) + 1j * srng.normal(size=1 << n)
        a /= np.linalg.norm(a)
        if n == 1:
            a = np.array([1, 1], dtype=np.complex128) / math.sqrt(2.0)  # SPEC.md:239 H|0>
        sv = statevec.StateVector(n, "fp64", a.astype(np.complex128))
        ct = statevec.sample_counts(sv, shots, seed)
        ks = sorted(ct.counts, key=statevec.index_of_bitstring)
        fx[f"sample{j}_amps"] = a
        fx[f"sample{j}_meta"] = np.array([n, shots, seed], dtype=np.int64)
        fx[f"sample{j}_index"] = np.array([statevec.index_of_bitstring(k) for k in ks], dtype=np.int64)
        fx[f"sample{j}_value"] = np.array([ct.counts[k] for k in ks], dtype=np.int64)

    # ---- partitioned executor: plan localities, message counts, W-vs-1 equality -------------
    for j, (circ, w) in enumerate([
        (generators.generate_random_gate_list(generators.RandomSpec(10, 60, 2)), 4),
        (generators.build_qft(generators.QftSpec(8)), 2),
        (ir.CircuitTensor.from_gates(ir.CircType.IMPORTED, 6, mixed_gates(ir, 6, 80, 7)), 8),
    ]):
        res = partition.execute_distributed(circ, w, statevec.SimOptions("fp64", 2000, 5))
        gt, gp, nq, ng = tensor_arrays(circ)
        fx[f"part{j}_type"], fx[f"part{j}_param"] = gt, gp
        fx[f"part{j}_meta"] = np.array([nq, ng, w], dtype=np.int64)
        fx[f"part{j}_state"] = res.state.amplitudes
        fx[f"part{j}_sent"] = np.array(res.messages_sent, dtype=np.int64)
        fx[f"part{j}_recv"] = np.array(res.messages_received, dtype=np.int64)
        fx[f"part{j}_masks"] = np.array([t.partner_mask for t in res.tasks], dtype=np.int64)
        ks = sorted(res.counts.counts, key=statevec.index_of_bitstring)
        fx[f"part{j}_cidx"] = np.array([statevec.index_of_bitstring(k) for k in ks], dtype=np.int64)
        fx[f"part{j}_cval"] = np.array([res.counts.counts[k] for k in ks], dtype=np.int64)

    # ---- encode / set_to_arrays: CR1 canonicalisation, padding ------------------------------
    GR = ir.GateRecord
    lists = [
        (ir.CircType.IMPORTED, 3, [GR.h(0), GR.cr1(0, 2, -1.0), GR.cr1(2, 1, 7.5), GR.rz(1, -9.0)]),
        (ir.CircType.QFT, 2, [GR.cr1(1, 0, 2 * math.pi), GR.measure(0), GR.measure(1)]),
        (ir.CircType.RANDOM, 4, []),
    ]
    cs = ir.encode_circuits(lists)
    h, gt, gp = ir.set_to_arrays(cs)
    fx["enc_headers"], fx["enc_type"], fx["enc_param"] = h, gt, gp

    path = os.path.join(OUT, "golden.npz")
    np.savez_compressed(path, **fx)
    print(f"wrote {path}: {len(fx)} arrays, {os.path.getsize(path) / 2**20:.2f} MiB")


if __name__ == "__main__":
    main()
