"""Generate QGIR1 container fixtures from the REFERENCE's own writer.

Run once in the dev container (the only place /root/reference exists):

    python tests/golden/make_golden_qgir.py

Imports /root/reference/pkg/src/qgear/container.py with a stub `h5py` module
(h5py is not installed; only the QGIR1 binary path is exercised) and writes:
  tests/golden/qgir/set{0,1,2}.qgir  reference write_binary  (container.py:71-84)
  tests/golden/qgir/expected.npz     the reference read_binary -> set_to_arrays
                                     arrays and metadata of each file
Reference entry points: container.write_binary / read_binary container.py:71-115,
ir.encode_circuits / set_to_arrays ir.py:219-303, generators.py:61-101.
"""

from __future__ import annotations

import json
import os
import sys
import types

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "qgir")


def main():
    sys.modules.setdefault("h5py", types.ModuleType("h5py"))
    sys.path.insert(0, REF_SRC)
    from qgear import container, generators, ir

    os.makedirs(OUT, exist_ok=True)
    sets = [ir.encode_circuits([(ir.CircType.RANDOM, 6, list(
        generators.generate_random_gate_list(generators.RandomSpec(6, 10, 3)).active_gates))])]
    # a richer set: random (with trailing measures), QFT, reversed QFT, with metadata
    r1 = list(generators.generate_random_gate_list(generators.RandomSpec(5, 7, 1, include_measure=True)).active_gates)
    q1 = list(generators.build_qft(generators.QftSpec(4)).active_gates)
    q2 = list(generators.build_qft(generators.QftSpec(3, reversed=True)).active_gates)
    sets.append(ir.encode_circuits([(ir.CircType.RANDOM, 5, r1), (ir.CircType.QFT, 4, q1), (ir.CircType.QFT, 3, q2)],
                                   metadata={"source": "make_golden_qgir", "note": "unicode é✓"}))
    sets.append(ir.encode_circuits([(ir.CircType.QFT, 2, list(generators.build_qft(generators.QftSpec(2)).active_gates))]))
    expected = {}
    meta = {}
    for i, cs in enumerate(sets):
        path = os.path.join(OUT, f"set{i}.qgir")
        container.write_binary(cs, path)
        back = container.read_binary(path)
        h, g, p = ir.set_to_arrays(back)
        expected[f"set{i}_headers"] = h
        expected[f"set{i}_gate_type"] = g
        expected[f"set{i}_gate_param"] = p
        meta[f"set{i}"] = back.metadata
    expected["metadata_json"] = np.array(json.dumps(meta, sort_keys=True))
    np.savez(os.path.join(OUT, "expected.npz"), **expected)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
