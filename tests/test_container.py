"""QGIR1 container ingest: the native parser / writer against
files written by the reference's own container.write_binary
(tests/golden/make_golden_qgir.py), plus the reference's error cases."""

import json
import os

import numpy as np
import pytest

from paper_2504_03967_b200 import container
from paper_2504_03967_b200.errors import ContainerFormatError
from paper_2504_03967_b200.ir import set_to_arrays
from paper_2504_03967_b200.statevec import CompiledCircuit

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "qgir")


def expected():
    with np.load(os.path.join(HERE, "expected.npz")) as z:
        d = {k: z[k] for k in z.files}
    d["meta"] = json.loads(str(d.pop("metadata_json")))
    return d


@pytest.mark.parametrize("i", [0, 1, 2])
def test_reads_reference_files_zero_copy(i):
    exp = expected()
    path = os.path.join(HERE, f"set{i}.qgir")
    h, g, p, meta = container.read_arrays(path)
    assert np.array_equal(h, exp[f"set{i}_headers"])
    assert np.array_equal(g, exp[f"set{i}_gate_type"])
    assert np.array_equal(p, exp[f"set{i}_gate_param"])
    assert meta == exp["meta"][f"set{i}"]
    assert not g.flags.owndata  # a view of the mapped file, not a copy


@pytest.mark.parametrize("i", [0, 1, 2])
def test_round_trip_is_byte_identical(i, tmp_path):
    path = os.path.join(HERE, f"set{i}.qgir")
    cs = container.read_binary(path)
    out = tmp_path / "x.qgir"
    container.write_binary(cs, out)
    assert out.read_bytes() == open(path, "rb").read()
    assert container.load_circuit_set(out) == cs
    h, g, p = set_to_arrays(cs)
    assert np.array_equal(g, expected()[f"set{i}_gate_type"])


def test_error_cases(tmp_path):
    good = open(os.path.join(HERE, "set1.qgir"), "rb").read()
    cases = {
        "bad magic": b"QGIR2" + good[5:],
        "truncated": good[:-3],
        "trailing": good + b"\0",
        "short": b"QGI",
        "header only": good[:17],
    }
    for name, blob in cases.items():
        f = tmp_path / f"{name.replace(' ', '_')}.qgir"
        f.write_bytes(blob)
        with pytest.raises(ContainerFormatError):
            container.read_binary(f)
    with pytest.raises(ContainerFormatError):
        container.load_circuit_set(tmp_path / "bad_magic.qgir")
    (tmp_path / "x.h5").write_bytes(b"\x89HDF\r\n\x1a\n")
    with pytest.raises(ContainerFormatError):
        container.load_circuit_set(tmp_path / "x.h5")


def test_mapped_arrays_feed_the_planner():
    h, g, p, _ = container.read_arrays(os.path.join(HERE, "set1.qgir"))
    for c in range(h.shape[0]):
        ng, n = int(h[c, 2]), int(h[c, 1])
        plan = CompiledCircuit(g[c, :ng], p[c, :ng], n, "fp64")
        assert plan.info["n_body_gates"] <= ng
