"""Bench harness: CSV columns and round trip, scaling fit,
SVG determinism (CPU); run_suite on a small grid (GPU)."""

import io
import xml.dom.minidom

import pytest

from paper_2504_03967_b200 import bench_suite as bs


def _recs(times):
    return [bs.BenchRecord("random", n, 3 * 100, "fp64", 1, rep, t, 0) for (n, rep, t) in times]


def test_csv_columns_and_round_trip():
    recs = _recs([(10, 0, 1.5), (10, 1, 1.25), (11, 0, 3.0)])
    buf = io.StringIO()
    bs.write_csv(recs, buf)
    text = buf.getvalue()
    assert text.splitlines()[0] == "workload,n_qubits,gates,precision,workers,rep,wall_ms,seed"
    back = bs.read_csv(text)
    assert [(r.workload, r.n_qubits, r.gates, r.precision, r.workers, r.rep, r.wall_ms, r.seed) for r in back] == \
        [(r.workload, r.n_qubits, r.gates, r.precision, r.workers, r.rep, r.wall_ms, r.seed) for r in recs]


def test_fit_scaling():
    exact = _recs([(n, 0, 0.37 * 2.0 ** n) for n in range(12, 18)])
    f = bs.fit_scaling(exact)
    assert abs(f["slope"] - 1.0) <= 1e-9 and f["conformant"]
    const = _recs([(n, r, 5.0) for n in range(12, 18) for r in range(3)])
    f = bs.fit_scaling(const)
    assert abs(f["slope"]) < 1e-9 and not f["conformant"]
    with pytest.raises(bs.InsufficientDataError):
        bs.fit_scaling(_recs([(10, 0, 1.0), (11, 0, 2.0), (12, 0, 4.0)]))


def test_chart_is_deterministic_svg():
    recs = _recs([(n, 0, 2.0 ** n) for n in range(10, 14)]) + \
        [bs.BenchRecord("random", n, 300, "fp32", 2, 0, 2.0 ** (n - 1), 0) for n in range(10, 14)]
    a, b = bs.emit_chart(recs), bs.emit_chart(list(recs))
    assert a == b and a.count("<polyline") == 2
    xml.dom.minidom.parseString(a)
    assert bs.emit_chart(_recs([(10, 0, 1.0)])).count("<polyline") == 1
    with pytest.raises(ValueError):
        bs.emit_chart([])


def test_empty_spec():
    with pytest.raises(bs.EmptySpecError):
        bs.run_suite(bs.BenchSpec(qubits=(12, 11)))


@pytest.mark.gpu
def test_run_suite_grid(tmp_path):
    spec = bs.BenchSpec("random", (10, 13), 20, ("fp32", "fp64"), (1, 2), 0, 2, 0)
    recs = bs.run_suite(spec, str(tmp_path / "a.csv"), str(tmp_path / "b.csv"))
    assert len(recs) == 4 * 2 * 2 * 2 and all(r.wall_ms > 0 for r in recs)
    assert len(bs.read_csv(str(tmp_path / "a.csv"))) == len(recs)
    assert all(r.extra.get("passes", 0) >= 1 for r in recs if r.workers == 1)
