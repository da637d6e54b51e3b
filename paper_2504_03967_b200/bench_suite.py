"""Benchmark harness of SPEC.md:519-586 ("bench-cli") over the B200 executor.

run_suite(spec) times run_circuit / execute_distributed only (generation and I/O
excluded) for every (workload, n, precision, workers, rep) grid point and writes
the CSV with exactly the SPEC's columns
    workload,n_qubits,gates,precision,workers,rep,wall_ms,seed
plus, in a second CSV (``extended=True``), the B200 columns: fused passes, HBM
bytes moved and GB/s, fraction of the measured HBM peak.  fit_scaling is the
SPEC's log2(median time) vs n slope; emit_chart the SVG
(SPEC.md:549-555).

    python -m paper_2504_03967_b200.bench_suite --workload random --qubits 20..24 \
        --blocks 100 --precision fp32,fp64 --workers 1 --reps 3 --seed 0 --csv out.csv [--svg out.svg]
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import math
import os
import sys
import time
from dataclasses import dataclass, field

import numpy as np

CSV_COLUMNS = ["workload", "n_qubits", "gates", "precision", "workers", "rep", "wall_ms", "seed"]
EXT_COLUMNS = CSV_COLUMNS + ["passes", "hbm_bytes", "hbm_gbs", "hbm_frac"]


class EmptySpecError(ValueError):
    """empty qubit range."""


class InsufficientDataError(ValueError):
    """fewer than 4 distinct n."""


@dataclass
class BenchSpec:
    workload: str = "random"                 # random | qft | qcrank
    qubits: tuple = (10, 14)                 # inclusive range
    blocks: int = 100
    precisions: tuple = ("fp64",)
    workers: tuple = (1,)
    shots: int = 0
    reps: int = 3
    seed: int = 0
    n_data: int = 2                          # qcrank: data qubits (address qubits = n - n_data)


@dataclass
class BenchRecord:
    workload: str
    n_qubits: int
    gates: int
    precision: str
    workers: int
    rep: int
    wall_ms: float
    seed: int
    extra: dict = field(default_factory=dict)

    def row(self, extended: bool = False) -> list:
        r = [self.workload, self.n_qubits, self.gates, self.precision, self.workers, self.rep,
             f"{self.wall_ms:.6f}", self.seed]
        if extended:
            r += [self.extra.get(k, "") for k in EXT_COLUMNS[len(CSV_COLUMNS):]]
        return r


def _circuit(spec: BenchSpec, n: int):
    from .generators import QftSpec, RandomSpec, build_qft, generate_random_gate_list

    if spec.workload == "random":
        return generate_random_gate_list(RandomSpec(n, spec.blocks, spec.seed))
    if spec.workload == "qft":
        return build_qft(QftSpec(n))
    if spec.workload == "qcrank":
        from . import qcrank
        from .ir import CircType, CircuitTensor

        m = n - spec.n_data
        rng = np.random.default_rng(spec.seed)
        px = rng.integers(0, 256, size=(1 << m) * spec.n_data, dtype=np.uint8)
        img = qcrank.ImageGray(px.size, 1, px)
        ang = qcrank.prepare_angles(img, m, spec.n_data)
        gt, gp, nq = qcrank.build_qcrank_circuit(ang, measure=False)
        return CircuitTensor.from_arrays(CircType.IMPORTED, nq, gt, gp)
    raise ValueError(f"unknown workload {spec.workload!r}")


def _peak_gbs() -> float:
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


def run_suite(spec: BenchSpec, csv_path: str | None = None, extended_csv: str | None = None,
              clock=time.perf_counter) -> list[BenchRecord]:
    """SPEC.md:535-540.  Each grid point: generate (untimed), run (timed with
    `clock`, after a device synchronize on both sides), repeat `reps` times.
    Rows already measured are flushed to the CSV before an error propagates."""
    import torch

    from . import partition as pt
    from . import statevec as sv

    lo, hi = spec.qubits
    if hi < lo:
        raise EmptySpecError(f"empty qubit range {lo}..{hi}")
    recs: list[BenchRecord] = []
    peak = _peak_gbs()
    try:
        for n in range(lo, hi + 1):
            circ = _circuit(spec, n)
            gates = int(circ.n_gates) if hasattr(circ, "n_gates") else len(list(circ.active_gates))
            for prec in spec.precisions:
                for w in spec.workers:
                    opts = sv.SimOptions(precision=prec, shots=spec.shots, rng_seed=spec.seed,
                                         memory_budget=1 << 45)
                    passes = None
                    if w == 1 and spec.workload != "qcrank":  # the pass count the timed call runs
                        passes = int(sv.compile_circuit(circ, opts).info["n_passes"])
                    for rep in range(spec.reps):
                        torch.cuda.synchronize()
                        t0 = clock()
                        if w == 1:
                            st, _ = sv.run_circuit(circ, opts)
                        else:
                            st = pt.execute_distributed(circ, w, opts).state
                        torch.cuda.synchronize()
                        ms = (clock() - t0) * 1000.0
                        extra = {}
                        if passes is not None:
                            byts = 2 * (1 << n) * (8 if prec == "fp32" else 16) * passes
                            gbs = byts / (ms / 1000.0) / 1e9
                            extra = {"passes": passes, "hbm_bytes": byts, "hbm_gbs": f"{gbs:.1f}",
                                     "hbm_frac": f"{gbs / peak:.4f}"}
                        recs.append(BenchRecord(spec.workload, n, gates, prec, w, rep, ms, spec.seed, extra))
                        del st
    finally:
        if csv_path:
            write_csv(recs, csv_path)
        if extended_csv:
            write_csv(recs, extended_csv, extended=True)
    return recs


def write_csv(recs: list[BenchRecord], path_or_buf, extended: bool = False) -> None:
    own = isinstance(path_or_buf, str)
    f = open(path_or_buf, "w", newline="") if own else path_or_buf
    try:
        w = csv.writer(f)
        w.writerow(EXT_COLUMNS if extended else CSV_COLUMNS)
        for r in recs:
            w.writerow(r.row(extended))
    finally:
        if own:
            f.close()


def read_csv(path_or_text: str) -> list[BenchRecord]:
    text = open(path_or_text).read() if os.path.exists(path_or_text) else path_or_text
    rows = list(csv.reader(io.StringIO(text)))
    if not rows or rows[0][: len(CSV_COLUMNS)] != CSV_COLUMNS:
        raise ValueError("not a bench CSV")
    out = []
    for r in rows[1:]:
        out.append(BenchRecord(r[0], int(r[1]), int(r[2]), r[3], int(r[4]), int(r[5]), float(r[6]), int(r[7])))
    return out


def fit_scaling(recs: list[BenchRecord]) -> dict:
    """least-squares slope of log2(median wall time) against n."""
    by_n: dict[int, list[float]] = {}
    for r in recs:
        by_n.setdefault(r.n_qubits, []).append(r.wall_ms)
    if len(by_n) < 4:
        raise InsufficientDataError(f"{len(by_n)} distinct n values (need >= 4)")
    ns = np.array(sorted(by_n), dtype=float)
    med = np.array([np.median(by_n[int(n)]) for n in ns])
    slope, icpt = np.polyfit(ns, np.log2(med), 1)
    return {"slope": float(slope), "intercept": float(icpt), "n": ns.astype(int).tolist(),
            "median_ms": med.tolist(), "conformant": bool(0.8 <= slope <= 1.3)}


def emit_chart(recs: list[BenchRecord], path: str | None = None) -> str:
    """SVG, time vs n on a log2 y axis, one polyline per
    (precision, workers) series; deterministic for identical input."""
    if not recs:
        raise ValueError("EmptyInput: no records")
    series: dict[str, dict[int, list[float]]] = {}
    for r in recs:
        series.setdefault(f"{r.precision} w{r.workers}", {}).setdefault(r.n_qubits, []).append(r.wall_ms)
    ns = sorted({r.n_qubits for r in recs})
    ys = [math.log2(max(r.wall_ms, 1e-9)) for r in recs]
    y0, y1 = min(ys), max(ys)
    y1 = y1 if y1 > y0 else y0 + 1
    x0, x1 = ns[0], ns[-1] if ns[-1] > ns[0] else ns[0] + 1
    W, H, M = 640, 400, 50
    colors = ["#1f77b4", "#d62728", "#2ca02c", "#9467bd", "#ff7f0e", "#8c564b"]

    def px(n, ms):
        x = M + (n - x0) / (x1 - x0) * (W - 2 * M)
        y = H - M - (math.log2(max(ms, 1e-9)) - y0) / (y1 - y0) * (H - 2 * M)
        return f"{x:.2f},{y:.2f}"

    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{H}">',
           f'<text x="{W / 2:.0f}" y="20" text-anchor="middle">wall time (ms, log2) vs qubits</text>']
    for i, key in enumerate(sorted(series)):
        pts = " ".join(px(n, float(np.median(v))) for n, v in sorted(series[key].items()))
        c = colors[i % len(colors)]
        out.append(f'<polyline fill="none" stroke="{c}" points="{pts}"/>')
        out.append(f'<text x="{W - M}" y="{M + 16 * i}" fill="{c}" text-anchor="end">{key}</text>')
    out.append("</svg>")
    svg = "\n".join(out) + "\n"
    if path:
        with open(path, "w") as f:
            f.write(svg)
    return svg


def _range(s: str) -> tuple:
    a, _, b = s.partition("..")
    return (int(a), int(b or a))


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="bench")
    ap.add_argument("--workload", default="random", choices=["random", "qft", "qcrank"])
    ap.add_argument("--qubits", default="10..14")
    ap.add_argument("--blocks", type=int, default=100)
    ap.add_argument("--precision", default="fp64")
    ap.add_argument("--workers", default="1")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--shots", type=int, default=0)
    ap.add_argument("--csv", default=None)
    ap.add_argument("--ext-csv", default=None)
    ap.add_argument("--svg", default=None)
    ap.add_argument("--check-scaling", action="store_true")
    a = ap.parse_args(argv)
    spec = BenchSpec(a.workload, _range(a.qubits), a.blocks, tuple(a.precision.split(",")),
                     tuple(int(w) for w in a.workers.split(",")), a.shots, a.reps, a.seed)
    recs = run_suite(spec, a.csv, a.ext_csv)
    if a.csv is None:
        write_csv(recs, sys.stdout)
    if a.svg:
        emit_chart(recs, a.svg)
    if a.check_scaling:
        fit = fit_scaling(recs)
        print(json.dumps(fit), file=sys.stderr)
        if not fit["conformant"]:
            return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
