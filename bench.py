#!/usr/bin/env python
"""bench.py — BASELINE.json metric: circuit wall-time, gates/s and HBM GB/s for the
32-qubit random CX-block circuit (configs[2]: RandomSpec(32, 1000 blocks, seed 0),
complex64) on 1 B200, or sharded over N GPUs under torchrun (strong scaling:
one circuit, N shards, qubit remaps over NCCL).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full circuit: |0..0> init of the (sharded) state in HBM + every
fused pass (+ remaps).  Device time per step is taken with CUDA events on the
launching stream, max over ranks.  The state (32 GiB) is far larger than L2
(126 MB), so no L2 flush is needed between steps.

e2e = the same circuit through the public API paper_2504_03967_b200.statevec.
run_circuit (host gate records -> planning -> JIT pass kernels (process-wide
cubin cache) -> execution -> per-shot sampler, --e2e-shots shots) with the (index,
count) pairs read back to the host.

--impl reference: the reference's own CPU executor from baseline/_ref (its
threaded partition.execute_distributed, the fastest CPU path it has for this
circuit), rank 0 only: a warm-up ladder n = 23..26 fixes the 2^n slope of the
per-gate time; each timed step is one bounded sample at 25 qubits scaled to 32.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIST_BACKEND = os.environ.get("QG_DIST_BACKEND", "nccl")  # "gloo": multi-rank test mode on one GPU
NVL_PEAK_GBS = 770.0  # B200_PROFILING.md: measured peer copy per direction per GPU
METRIC = "circuit wall-time, gates/s & HBM GB/s, 32q random-CX at 1/2/4/8 B200"


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# ----------------------------------------------------------------------------- CPU baseline
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _ref_modules():
    """The reference package itself (installed into baseline/_ref), else the oracle port."""
    if os.path.isdir(os.path.join(REF_DIR, "qgear")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        from qgear import generators as rg, partition as rp, statevec as rs  # noqa: E402

        return "reference", rg, rs, rp
    import oracle  # test infrastructure: the CPU restatement, used only as the baseline arm

    return "port", oracle, None, None


def _threads() -> int:
    c = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    w = 1
    while w * 2 <= min(8, c):
        w *= 2
    return w


def ref_sec_per_gate(n: int, blocks: int, seed: int = 0) -> tuple[float, int, str]:
    """Wall seconds per gate of the reference CPU executor on RandomSpec(n, blocks, seed).

    The reference's fastest CPU path for this circuit is its threaded partitioned
    executor (partition.execute_distributed, W = min(8, cores) worker threads; fp64
    only, partition.py:300-301) -- faster than the single-threaded fp32
    statevec.run_circuit from 22 qubits up (measured in this container: 22 q x 30
    gates 1.50 s vs 2.31 s)."""
    kind, rg, rs, rp = _ref_modules()
    if kind == "reference":
        circ = rg.generate_random_gate_list(rg.RandomSpec(n, blocks, seed))
        w = _threads()
        t0 = time.perf_counter()
        rp.execute_distributed(circ, w, rs.SimOptions(precision="fp64", memory_budget=1 << 40))
        dt = time.perf_counter() - t0
        return dt / (3 * blocks), w, "partition.execute_distributed(fp64, %d threads)" % w
    from paper_2504_03967_b200.generators import RandomSpec, random_arrays

    gt, gp = random_arrays(RandomSpec(n, blocks, seed))
    t0 = time.perf_counter()
    rg.run_arrays(gt, gp, n, gt.shape[0], "fp32")
    return (time.perf_counter() - t0) / gt.shape[0], 1, "oracle port of statevec.run_circuit (fp32, 1 thread)"


def ref_ladder(ladder=(20, 21, 22, 23, 24), blocks: int = 10) -> dict:
    """Per-gate time at n = ladder, fitted log2(t) = a + b n (the 2^n cost of a
    state-vector gate); the fit extrapolates to sizes the host cannot hold."""
    pts = []
    for n in ladder:
        spg, w, how = ref_sec_per_gate(n, blocks)
        pts.append((n, spg))
    x = np.array([p[0] for p in pts], dtype=float)
    y = np.log2(np.array([p[1] for p in pts]))
    b, a = np.polyfit(x, y, 1)
    return {"points_sec_per_gate": [[int(n), float(s)] for n, s in pts], "fit_log2": [float(a), float(b)],
            "blocks": blocks, "threads": w, "how": how}


def ref_rate(fit: dict, n_target: int, sample_n: int, blocks: int) -> tuple[float, float]:
    """One bounded sample at sample_n, scaled to n_target with the fitted slope."""
    spg, _, _ = ref_sec_per_gate(sample_n, blocks)
    b = fit["fit_log2"][1]
    spg_target = spg * 2.0 ** (b * (n_target - sample_n))
    return 1.0 / spg_target, spg


def ref_c1_ms() -> float | None:
    """BASELINE configs[0] run directly: RandomSpec(16, 100, 0), complex128, 3000 shots."""
    kind, rg, rs, _ = _ref_modules()
    if kind != "reference":
        return None
    circ = rg.generate_random_gate_list(rg.RandomSpec(16, 100, 0))
    best = 1e30
    for _ in range(3):
        t0 = time.perf_counter()
        rs.run_circuit(circ, rs.SimOptions(precision="fp64", shots=3000, rng_seed=0))
        best = min(best, time.perf_counter() - t0)
    return best * 1000.0


def _ladder(s: str) -> tuple:
    return tuple(int(x) for x in s.split(","))


def cpu_baseline_entry(n_target: int, sample_n: int, blocks: int, ladder: str, steps: int = 1) -> dict:
    fit = ref_ladder(_ladder(ladder), blocks)
    vals = [ref_rate(fit, n_target, sample_n, blocks)[0] for _ in range(steps)]
    kind = _ref_modules()[0]
    return {"value": float(np.mean(vals)), "unit": "gates/s", "cores": fit["threads"], "kind": kind,
            "sample": (f"{fit['how']} on RandomSpec(n, {blocks} blocks, seed 0), n = {ladder}; "
                       f"log2(sec/gate) fitted linear in n (slope {fit['fit_log2'][1]:.3f}) and extrapolated from "
                       f"the n = {sample_n} sample to {n_target} qubits (the host cannot hold a {n_target}-qubit state)"),
            "ladder": fit, "steps_values": vals, "c1_ms": ref_c1_ms(), "host": host_info()}


def host_info() -> dict:
    """The host the CPU arm ran on (cpu_count, affinity, CPU model)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)), "model": model,
            "threads": "the reference's threaded executor partition.execute_distributed (fp64 only, "
                       "partition.py:300-301) with min(8, cores) worker threads"}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank: int):
    """The reference's own CPU executor (baseline/_ref), rank 0 only, all host threads
    it can use.  Warm-up = the n ladder that fixes the 2^n slope (once); each timed
    step = one bounded sample at --ref-sample-qubits scaled to --qubits."""
    if rank != 0:
        return
    steps = args.steps
    fit = ref_ladder(_ladder(args.ref_ladder), args.ref_sample_blocks)
    vals, spgs = [], []
    for _ in range(steps):
        v, spg = ref_rate(fit, args.qubits, args.ref_sample_qubits, args.ref_sample_blocks)
        vals.append(v)
        spgs.append(spg)
    value = float(np.mean(vals))
    kind = _ref_modules()[0]
    sample = (f"{fit['how']} on RandomSpec({args.ref_sample_qubits}, {args.ref_sample_blocks} blocks, seed 0) "
              f"per step; sec/gate scaled to {args.qubits} qubits by the slope of log2(sec/gate) fitted over "
              f"n = {args.ref_ladder} (warm-up ladder)")
    ms_per_step = 3 * args.blocks / value * 1000.0
    out = {"metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": args.gpus, "steps": steps,
           "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "c128" if kind == "reference" else "c64",
           "data": "synthetic (reference generator stream, PCG64 seed 0)", "impl": "reference",
           "config": {"workload": f"random CX-block, {args.qubits} qubits, {args.blocks} blocks "
                                  f"(extrapolated from fit over n={args.ref_ladder})",
                      "n_qubits": args.qubits, "blocks": args.blocks, "gates": 3 * args.blocks},
           "cpu_baseline": {"value": value, "unit": "gates/s", "cores": fit["threads"], "kind": kind,
                            "sample": sample, "ladder": fit, "sample_sec_per_gate": spgs,
                            "c1_ms": ref_c1_ms(), "host": host_info()},
           "e2e": {"value": value, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------------------- our arm
def run_ours(args, rank: int, world: int, local_rank: int):
    import ctypes as C

    import torch

    from paper_2504_03967_b200 import partition as pt
    from paper_2504_03967_b200 import statevec as sv
    from paper_2504_03967_b200.generators import (QftSpec, RandomSpec, build_qft, generate_random_gate_list,
                                                   qft_arrays, random_arrays)

    # QG_DIST_BACKEND=gloo (a test mode): ranks may share a GPU, collectives go through host memory
    dev_index = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    gloo = DIST_BACKEND == "gloo"

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device="cpu" if gloo else dev)
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()
    dist = None
    if world > 1:
        import torch.distributed as dist_mod

        dist = dist_mod
    n, prec = args.qubits, args.precision
    g = world.bit_length() - 1
    qft = args.circuit == "qft"  # BASELINE configs[1] (C2): QFT on n qubits, build_qft's gate order
    gt, gp = qft_arrays(n) if qft else random_arrays(RandomSpec(n, args.blocks, args.seed))
    # circuit-specialised pass kernels for every shard size (complex64), compiled before the
    # warm-up so that every timed step runs them (at N > 1 the auto policy would tier up in the
    # background); later plans of the same circuit (the e2e leg) hit the process cubin cache
    plan = sv.CompiledCircuit(gt, gp, n, prec, g, tile_qubits=args.tile_qubits, max_stages=args.max_stages,
                              max_cost=args.max_cost, jit=1 if prec == "fp32" else 0)
    jit_info = plan.jit_status(wait=True)
    n_local = plan.n_local
    amp_bytes = 8 if prec == "fp32" else 16
    shard_bytes = (1 << n_local) * amp_bytes
    shard = torch.empty(1 << n_local, dtype=sv._DTYPES[prec], device=dev)
    stream = torch.cuda.current_stream(dev)
    staging = None

    remap_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(plan.n_segments - 1)]
    remap_egress = [shard_bytes * ((1 << len(g_)) - 1) // (1 << len(g_)) for g_, _ in plan.remaps]

    def step(timed_passes: bool, timed_remaps: bool = False):
        sv.N.call("qg_state_init_zero", C.c_void_p(shard.data_ptr()), n_local, sv._QG_DTYPE[prec], rank,
                  C.c_void_p(stream.cuda_stream))
        pms, launches = 0.0, 0
        for seg in range(plan.n_segments):
            st = plan.execute_segment(seg, shard, rank, timed=timed_passes)
            pms += st.pass_ms
            launches += st.pass_launches
            if seg < plan.n_segments - 1:
                gpos, lpos = plan.remaps[seg]
                if timed_remaps:
                    remap_ev[seg][0].record(stream)
                pt.remap_dist(shard, n_local, gpos, lpos, rank, None, staging)
                if timed_remaps:
                    remap_ev[seg][1].record(stream)
        return pms, launches

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step(False)
    barrier()
    clocks = ClockSampler(dev_index) if rank == 0 else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step(False)
    e1.record(stream)
    barrier()
    total_ms = e0.elapsed_time(e1)
    # pass-kernel time on the launching stream (library CUDA events), same steps again;
    # each remap bracketed by CUDA events on the same stream (NCCL waits on it, and it
    # waits on NCCL before the copy-back)
    pass_ms, launches, remap_ms = 0.0, 0, []
    for _ in range(args.steps):
        pm, ln = step(True, True)
        pass_ms += pm
        launches += ln
        torch.cuda.synchronize(dev)
        remap_ms.append([a.elapsed_time(b) for a, b in remap_ev])
    barrier()
    clock_info = clocks.stop() if clocks else None
    remap_tot = float(np.sum(remap_ms)) / max(1, args.steps)  # per step, this rank
    total_ms, pass_ms, remap_tot = max_over_ranks([total_ms, pass_ms, remap_tot])
    ms_per_step = total_ms / args.steps
    gates = gt.shape[0]
    value = gates / (ms_per_step / 1000.0)

    # ---- e2e through the public API (host gate tensor -> plan -> kernels -> norm to host)
    e2e = None
    if not args.no_e2e:
        opts = sv.SimOptions(precision=prec, shots=args.e2e_shots, rng_seed=args.seed, memory_budget=1 << 45,
                             device=dev_index, tile_qubits=args.tile_qubits, max_stages=args.max_stages,
                             max_cost=args.max_cost)
        circ = build_qft(QftSpec(n)) if qft else generate_random_gate_list(RandomSpec(n, args.blocks, args.seed))
        del shard
        torch.cuda.empty_cache()

        def e2e_step():
            # host gate records in -> plan (+ JIT, cubins from the process-wide cache after the
            # warm-up call) -> passes (+ remaps) -> sampler -> counts on the host
            if world > 1:
                res = pt.execute_distributed(circ, world, opts, gather=False)
            else:
                _, counts = sv.run_circuit(circ, opts)
                res = type("R", (), {"counts": counts})
            c = res.counts
            return 16 * (len(c.indices) if c is not None else 0) + 16  # (index, count) pairs + mass/nunique

        e2e_step()
        barrier()
        w0 = time.perf_counter()
        for _ in range(max(1, args.e2e_steps)):
            d2h = e2e_step()
        barrier()
        e2e_ms = (time.perf_counter() - w0) * 1000.0 / max(1, args.e2e_steps)
        e2e_ms = max_over_ranks([e2e_ms])[0]
        e2e = {"value": gates / (e2e_ms / 1000.0), "unit": "gates/s",
               "h2d_bytes_per_step": int(plan.info["param_bytes"] + gt.nbytes + gp.nbytes),
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
               "shots": args.e2e_shots,
               "note": ("host gate records -> plan + JIT (cubin cache warm after one warm-up call) -> kernels "
                        "-> sampler (Philox, per shot); (index, count) pairs of the shots read back to the host; the state "
                        "stays in HBM")}

    if rank != 0:
        return
    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    peak = peaks.get("hbm_gbs", 6650.0)
    avg_launch_ms = pass_ms / max(1, launches)
    achieved = 2.0 * shard_bytes / (avg_launch_ms / 1000.0) / 1e9
    prof = load_json(os.path.join(ROOT, "profiles", "fused_pass_traffic.json")) or {}
    traffic = prof.get(f"{n_local}q_{prec}", {}).get("dram_bytes_per_launch")
    cpu = None
    if not args.no_cpu_baseline and world == 1 and not qft:
        cpu = cpu_baseline_entry(n, args.cpu_sample_qubits, args.cpu_sample_blocks, args.ref_ladder)
    out = {
        "metric": METRIC, "value": value, "unit": "gates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c64" if prec == "fp32" else "c128",
        "data": (f"synthetic: build_qft(QftSpec({n})) gate order, state |0..0>" if qft else
                 f"synthetic: reference generator stream RandomSpec({n}, {args.blocks}, seed {args.seed}) (PCG64), "
                 "state |0..0>"),
        "config": {"workload": (f"QFT, {n} qubits" if qft else
                                f"random CX-block circuit, {n} qubits, {args.blocks} blocks") +
                               f", {'complex64' if prec == 'fp32' else 'complex128'}, {world} GPU(s)",
                   "n_qubits": n, "blocks": None if qft else args.blocks, "gates": int(gates), "seed": args.seed,
                   "fused_passes": int(plan.info["n_passes"]), "remaps": int(plan.info["n_remaps"]),
                   "tile_qubits": int(plan.info["tile_qubits"]), "shard_bytes": shard_bytes,
                   "jit_passes": int(jit_info["n_jit"]), "jit_compile_ms_wall": jit_info["compile_ms_wall"],
                   "l2": "no flush needed: state >> 126 MB L2",
                   "parallelism": f"sv-shard{world}" if world > 1 else "single",
                   **({"dist_backend": DIST_BACKEND} if world > 1 else {})},
        "hbm_gbs_step": 2.0 * shard_bytes * plan.info["n_passes"] / (ms_per_step / 1000.0) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "qg_jit_pass (circuit-specialised fused pass)" if jit_info["n_jit"] else "fused_pass_kernel",
                     "peak_source": "MEASURED_PEAKS.json:hbm_gbs (measured copy)" if "hbm_gbs" in peaks
                     else "fallback 6.65 TB/s (B200_PROFILING.md)",
                     "algorithmic_bytes_per_launch": 2 * shard_bytes, "avg_launch_ms": avg_launch_ms},
        "roofline_nvl": None if not plan.remaps else {
            "bound": "nvlink" if DIST_BACKEND == "nccl" else f"{DIST_BACKEND} host staging (test mode)",
            "achieved": sum(remap_egress) / (remap_tot / 1000.0) / 1e9,
            "peak": NVL_PEAK_GBS, "unit": "GB/s",
            "frac": sum(remap_egress) / (remap_tot / 1000.0) / 1e9 / NVL_PEAK_GBS,
            "peak_source": "B200_PROFILING.md: measured peer copy 770 GB/s per direction (900 nominal)",
            "egress_bytes_per_step_per_rank": int(sum(remap_egress)), "remap_ms_per_step": remap_tot,
            "remaps": len(plan.remaps),
            "per_remap": [{"s": len(g_), "egress_bytes": int(e_), "ms": float(np.mean([r[i] for r in remap_ms])),
                           "gbs": e_ / (float(np.mean([r[i] for r in remap_ms])) / 1000.0) / 1e9}
                          for i, ((g_, _), e_) in enumerate(zip(plan.remaps, remap_egress))]},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int((plan.info["n_passes"] + 1) * args.steps),
        "clocks": clock_info,
    }
    print(json.dumps(out), flush=True)


def relaunch(n: int) -> int:
    """`bench.py --gpus N` without torchrun: start N ranks (one per GPU) under
    torch.distributed.run on this node, or fail if the node has fewer GPUs."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py: --gpus {n} requested but this node has {have} CUDA device(s)", file=sys.stderr)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the init log shows the communicator's rank count
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--qubits", type=int, default=32)
    ap.add_argument("--blocks", type=int, default=1000)
    ap.add_argument("--circuit", choices=["random", "qft"], default="random")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--tile-qubits", type=int, default=0)
    ap.add_argument("--max-stages", type=int, default=0)
    ap.add_argument("--max-cost", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--e2e-shots", type=int, default=100_000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-qubits", type=int, default=25)
    ap.add_argument("--cpu-sample-blocks", type=int, default=10)
    ap.add_argument("--ref-sample-qubits", type=int, default=25)
    ap.add_argument("--ref-ladder", default="23,24,25,26")
    ap.add_argument("--ref-sample-blocks", type=int, default=10)
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args.gpus))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to report a different GPU count",
              file=sys.stderr)
        sys.exit(2)
    if world > 1:
        import torch
        import torch.distributed as dist

        if DIST_BACKEND == "nccl":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(DIST_BACKEND)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
