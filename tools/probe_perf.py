"""Quick device timing of run paths (development probe, not the bench contract)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2504_03967_b200 import statevec as sv
from paper_2504_03967_b200.generators import RandomSpec, random_arrays, qft_arrays

def time_plan(name, gt, gp, n, prec, reps=3, **kw):
    plan = sv.CompiledCircuit(gt, gp, n, prec, **kw)
    st = sv.init_zero_state(n, prec, 1 << 40)
    plan.execute(st)  # warm
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s = plan.execute(st, timed=True)
        best = min(best, s.pass_ms)
    S = (1 << n) * (8 if prec == "fp32" else 16)
    passes = plan.info["n_passes"]
    gbs = 2 * S * passes / (best / 1e3) / 1e9
    print(json.dumps(dict(name=name, n=n, prec=prec, passes=passes, stages=plan.info["n_stages"], ms=round(best, 3),
                          ms_per_pass=round(best / passes, 4), gbs=round(gbs, 1), gates_per_s=round(gt.shape[0] / best * 1e3), kw=kw)), flush=True)
    del st

n_list = [int(x) for x in sys.argv[1:]] or [28, 30, 32]
for n in n_list:
    gt, gp = random_arrays(RandomSpec(n, 1000, 0))
    time_plan("random", gt, gp, n, "fp32")
    if n <= 31:
        time_plan("random", gt, gp, n, "fp64")
    gt, gp = qft_arrays(n)
    time_plan("qft", gt, gp, n, "fp32")
gt, gp = random_arrays(RandomSpec(28, 1000, 0))
for kw in [dict(max_stages=1), dict(max_stages=2), dict(max_cost=60), dict(max_cost=150), dict(max_stages=6, max_cost=200), dict(tile_qubits=12), dict(tile_qubits=11)]:
    time_plan("random", gt, gp, 28, "fp32", **kw)
time_plan("random-unfused", gt[:300], gp[:300], 28, "fp32", fuse=False)
