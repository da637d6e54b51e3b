"""Time fused-kernel configurations against each other (development probe)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2504_03967_b200 import statevec as sv
from paper_2504_03967_b200.generators import RandomSpec, random_arrays, qft_arrays


def run(gt, gp, n, prec, reps=2, **kw):
    plan = sv.CompiledCircuit(gt, gp, n, prec, **kw)
    st = sv.init_zero_state(n, prec, 1 << 40)
    plan.execute(st)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        sv._init_into(st) if hasattr(sv, "_init_into") else None
        s = plan.execute(st, timed=True)
        best = min(best, s.pass_ms)
    return plan, st, best


specs = eval(os.environ.get("QG_CFGS", "[dict(kernel_cfg=1), dict(kernel_cfg=5)]"))
ns = [int(x) for x in sys.argv[1:]] or [28]
for n in ns:
    for kind in ("random", "qft"):
        gt, gp = random_arrays(RandomSpec(n, 1000, 0)) if kind == "random" else qft_arrays(n)
        ref = None
        for kw in specs:
            prec = os.environ.get("QG_PREC", "fp32")
            plan, st, ms = run(gt, gp, n, prec, **kw)
            S = (1 << n) * (8 if prec == "fp32" else 16)
            out = dict(kind=kind, n=n, kw=kw, passes=plan.info["n_passes"], stages=plan.info["n_stages"],
                       cxm=plan.info["n_cxm"], ms=round(ms, 3), ms_per_pass=round(ms / plan.info["n_passes"], 4),
                       gbs=round(2 * S * plan.info["n_passes"] / ms / 1e6, 1), gates_per_s=round(gt.shape[0] / ms * 1e3))
            if n <= 28:
                # states after 1 + reps executions must agree between configurations
                v = st.amplitudes.to(torch.complex128)
                if ref is None:
                    ref = v
                else:
                    out["rel_vs_first"] = float((v - ref).norm() / ref.norm())
            print(json.dumps(out), flush=True)
            del st
