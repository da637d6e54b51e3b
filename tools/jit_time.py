"""Device time per fused pass of the JIT kernels for one circuit (dev probe; the
kernel variant comes from QG_JIT_VARIANT, read once per process)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03967_b200 import statevec as sv  # noqa: E402
from paper_2504_03967_b200.generators import RandomSpec, qft_arrays, random_arrays  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
kind = sys.argv[2] if len(sys.argv) > 2 else "random"
kw = eval(os.environ.get("QG_KW", "{}"))
gt, gp = random_arrays(RandomSpec(n, 1000, 0)) if kind == "random" else qft_arrays(n)
plan = sv.CompiledCircuit(gt, gp, n, "fp32", jit=1, **kw)
js = plan.jit_status(wait=True)
st = sv.init_zero_state(n, "fp32", 1 << 40)
plan.execute(st)
torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    best = min(best, plan.execute(st, timed=True).pass_ms)
S = (1 << n) * 8
p = plan.info["n_passes"]
print(json.dumps(dict(variant=os.environ.get("QG_JIT_VARIANT", "0"), kind=kind, n=n, kw=kw, passes=p,
                      jit=js["n_jit"], ms=round(best, 2), ms_per_pass=round(best / p, 3),
                      gbs=round(2 * S * p / best / 1e6, 1))), flush=True)
