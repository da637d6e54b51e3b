"""Run one planned circuit a couple of times (target for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_03967_b200 import statevec as sv
from paper_2504_03967_b200.generators import RandomSpec, random_arrays, qft_arrays

n = int(os.environ.get("QG_N", "26"))
kind = os.environ.get("QG_KIND", "random")
prec = os.environ.get("QG_PREC", "fp32")
kw = eval(os.environ.get("QG_KW", "{}"))
gt, gp = random_arrays(RandomSpec(n, int(os.environ.get("QG_BLOCKS", "200")), 0)) if kind == "random" else qft_arrays(n)
plan = sv.CompiledCircuit(gt, gp, n, prec, **kw)
print(plan.info, flush=True)
st = sv.init_zero_state(n, prec, 1 << 40)
for _ in range(int(os.environ.get("QG_REPS", "2"))):
    plan.execute(st)
torch.cuda.synchronize()
print("norm", st.norm_sq())
