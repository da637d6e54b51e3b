"""JIT vs interpreter on the 16-warp complex64 tile (kernel_cfg=1, dev probe QG_DEV_JIT_CFG0)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_03967_b200 import statevec as sv  # noqa: E402
from paper_2504_03967_b200.generators import RandomSpec, qft_arrays, random_arrays  # noqa: E402

for n in (24, 28):
    for kind in ("random", "qft"):
        gt, gp = random_arrays(RandomSpec(n, 300, 1)) if kind == "random" else qft_arrays(n)
        out = []
        for jit in (-1, 1):
            plan = sv.CompiledCircuit(gt, gp, n, "fp32", jit=jit, kernel_cfg=1)
            js = plan.jit_status(wait=True)
            st = sv.init_zero_state(n, "fp32")
            plan.execute(st)
            torch.cuda.synchronize()
            out.append((st.amplitudes.clone(), js["n_jit"]))
        same = torch.equal(torch.view_as_real(out[0][0]), torch.view_as_real(out[1][0]))
        print(f"n={n} {kind}: jit {out[1][1]} bitexact={same}", flush=True)
