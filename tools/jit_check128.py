"""complex128 JIT pass kernels vs the interpreter on the GPU (dev tool): relative
L2 difference of the final states and device time per circuit."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_03967_b200 import statevec as sv  # noqa: E402
from paper_2504_03967_b200.generators import RandomSpec, qft_arrays, random_arrays  # noqa: E402


def run(gt, gp, n, jit, reps):
    plan = sv.CompiledCircuit(gt, gp, n, "fp64", jit=jit)
    st = plan.jit_status(wait=True)
    best = 1e9
    for _ in range(reps):
        state = sv.init_zero_state(n, "fp64", 1 << 40)
        torch.cuda.synchronize()
        best = min(best, plan.execute(state, timed=True).pass_ms)
    return state.amplitudes, best, plan.info["n_passes"], st


for n in [int(x) for x in sys.argv[1:]] or [20, 24, 28]:
    for kind in ("random", "qft"):
        gt, gp = random_arrays(RandomSpec(n, 1000 if n >= 24 else 300, 1)) if kind == "random" else qft_arrays(n)
        reps = 3 if n >= 28 else 1
        a0, t0, npass, _ = run(gt, gp, n, -1, reps)
        a0 = a0.clone()
        a1, t1, _, st = run(gt, gp, n, 1, reps)
        rel = ((a0 - a1).norm() / a0.norm()).item()
        S = (1 << n) * 16
        print(f"n={n} {kind} c128: passes {npass} jit {st['n_jit']}/{st['n_passes']} rel_l2 {rel:.2e} "
              f"interp {t0:.2f} ms jit {t1:.2f} ms ({2 * S * npass / t1 / 1e6:.0f} GB/s) "
              f"compile wall {st['compile_ms_wall']:.0f} ms", flush=True)
        del a0, a1
        torch.cuda.empty_cache()
