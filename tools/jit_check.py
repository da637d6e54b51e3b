"""JIT pass kernels vs the op-stream interpreter on the GPU: bit-exact states and
device time per circuit (dev tool; the committed checks are in tests/)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2504_03967_b200 import statevec as sv  # noqa: E402
from paper_2504_03967_b200.generators import RandomSpec, qft_arrays, random_arrays  # noqa: E402


def run(gt, gp, n, jit, reps=1):
    plan = sv.CompiledCircuit(gt, gp, n, "fp32", jit=jit)
    st = plan.jit_status(wait=True)
    state = sv.init_zero_state(n, "fp32", 1 << 40)
    ms = []
    for _ in range(reps):
        state = sv.init_zero_state(n, "fp32", 1 << 40) if reps > 1 else state
        torch.cuda.synchronize()
        s = plan.execute(state, timed=True)
        ms.append(s.pass_ms)
    return state.amplitudes, min(ms), plan.info["n_passes"], st


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [20, 24, 26]
    for n in sizes:
        for kind in ("random", "qft"):
            gt, gp = random_arrays(RandomSpec(n, 1000 if n >= 24 else 300, 1)) if kind == "random" else qft_arrays(n)
            reps = 3 if n >= 28 else 1
            a0, t0, npass, _ = run(gt, gp, n, -1, reps)
            a0 = a0.clone()
            a1, t1, _, st = run(gt, gp, n, 1, reps)
            same = torch.equal(torch.view_as_real(a0), torch.view_as_real(a1))
            diff = (a0 - a1).abs().max().item()
            print(f"n={n} {kind}: passes {npass} jit {st['n_jit']}/{st['n_passes']} fallback {st['n_fallback']} "
                  f"bitexact={same} maxdiff={diff:.3e} interp {t0:.2f} ms jit {t1:.2f} ms "
                  f"compile sum {st['compile_ms_sum']:.0f} ms wall {st['compile_ms_wall']:.0f} ms threads {st['threads']}",
                  flush=True)
            del a0, a1
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
