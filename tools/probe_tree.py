"""Tree-sampler timing by phase (dev probe): prepare / draw (compact and dense)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2504_03967_b200 import statevec as sv  # noqa: E402
from paper_2504_03967_b200.generators import RandomSpec, qft_arrays, random_arrays  # noqa: E402


def ev(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for n, kind, shots in [(28, "qft", 100_000), (24, "random", 100_000), (24, "random", 50_000_000_000),
                       (28, "random", 10**9)]:
    gt, gp = qft_arrays(n) if kind == "qft" else random_arrays(RandomSpec(n, 200, 0))
    plan = sv.CompiledCircuit(gt, gp, n, "fp32")
    st = sv.init_zero_state(n, "fp32", 1 << 40)
    plan.execute(st)
    ts = sv.TreeSampler(st.amplitudes)
    t_prep = ev(ts.prepare_async)
    t_draw = ev(lambda: ts.draw(shots, 1), 2)
    t_dense = ev(lambda: ts.draw(shots, 1, dense=True), 2)
    print(f"n={n} {kind} shots={shots:.3g}: prepare {t_prep:.3f} ms, draw {t_draw:.3f} ms, dense {t_dense:.3f} ms",
          flush=True)
