"""C1 (16q c128 x 100 blocks + 3000 shots) CUDA-graph replay with the interpreter vs the JIT
pass kernels (dev probe)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_03967_b200 import statevec as sv  # noqa: E402
from paper_2504_03967_b200.generators import RandomSpec, random_arrays  # noqa: E402

gt, gp = random_arrays(RandomSpec(16, 100, 0))
ref = None
for jit in (-1, 1):
    plan = sv.CompiledCircuit(gt, gp, 16, "fp64", jit=jit)
    js = plan.jit_status(wait=True)
    g = sv.CircuitGraph(plan, 3000, 0)
    for _ in range(10):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    _, counts = g.result()
    same = ref is None or counts.counts == ref
    ref = ref or counts.counts
    print(f"jit={jit} n_jit={js['n_jit']}/{js['n_passes']} replay {e0.elapsed_time(e1) / 200 * 1000:.1f} us "
          f"counts same as interpreter: {same}", flush=True)
