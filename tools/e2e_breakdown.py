"""Where the e2e time of bench.py's run_circuit leg goes (dev probe, GPU): the public call
split into its phases, each bracketed by a device synchronize (so the sum is slightly
above the overlapped call)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03967_b200 import statevec as sv  # noqa: E402
from paper_2504_03967_b200.generators import RandomSpec, generate_random_gate_list  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
shots = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
circ = generate_random_gate_list(RandomSpec(n, 1000, 0))
opts = sv.SimOptions(precision="fp32", shots=shots, rng_seed=0, memory_budget=1 << 45, device=0)
sv.run_circuit(circ, opts)  # warm: cubin cache, allocator
torch.cuda.synchronize()
for rep in range(3):
    t = {}
    t0 = time.perf_counter()
    s = time.perf_counter(); w = time.perf_counter()
    st, counts = sv.run_circuit(circ, opts)
    torch.cuda.synchronize()
    t["run_circuit"] = time.perf_counter() - s
    s = time.perf_counter()
    gt, gp, nq = sv.circuit_arrays(circ)
    t["arrays"] = time.perf_counter() - s
    s = time.perf_counter()
    plan = sv.CompiledCircuit(gt, gp, nq, "fp32", jit=opts.jit)
    t["plan"] = time.perf_counter() - s
    s = time.perf_counter()
    del st
    state = sv.init_zero_state(nq, "fp32", opts.memory_budget, 0)
    torch.cuda.synchronize()
    t["init"] = time.perf_counter() - s
    s = time.perf_counter()
    plan.execute(state)
    torch.cuda.synchronize()
    t["execute"] = time.perf_counter() - s
    s = time.perf_counter()
    idx, cnt = sv.sample_indices(state.amplitudes, shots, 0, "philox", sv.NORM_TOL["fp32"])
    torch.cuda.synchronize()
    t["sample_device"] = time.perf_counter() - s
    s = time.perf_counter()
    a, b = idx.cpu().numpy(), cnt.cpu().numpy()
    t["d2h"] = time.perf_counter() - s
    s = time.perf_counter()
    sv.counts_from_arrays(a, b, shots, nq)
    t["counts_dict"] = time.perf_counter() - s
    del state
    print(json.dumps({k: round(v * 1e3, 2) for k, v in t.items()}), flush=True)
