"""Device time of the sampler stages (prefix pass, draws + sort) at N qubits (dev probe).
usage: python tools/probe_sample.py N [SHOTS]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_03967_b200 import statevec as sv

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
shots = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
st = sv.init_zero_state(n, "fp32", 1 << 40)
a = torch.randn(1 << n, dtype=torch.complex64, device=st.amplitudes.device)
st.amplitudes.copy_(a / torch.linalg.vector_norm(a.view(torch.float32).double()).float())
for _ in range(3):
    sv.sample_indices(st.amplitudes, shots, 0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 10
e0.record()
for _ in range(reps):
    sv.sample_indices(st.amplitudes, shots, 0)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
gb = (1 << n) * 8 / 1e9
print({"n": n, "shots": shots, "ms": round(ms, 4), "state_read_GBps": round(gb / ms * 1e3, 1)})
