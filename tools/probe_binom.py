"""Binomial generator throughput (dev probe): 2^24 draws per (n, p) on the device."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_03967_b200 import _native as N  # noqa: E402
from paper_2504_03967_b200 import statevec as sv  # noqa: E402

cnt = 1 << 24
out = torch.empty(cnt, dtype=torch.int64, device="cuda")
for n, p in [(5, 0.3), (12, 0.5), (40, 0.5), (100, 0.3), (3000, 0.5), (10**6, 0.5), (5e10, 0.5), (1e9, 1e-9)]:
    f = lambda: N.call("qg_binomial_test", float(n), float(p), 1, cnt, sv.C.c_void_p(out.data_ptr()),  # noqa: E731
                       sv._stream(out.device))
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    f()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"n={n:g} p={p:g}: {ms:.3f} ms for 2^24 draws = {ms * 1e6 / cnt:.2f} ns/draw, mean {out.double().mean().item():.4g}",
          flush=True)
