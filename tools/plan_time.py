"""Planner wall time and pass count for the 32 q random circuit (dev probe; QG_DEV_TILE_K
sets the independent tile searches per pass)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03967_b200 import statevec as sv  # noqa: E402
from paper_2504_03967_b200.generators import RandomSpec, random_arrays  # noqa: E402

out = {"K": os.environ.get("QG_DEV_TILE_K", "8"), "cpus": os.cpu_count()}
for seed in (0, 1, 2):
    gt, gp = random_arrays(RandomSpec(32, 1000, seed))
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        p = sv.CompiledCircuit(gt, gp, 32, "fp32", jit=-1)
        ts.append(time.perf_counter() - t)
        n = p.info["n_passes"]
        del p
    out[f"seed{seed}"] = {"passes": n, "plan_ms": round(min(ts) * 1e3, 1)}
print(json.dumps(out), flush=True)
