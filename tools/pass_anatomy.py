"""Per-pass anatomy of a fused plan (dev probe, CPU-runnable): the physical qubits the
stage headers of each pass map into registers, the contiguous low run those make, and
the op counts per kind.  With --time (GPU) it also times each pass alone with CUDA
events by executing single-pass copies of the plan is not possible through the C-ABI,
so the per-launch times come from an ncu launch list of tools/jit_time.py instead."""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_03967_b200 import statevec as sv  # noqa: E402
from paper_2504_03967_b200.generators import RandomSpec, qft_arrays, random_arrays  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
kind = sys.argv[2] if len(sys.argv) > 2 else "random"
gt, gp = random_arrays(RandomSpec(n, 1000, 0)) if kind == "random" else qft_arrays(n)
plan = sv.CompiledCircuit(gt, gp, n, "fp32", jit=0)
rec, mats = plan.export()
names = {0: "RD", 1: "CD", 2: "PH", 3: "CXM", 4: "PH2", 5: "XF", 6: "TPH"}
passes = collections.OrderedDict()
for r in rec:
    p, s, k = int(r[0]), int(r[1]), int(r[2])
    d = passes.setdefault(p, {"qubits": set(), "stages": 0, "ops": collections.Counter()})
    if k == 200:
        d["stages"] += 1
        row = mats[int(r[7])] if r[7] >= 0 else []
        for j in range(int(r[3])):
            d["qubits"].add(int(row[j]))
    elif k in names:
        d["ops"][names[k]] += 1
for p, d in passes.items():
    q = sorted(d["qubits"])
    low = 0
    while low in d["qubits"]:
        low += 1
    print(json.dumps({"pass": p, "stages": d["stages"], "reg_qubits": q, "low_run": low,
                      "ops": dict(d["ops"]), "n_ops": sum(d["ops"].values())}))
